"""Throughput of batched multistart f+grad at a config (k starts per pass), host API e2e."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1911_03813_b200 as mcp
from paper_1911_03813_b200 import synth

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--ks", default="1,2,4,8,16")
ap.add_argument("--steps", type=int, default=50)
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
V = synth.device_observations(cfg, 2024)
obs = mcp.ObservationSet.from_device(V, p_total=cfg.p)
res = {}
for k in [int(x) for x in a.ks.split(",")]:
    X = np.stack([mcp.pack(*synth.initial_point(cfg, 2024 + s)) for s in range(k)])
    fg = mcp.packed_fg_implicit_batched(obs, cfg.d, cfg.r)
    for _ in range(3):
        fg(X)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(a.steps):
        F, G = fg(X)
    dt = (time.perf_counter() - t0) / a.steps
    res[k] = {"ms_per_batch": dt * 1e3, "evals_per_s": k / dt,
              "kernel": obs.device_context().last_variant}
    print(json.dumps({"config": a.config, "k": k, **res[k]}), flush=True)
