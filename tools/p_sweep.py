"""ms per device-resident f+grad evaluation versus p (fixed/marginal cost split of K1).

  python tools/p_sweep.py --config c2 [--mode fp64] [--ps 125000,250000,...]
"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1911_03813_b200 as mcp  # noqa: E402
from paper_1911_03813_b200 import _native, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--mode", default=None)
ap.add_argument("--ps", default="62500,125000,250000,500000,1000000,2000000")
ap.add_argument("--steps", type=int, default=100)
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
stream = torch.cuda.current_stream()
sh = _native.stream_handle(stream)
rows = []
for p in [int(v) for v in a.ps.split(",")]:
    V = synth.device_observations(cfg, 2024, p=p)
    obs = mcp.ObservationSet.from_device(V, p_total=p)
    ctx = obs.device_context()
    lam, A = synth.initial_point(cfg, 2024)
    x = torch.as_tensor(mcp.pack(lam, A), device="cuda")
    out = torch.empty(1 + cfg.r + cfg.n * cfg.r, dtype=torch.float64, device="cuda")
    ts = []
    for rep in range(3):
        for _ in range(5):
            ctx.fg_device(cfg.d, cfg.r, x.data_ptr(), 0.0, a.mode, out.data_ptr(), sh)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(a.steps):
            ctx.fg_device(cfg.d, cfg.r, x.data_ptr(), 0.0, a.mode, out.data_ptr(), sh)
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / a.steps)
    ms = statistics.median(ts)
    bytes_ = p * cfg.n * (8 if cfg.dtype == "f64" else 4)
    print(f"p={p:9d}  {ms * 1e3:9.2f} us/eval  {bytes_ / ms / 1e6:8.1f} GB/s  variant={ctx.last_variant}",
          flush=True)
    del obs, ctx, V
    torch.cuda.empty_cache()
