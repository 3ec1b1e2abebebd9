"""Short device-resident f+grad loop for ncu captures (never a bench number)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1911_03813_b200 as mcp  # noqa: E402
from paper_1911_03813_b200 import _native, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--evals", type=int, default=4)
ap.add_argument("--p", type=int, default=None)
ap.add_argument("--dnorm", action="store_true")
ap.add_argument("--mode", default=None)
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
V = synth.device_observations(cfg, 2024, p=a.p)
obs = mcp.ObservationSet.from_device(V, p_total=V.shape[0], release=True)
del V
ctx = obs.device_context()
torch.cuda.empty_cache()   # the released upload source goes back to the driver (V_lo needs it)
if a.dnorm:
    for _ in range(a.evals):
        print("dnorm", ctx.data_norm_sq(cfg.d, None), ctx.last_variant)
else:
    lam, A = synth.initial_point(cfg, 2024)
    x = torch.as_tensor(mcp.pack(lam, A), device="cuda")
    out = torch.empty(1 + cfg.r + cfg.n * cfg.r, dtype=torch.float64, device="cuda")
    s = _native.stream_handle(torch.cuda.current_stream())
    for _ in range(a.evals):
        ctx.fg_device(cfg.d, cfg.r, x.data_ptr(), 0.0, a.mode, out.data_ptr(), s)
    torch.cuda.synchronize()
    print("f", float(out[0]), ctx.last_variant)
