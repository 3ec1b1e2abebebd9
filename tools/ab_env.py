"""In-process A/B of environment toggles on the device-resident f+grad loop (kernel experiments).

  python tools/ab_env.py --config c2 --steps 50 --reps 5 VAR=VALUE [VAR2=VALUE ...]
Alternates the baseline (no toggles) and each toggle, CUDA-event timed, and prints the median
ms/step of each.  Toggles are read by the library at launch time (e.g. MCP_NO_FUSED_TAIL=1).
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
ap.add_argument("--steps", type=int, default=50)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--mode", default=None)
ap.add_argument("--p", type=int, default=None)
ap.add_argument("--timing", action="store_true", help="per-launch kernel event timing on")
ap.add_argument("toggles", nargs="*")
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
V = synth.device_observations(cfg, 2024, p=a.p)
obs = mcp.ObservationSet.from_device(V, p_total=V.shape[0])
ctx = obs.device_context()
lam, A = synth.initial_point(cfg, 2024)
x = torch.as_tensor(mcp.pack(lam, A), device="cuda")
out = torch.empty(1 + cfg.r + cfg.n * cfg.r, dtype=torch.float64, device="cuda")
stream = torch.cuda.current_stream()
sh = _native.stream_handle(stream)
if a.timing:
    ctx.set_kernel_timing(True)
variants = [("base", {})] + [(t, dict(kv.split("=", 1) for kv in t.split(","))) for t in a.toggles]
res = {name: [] for name, _ in variants}
vnames = {}
outs = {}
for rep in range(a.reps):
    for name, env in variants:
        for k, v in env.items():
            os.environ[k] = v
        for _ in range(3):
            ctx.fg_device(cfg.d, cfg.r, x.data_ptr(), 0.0, a.mode, out.data_ptr(), sh)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(a.steps):
            ctx.fg_device(cfg.d, cfg.r, x.data_ptr(), 0.0, a.mode, out.data_ptr(), sh)
        e1.record(stream)
        torch.cuda.synchronize()
        res[name].append(e0.elapsed_time(e1) / a.steps)
        outs[name] = out.clone()
        vnames[name] = ctx.last_variant
        for k in env:
            del os.environ[k]
ref = None
if a.mode not in (None, "fp64"):
    ref = torch.empty_like(out)
    ctx.fg_device(cfg.d, cfg.r, x.data_ptr(), 0.0, "fp64", ref.data_ptr(), sh)
    torch.cuda.synchronize()
for name, _ in variants:
    v = res[name]
    same = torch.equal(outs[name], outs["base"])
    err = ""
    if ref is not None:
        o = outs[name]
        err = (f"  rel_err_vs_fp64 f {abs(float(o[0] - ref[0])) / abs(float(ref[0])):.2e}"
               f" g {float((o[1:] - ref[1:]).norm() / ref[1:].norm()):.2e}")
    print(f"{name:30s} median {statistics.median(v):.4f} ms  min {min(v):.4f}  "
          f"bitwise_equal_to_base={same}{err}  variant={vnames[name]}")
