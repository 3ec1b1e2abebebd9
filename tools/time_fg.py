"""Device-resident f+grad timing for arbitrary shapes (kernel experiments, not bench numbers).

    python tools/time_fg.py n p r d [f32|f64] [fp64|tf32x3] ...   (groups of 6 arguments)
Prints ms per evaluation (CUDA events over 10 evaluations after 3 warm-ups), FP64 TF/s of the
4 n p r algorithmic flops and the kernel variant.
"""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_1911_03813_b200 as mcp  # noqa: E402
from paper_1911_03813_b200 import _native  # noqa: E402

args = sys.argv[1:]
for i in range(0, len(args), 6):
    n, p, r, d = (int(v) for v in args[i:i + 4])
    dt = torch.float32 if args[i + 4] == "f32" else torch.float64
    mode = args[i + 5]
    g = torch.Generator(device="cuda").manual_seed(1)
    V = (torch.randn(p, n, generator=g, device="cuda", dtype=torch.float32) / n ** 0.5).to(dt)
    obs = mcp.ObservationSet.from_device(V, release=True)
    del V
    ctx = obs.device_context()
    x = torch.randn(r + n * r, generator=g, device="cuda", dtype=torch.float64) / n ** 0.5
    out = torch.empty(1 + r + n * r, dtype=torch.float64, device="cuda")
    s = _native.stream_handle(torch.cuda.current_stream())
    for _ in range(3):
        ctx.fg_device(d, r, x.data_ptr(), 0.0, mode, out.data_ptr(), s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        ctx.fg_device(d, r, x.data_ptr(), 0.0, mode, out.data_ptr(), s)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"n={n} p={p} r={r} d={d} {args[i + 4]} {mode}: {ms:.3f} ms  "
          f"{4.0 * n * p * r / ms / 1e9:.2f} TF  {ctx.last_variant}", flush=True)
    del obs, ctx
    torch.cuda.empty_cache()
