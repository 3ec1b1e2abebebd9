"""Warm device-resident f+grad latency over small shapes: K1Z (single launch) against the general
K1 -> reduce+finish chain (MCP_OPT_SMALL_KERNEL = 0), CUDA-event timed over back-to-back
evaluations (the optimizer-loop regime: V, x and the code stay in L2).  One line per shape."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_1911_03813_b200 as mcp
from paper_1911_03813_b200 import _native

SHAPES = [(20, 5, 3, 10000), (20, 5, 3, 1000), (20, 5, 3, 100), (100, 10, 4, 3000),
          (100, 10, 4, 300), (500, 10, 3, 10), (500, 10, 3, 100), (500, 10, 3, 1000),
          (500, 10, 3, 3000), (256, 16, 3, 2000), (64, 8, 4, 20000), (128, 4, 3, 500)]


def time_evals(ctx, d, r, x, out, s, iters=300):
    for _ in range(20):
        ctx.fg_device(d, r, x.data_ptr(), 0.0, None, out.data_ptr(), s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        ctx.fg_device(d, r, x.data_ptr(), 0.0, None, out.data_ptr(), s)
    e1.record()
    torch.cuda.synchronize()
    return 1e3 * e0.elapsed_time(e1) / iters


def main():
    rng = np.random.default_rng(0)
    shapes = SHAPES
    if len(sys.argv) > 1:   # "n,r,d,p n,r,d,p ..."
        shapes = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]]
    for n, r, d, p in shapes:
        V = rng.standard_normal((n, p)) / np.sqrt(n)
        obs = mcp.ObservationSet(V)
        ctx = obs.device_context()
        lam, A = rng.standard_normal(r), rng.standard_normal((n, r)) / np.sqrt(n)
        x = torch.as_tensor(mcp.pack(lam, A), device="cuda")
        out = torch.empty(1 + r + n * r, dtype=torch.float64, device="cuda")
        s = _native.stream_handle(torch.cuda.current_stream())
        res = {}
        for small in (1, 0):
            ctx.set_option(_native.MCP_OPT_SMALL_KERNEL, small)
            us = time_evals(ctx, d, r, x, out, s)
            res["k1z" if small else "general"] = {"us": round(us, 2), "kernel": ctx.last_variant,
                                                  "launches": ctx.last_launch_count}
        print(json.dumps({"n": n, "r": r, "d": d, "p": p, **res}), flush=True)


if __name__ == "__main__":
    main()
