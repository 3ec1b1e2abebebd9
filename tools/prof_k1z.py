"""Per-phase clocks of K1Z (build with tools/build_variant.py z_prof -DMCP_K1Z_PROF=1 and run with
MCP_LIBRARY pointing at it): a few warm device-resident evaluations of a synth config or a
(n, r, d, p) shape."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_1911_03813_b200 as mcp
from paper_1911_03813_b200 import _native


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="20,5,3,10000")
    ap.add_argument("--evals", type=int, default=4)
    args = ap.parse_args()
    n, r, d, p = (int(v) for v in args.shape.split(","))
    rng = np.random.default_rng(0)
    V = rng.standard_normal((n, p)) / np.sqrt(n)
    obs = mcp.ObservationSet(V)
    ctx = obs.device_context()
    lam, A = rng.standard_normal(r), rng.standard_normal((n, r)) / np.sqrt(n)
    x = torch.as_tensor(mcp.pack(lam, A), device="cuda")
    out = torch.empty(1 + r + n * r, dtype=torch.float64, device="cuda")
    s = _native.stream_handle(torch.cuda.current_stream())
    for k in range(args.evals):
        ctx.fg_device(d, r, x.data_ptr(), 0.0, None, out.data_ptr(), s)
        torch.cuda.synchronize()
        print(f"-- eval {k} {ctx.last_variant}", flush=True)


if __name__ == "__main__":
    main()
