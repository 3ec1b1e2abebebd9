"""Device time of one f+grad evaluation with the host out of the loop: N back-to-back evaluations
captured into ONE CUDA graph on the caller's stream (the library launches on the stream it is
given), replayed and CUDA-event timed.  This is the regime of the device-resident solvers."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_1911_03813_b200 as mcp
from paper_1911_03813_b200 import _native

SHAPES = [(20, 5, 3, 10000), (20, 5, 3, 1000), (100, 10, 4, 3000), (500, 10, 3, 1000),
          (500, 10, 3, 100), (500, 10, 3, 10), (500, 10, 3, 4000), (256, 16, 3, 2000),
          (500, 32, 3, 1000)]


def main():
    rng = np.random.default_rng(0)
    n_evals = 200
    for n, r, d, p in SHAPES:
        V = rng.standard_normal((n, p)) / np.sqrt(n)
        obs = mcp.ObservationSet(V)
        ctx = obs.device_context()
        lam, A = rng.standard_normal(r), rng.standard_normal((n, r)) / np.sqrt(n)
        x = torch.as_tensor(mcp.pack(lam, A), device="cuda")
        out = torch.empty(1 + r + n * r, dtype=torch.float64, device="cuda")
        side = torch.cuda.Stream()
        with torch.cuda.stream(side):
            s = _native.stream_handle(torch.cuda.current_stream())
            for _ in range(5):
                ctx.fg_device(d, r, x.data_ptr(), 0.0, None, out.data_ptr(), s)
            torch.cuda.synchronize()
            ref = out.clone()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                s = _native.stream_handle(torch.cuda.current_stream())
                for _ in range(n_evals):
                    ctx.fg_device(d, r, x.data_ptr(), 0.0, None, out.data_ptr(), s)
            for _ in range(3):
                g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                g.replay()
            e1.record()
            torch.cuda.synchronize()
        assert torch.equal(out, ref)
        print(json.dumps({"n": n, "r": r, "d": d, "p": p, "kernel": ctx.last_variant,
                          "launches": ctx.last_launch_count,
                          "us_per_eval_in_graph": round(1e3 * e0.elapsed_time(e1) / (5 * n_evals), 2)}),
              flush=True)


if __name__ == "__main__":
    main()
