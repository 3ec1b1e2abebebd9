"""Host-side cost of one device-resident evaluation call (Python -> ctypes -> plan -> launch):
wall clock per call of a long asynchronous run against the CUDA-event time of the same run, for a
small shape whose kernel is shorter than the call."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_1911_03813_b200 as mcp
from paper_1911_03813_b200 import _native


def main():
    rng = np.random.default_rng(0)
    for n, r, d, p in ((500, 10, 3, 100), (20, 5, 3, 1000)):
        V = rng.standard_normal((n, p)) / np.sqrt(n)
        obs = mcp.ObservationSet(V)
        ctx = obs.device_context()
        lam, A = rng.standard_normal(r), rng.standard_normal((n, r)) / np.sqrt(n)
        x = torch.as_tensor(mcp.pack(lam, A), device="cuda")
        out = torch.empty(1 + r + n * r, dtype=torch.float64, device="cuda")
        s = _native.stream_handle(torch.cuda.current_stream())
        xp, op = x.data_ptr(), out.data_ptr()
        for _ in range(50):
            ctx.fg_device(d, r, xp, 0.0, None, op, s)
        torch.cuda.synchronize()
        iters = 3000
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        t0 = time.perf_counter()
        for _ in range(iters):
            ctx.fg_device(d, r, xp, 0.0, None, op, s)
        t_host = time.perf_counter() - t0
        e1.record()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        for _ in range(iters):
            ctx.last_launch_count
        t_triv = time.perf_counter() - t1
        print(f"n={n} r={r} p={p} {ctx.last_variant}: host {1e6 * t_host / iters:.2f} us/call, "
              f"device {1e3 * e0.elapsed_time(e1) / iters:.2f} us/eval, trivial ABI call "
              f"{1e6 * t_triv / iters:.2f} us", flush=True)


if __name__ == "__main__":
    main()
