"""Device L-BFGS per-step time on small problems (a c1-like set and an n = 200 set solved on the
single-launch K1Z path), for A/B builds selected with MCP_LIBRARY."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np

import paper_1911_03813_b200 as mcp


def main():
    rng = np.random.default_rng(3)
    for n, p, r, d in ((20, 10_000, 5, 3), (200, 2_000, 10, 3), (100, 3_000, 10, 4)):
        means = rng.standard_normal((n, r))
        means /= np.linalg.norm(means, axis=0)
        V = means[:, rng.integers(0, r, p)] + 0.1 * rng.standard_normal((n, p))
        obs = mcp.ObservationSet(V)
        A0 = rng.standard_normal((n, r))
        x0 = mcp.pack(np.full(r, 1.0 / r), A0 / np.linalg.norm(A0, axis=0))
        fg = mcp.packed_fg_implicit(obs, d, r)
        cfg = mcp.OptConfig(max_iters=60, pgtol=1e-12)
        mcp.lbfgs_minimize(fg, x0, mcp.OptConfig(max_iters=3))
        best = None
        for _ in range(5):
            t = time.perf_counter()
            rep = mcp.lbfgs_minimize(fg, x0, cfg)
            dt = time.perf_counter() - t
            best = dt if best is None else min(best, dt)
        print(json.dumps({"n": n, "p": p, "r": r, "N": r + n * r, "steps": rep.n_steps,
                          "n_fg": rep.n_fg, "us_per_step": round(1e6 * best / rep.n_steps, 2),
                          "us_per_eval": round(1e6 * best / rep.n_fg, 2), "f": rep.f,
                          "kernel": obs.device_context().last_variant}), flush=True)


if __name__ == "__main__":
    main()
