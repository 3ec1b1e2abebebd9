"""Device-resident L-BFGS vs the host-driven solver with the same GPU f+grad.

Prints one JSON line per config: evaluations/s and ms per L-BFGS step for
  device : mcp.lbfgs_minimize (mcp_lbfgs: x, g, history on the GPU, scalars to the host)
  host   : the restated reference loop (oracle/lbfgs_oracle.py, numpy on the host) calling
           packed_fg_implicit -- the reference's own solver structure on the B200 f+grad.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden"))

import numpy as np

import paper_1911_03813_b200 as mcp
from paper_1911_03813_b200 import synth
from oracle import lbfgs_oracle as lo


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2")
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--mode", default="fp64")
    ap.add_argument("--pgtol", type=float, default=1e-4)
    ap.add_argument("--skip-host", action="store_true")
    ap.add_argument("--k", type=int, default=0, help="also time k lock-step starts")
    args = ap.parse_args()
    for name in args.configs.split(","):
        cfg = synth.CONFIGS[name]
        V = synth.host_observations(cfg, 0)
        lam, A = synth.initial_point(cfg, 0)
        obs = mcp.ObservationSet(V)
        fg = mcp.packed_fg_implicit(obs, cfg.d, cfg.r, mode=args.mode)
        x0 = mcp.pack(lam, A)
        oc = mcp.OptConfig(max_iters=args.iters, pgtol=args.pgtol)
        mcp.lbfgs_minimize(fg, x0, mcp.OptConfig(max_iters=3))  # warm-up (graphs, buffers)
        t = time.perf_counter()
        dev = mcp.lbfgs_minimize(fg, x0, oc)
        td = time.perf_counter() - t
        fg(x0)
        t = time.perf_counter()
        host = (lo.lbfgs(fg, x0, max_iters=args.iters, pgtol=args.pgtol) if not args.skip_host
                else {"n_fg": 0, "n_steps": 0, "f": None})
        th = time.perf_counter() - t
        batched = None
        if args.k > 1:
            rng = np.random.default_rng(5)
            X0 = np.stack([x0] + [mcp.pack(lam, rng.standard_normal(A.shape) / np.sqrt(cfg.n))
                                  for _ in range(args.k - 1)])
            mcp.lbfgs_minimize_batched(fg, X0, mcp.OptConfig(max_iters=2))   # warm-up
            t = time.perf_counter()
            reps = mcp.lbfgs_minimize_batched(fg, X0, oc)
            tb = time.perf_counter() - t
            ev = sum(rp.n_fg for rp in reps)
            batched = {"k": args.k, "n_fg_total": ev, "s": tb, "evals_per_s": ev / tb,
                       "steps": [rp.n_steps for rp in reps]}
        print(json.dumps({
            "config": name, "mode": args.mode, "iters": args.iters, "batched": batched,
            "device": {"n_fg": dev.n_fg, "n_steps": dev.n_steps, "s": td,
                       "evals_per_s": dev.n_fg / td, "ms_per_step": 1e3 * td / max(dev.n_steps, 1),
                       "f": dev.f},
            "host": {"n_fg": host["n_fg"], "n_steps": host["n_steps"], "s": th,
                     "evals_per_s": host["n_fg"] / th,
                     "ms_per_step": 1e3 * th / max(host["n_steps"], 1), "f": host["f"]},
        }), flush=True)


if __name__ == "__main__":
    main()
