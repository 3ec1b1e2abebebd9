"""Stochastic path at the paper's Table 2 workload (synth config t2:
n=500, p=500,000, r=10, d=3, epoch 100, estimate on 1000 rows), batch s in {10, 100, 1000}.

device : mcp.adam_minimize (gather + f+grad + Adam update per iteration, one graph each)
cpu    : the restated reference Adam (oracle/adam_oracle.py, numpy) for a bounded number of
         epochs -- the reference's own per-iteration cost on this host.
Prints one JSON line per batch size with inner iterations/s for both.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np

import paper_1911_03813_b200 as mcp
from paper_1911_03813_b200 import synth
from oracle import adam_oracle as ao


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", default="10,100,1000")
    ap.add_argument("--epochs", type=int, default=30)
    ap.add_argument("--cpu-epochs", type=int, default=2)
    args = ap.parse_args()
    cfg = synth.CONFIGS["t2"]
    V = synth.host_observations(cfg, 0)
    lam, A = synth.initial_point(cfg, 0)
    x0 = mcp.pack(lam, A)
    obs = mcp.ObservationSet(V)
    for s in [int(b) for b in args.batches.split(",")]:
        ac = mcp.AdamConfig(batch=s, max_epochs=args.epochs)
        mcp.adam_minimize(obs, cfg.d, cfg.r, x0, mcp.AdamConfig(batch=s, max_epochs=1),
                          np.random.default_rng(1))  # warm-up
        t = time.perf_counter()
        rep = mcp.adam_minimize(obs, cfg.d, cfg.r, x0, ac, np.random.default_rng(1))
        td = time.perf_counter() - t
        t = time.perf_counter()
        host = (ao.adam(V, cfg.d, cfg.r, x0, np.random.default_rng(1), batch=s,
                        max_epochs=args.cpu_epochs) if args.cpu_epochs > 0 else {"n_iter": 0})
        th = time.perf_counter() - t
        print(json.dumps({
            "workload": "t2 (paper Table 2)", "batch": s,
            "device": {"inner_iters": rep.n_fg, "epochs": len(rep.trace) - 1, "s": td,
                       "iters_per_s": rep.n_fg / td, "us_per_iter": 1e6 * td / rep.n_fg,
                       # epochs only (sampling callback + graph replays + estimate), no set-up
                       "us_per_iter_steady": 1e6 * (rep.trace[-1][1] - rep.trace[0][1]) / rep.n_fg,
                       "reason": rep.reason, "f": rep.f},
            "cpu_port": {"inner_iters": host["n_iter"], "s": th,
                         "iters_per_s": host["n_iter"] / th,
                         "us_per_iter": 1e6 * th / host["n_iter"] if host["n_iter"] else None,
                         "threads": os.cpu_count()},
        }), flush=True)


if __name__ == "__main__":
    main()
