"""Per-call latency of the public host path (packed_fg_implicit) -- e2e components."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1911_03813_b200 as mcp
from paper_1911_03813_b200 import synth

for name in sys.argv[1:] or ["c1", "c2"]:
    cfg = synth.CONFIGS[name]
    V = synth.host_observations(cfg, 0)
    lam, A = synth.initial_point(cfg, 0)
    fg = mcp.packed_fg_implicit(mcp.ObservationSet(V), cfg.d, cfg.r)
    x = mcp.pack(lam, A)
    for _ in range(20):
        fg(x)
    best = []
    for rep in range(5):
        t = time.perf_counter()
        for _ in range(200):
            fg(x)
        best.append((time.perf_counter() - t) / 200)
    print(f"{name}: e2e {1e6 * min(best):.1f} us/eval  ({1 / min(best):.0f} evals/s)")
