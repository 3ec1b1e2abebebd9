import sys, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests/golden')
import numpy as np
import paper_1911_03813_b200 as mcp
from oracle import momentcp_oracle as om
rng = np.random.default_rng(27)
for it in range(8):
    n, p, r, d = int(rng.integers(2, 7)), int(rng.integers(2, 9)), int(rng.integers(1, 4)), int(rng.choice([2, 3, 4]))
    V = rng.standard_normal((n, p))
    obs = mcp.ObservationSet(V)
    lam = rng.uniform(0.5, 1.5, r) * rng.choice([-1.0, 1.0], r)
    A = rng.standard_normal((n, r)); A /= np.linalg.norm(A, axis=0)
    fg = mcp.packed_fg_implicit(obs, d, r)
    x = mcp.pack(lam, A)
    f1, g1 = fg(x); f2, g2 = fg(x)
    fo, go = om.packed_fg(V, np.full(p, 1/p), d, r)(x)
    print(it, n, p, r, d, "repeat-equal", f1 == f2 and np.array_equal(g1, g2), "f err", abs(f1 - fo), "g err", np.abs(g1 - go).max(), obs.device_context().last_variant)
    for i in range(x.size):
        e = np.zeros_like(x); e[i] = 1e-6
        fp = fg(x + e)[0]; fpo = om.packed_fg(V, np.full(p, 1/p), d, r)(x + e)[0]
        if abs(fp - fpo) > 1e-12 * max(1, abs(fpo)):
            print("   mismatch at perturbation", i, fp, fpo); break
