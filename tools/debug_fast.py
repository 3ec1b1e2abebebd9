"""Localise fast-mode (tf32x3) errors: Y from mode=tf32x3 vs fp64 for small shapes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1911_03813_b200 as mcp

for (n, p, r, d) in [(32, 128, 16, 2), (32, 256, 16, 2), (64, 128, 16, 2), (128, 128, 16, 2),
                     (32, 128, 16, 3), (100, 1000, 10, 4), (160, 300, 40, 3)]:
    rng = np.random.default_rng(0)
    V = rng.standard_normal((n, p)).astype(np.float32)
    A = rng.standard_normal((n, r))
    obs = mcp.ObservationSet(V)
    Y64 = mcp.ttsv_batch(obs, A, d)
    Yf = mcp.ttsv_batch(obs, A, d, mode="tf32x3")
    err = np.abs(Yf - Y64) / (np.abs(Y64).max() + 1e-300)
    print(f"n={n} p={p} r={r} d={d}: max rel {err.max():.2e}; variant {obs.device_context().last_variant}")
    if err.max() > 1e-5:
        rows = err.max(axis=1); cols = err.max(axis=0)
        print("  worst rows (i):", np.argsort(-rows)[:8], rows[np.argsort(-rows)[:8]])
        print("  worst cols (j):", np.argsort(-cols)[:8])
        print("  Y64[0,:4]", Y64[0, :4], "Yf[0,:4]", Yf[0, :4])
        print("  ratio Yf/Y64 [0:4,0]", (Yf[:4, 0] / Y64[:4, 0]))
