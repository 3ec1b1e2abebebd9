import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1911_03813_b200 as mcp
rng = np.random.default_rng(0)
n, p, r, d = 128, 200000, 32, 3
for kind in ["gauss", "tf32exact", "allpos"]:
    V = rng.standard_normal((n, p)).astype(np.float32)
    if kind == "tf32exact":
        V = (V.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)
    if kind == "allpos":
        V = np.abs(V) + 0.5
    lam = rng.standard_normal(r); A = rng.standard_normal((n, r))
    obs = mcp.ObservationSet(V)
    ref = mcp.fg_implicit(obs, lam, A, d)
    fast = mcp.fg_implicit(obs, lam, A, d, mode="tf32x3")
    e = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
    print(kind, "f", abs(fast.f - ref.f) / abs(ref.f), "g_lam", e(fast.g_lam, ref.g_lam), "g_A", e(fast.g_A, ref.g_A), flush=True)
