"""K1X (fp32 observations, n in (384, 512] and (768, 1024]: 16 warps, double-buffered TMA tiles,
resident factor block) and the other large-n FP64 kernels against the CPU oracle.

Covers the work split (groups of one CTA per column block striding the main tiles, block-major
ranges for the leftover CTAs -- including grids capped at the unit count for small p, and
zero-filled partial slots), ragged n and r, every order d, and bitwise determinism /
nu-linearity (the reference invariants, pkg/tests/test_implicit.py:53-57).  FP64 mode
tolerance: 1e-10 term-scale (pkg/tests/test_acceptance.py:65-74).
"""

import numpy as np
import pytest

import paper_1911_03813_b200 as mcp
from paper_1911_03813_b200 import _native
from oracle import momentcp_oracle as om

pytestmark = pytest.mark.gpu


def _case(n, p, r, d, seed, weights=False):
    rng = np.random.default_rng(seed)
    V = (rng.standard_normal((n, p)) / np.sqrt(n) + 0.3 * rng.standard_normal((n, 1)) / np.sqrt(n))
    V = V.astype(np.float32)
    nu = rng.uniform(0.5, 2.0, p) / p if weights else None
    lam = rng.standard_normal(r)
    A = rng.standard_normal((n, r)) / np.sqrt(n)
    return V, nu, lam, A


@pytest.mark.parametrize("n,p,r,d,k1x", [
    (512, 300_000, 64, 6, True),    # c3 shape: 4 blocks, 37 groups strided (148 CTAs)
    (512, 300_000, 96, 3, True),    # 6 blocks: 24 groups + 4 leftover CTAs on block-major ranges
    (512, 5_000, 64, 4, True),      # small p: grid capped at the unit count
    (512, 2_000, 16, 3, True),      # one column block, fewer tiles than SMs
    (400, 30_000, 20, 5, True),     # ragged n and r
    (512, 60_000, 48, 6, True),     # 3 blocks: 49 groups + 1 leftover CTA
    (500, 40_000, 40, 2, True),     # ragged n and r, d = 2
    (256, 50_000, 32, 5, False),    # n <= 384: the register-tiled K1
    (1024, 60_000, 256, 3, False),  # c5 shape: K1GT (Y partial in TMEM)
    (900, 20_000, 33, 4, False),    # large ragged n
    (700, 20_000, 20, 3, False),    # 512 < n <= 768: K1G
])
@pytest.mark.parametrize("weights", [False, True])
def test_large_n_fp32_vs_oracle(n, p, r, d, k1x, weights):
    V, nu, lam, A = _case(n, p, r, d, seed=n + p + r, weights=weights)
    obs = mcp.ObservationSet(V, nu)
    # the large-n kernels are the subject here: keep the smallest case off the single-launch K1Z
    obs.device_context().set_option(_native.MCP_OPT_SMALL_KERNEL, 0)
    res = mcp.fg_implicit(obs, lam, A, d, 0.3)
    assert obs.device_context().last_variant.startswith("k1x_fg_dmma") == k1x, \
        obs.device_context().last_variant
    V64 = V.astype(np.float64)
    nu64 = np.full(p, 1.0 / p) if nu is None else nu
    f, gl, gA = om.fg_implicit(V64, nu64, lam, A, d, 0.3)
    fs, gls, gAs, _ = om.term_scales(V64, nu64, lam, A, d, 0.3)
    e = max(om.term_rel_err(res.f, f, fs), om.term_rel_err(res.g_lam, gl, gls),
            om.term_rel_err(res.g_A, gA, gAs))
    print(f"n={n} p={p} r={r} d={d}: {obs.device_context().last_variant} term-scale {e:.2e}")
    assert e <= 1e-10


def test_k1x_deterministic_and_linear_in_nu():
    n, p, r, d = 512, 40_000, 64, 4
    V, _, lam, A = _case(n, p, r, d, seed=3)
    nu = np.random.default_rng(4).uniform(0.5, 2.0, p) / p
    Y1 = mcp.ttsv_batch(mcp.ObservationSet(V, nu), A, d)
    Y1b = mcp.ttsv_batch(mcp.ObservationSet(V, nu), A, d)
    Y2 = mcp.ttsv_batch(mcp.ObservationSet(V, 2.0 * nu), A, d)
    assert np.array_equal(Y1, Y1b)
    assert np.array_equal(2.0 * Y1, Y2)


def test_k1x_zero_lambda_exact():
    V, _, _, A = _case(512, 9_000, 64, 3, seed=5)
    res = mcp.fg_implicit(mcp.ObservationSet(V), np.zeros(64), A, 3, 0.0)
    assert res.f == 0.0 and np.array_equal(res.g_A, np.zeros_like(A))


@pytest.mark.parametrize("n,p,r,d,dt,rb", [
    (1024, 40_000, 256, 3, np.float32, 64),   # c5 shape: chunks 0-7 in TMEM, 8-15 in L2
    (900, 20_000, 33, 4, np.float32, 64),     # ragged n and r (15 chunks: 8 TMEM + 7 L2)
    (1024, 12_000, 64, 5, np.float64, 64),    # fp64 rows
    (2000, 6_000, 40, 3, np.float64, 16),     # 32 chunks: RB = 16 fills all 512 TMEM columns
    (1024, 1_500, 100, 4, np.float32, 64),    # 56 tiles x 2 blocks < 148 SMs: grid capped
    (960, 9_500, 136, 3, np.float32, 64),     # 3 blocks: 49 groups + 1 leftover CTA
])
def test_k1gt_tmem_partial_vs_oracle(n, p, r, d, dt, rb):
    """K1GT (K1G with the Y partial in TMEM): oracle parity, then bitwise determinism and exact
    nu-linearity (pkg/tests/test_implicit.py:53-57) -- the TMEM read-modify-write keeps K1G's
    per-element sum order."""
    rng = np.random.default_rng(n + r)
    V = (rng.standard_normal((n, p)) / np.sqrt(n)).astype(dt)
    nu = rng.uniform(0.5, 2.0, p) / p
    lam = rng.standard_normal(r)
    A = rng.standard_normal((n, r)) / np.sqrt(n)
    obs = mcp.ObservationSet(V, nu)
    res = mcp.fg_implicit(obs, lam, A, d, 0.1)
    var = obs.device_context().last_variant
    assert var.startswith("k1gt_fg_dmma") and f"RB={rb}" in var, var
    V64 = V.astype(np.float64)
    f, gl, gA = om.fg_implicit(V64, nu, lam, A, d, 0.1)
    fs, gls, gAs, _ = om.term_scales(V64, nu, lam, A, d, 0.1)
    e = max(om.term_rel_err(res.f, f, fs), om.term_rel_err(res.g_lam, gl, gls),
            om.term_rel_err(res.g_A, gA, gAs))
    print(f"n={n} p={p} r={r} d={d}: {var} term-scale {e:.2e}")
    assert e <= 1e-10
    Y1 = mcp.ttsv_batch(obs, A, d)
    assert np.array_equal(Y1, mcp.ttsv_batch(obs, A, d))
    assert np.array_equal(2.0 * Y1, mcp.ttsv_batch(mcp.ObservationSet(V, 2.0 * nu), A, d))
