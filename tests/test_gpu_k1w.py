"""K1W (fp32 observations, large n: resident TMA tile, cluster n-split) against the CPU oracle.

Covers both work splits (strided column blocks when the clusters divide evenly, block-major
ranges otherwise -- including grids larger than the tile count, where clusters own no tiles and
partial slots are zero-filled), the 2-CTA cluster (n > 512), ragged n and r, weights, every
order d, and bitwise determinism / nu-linearity (the reference invariants,
pkg/tests/test_implicit.py:53-57).  FP64 mode tolerance: 1e-10 term-scale
(pkg/tests/test_acceptance.py:65-74).
"""

import numpy as np
import pytest

import paper_1911_03813_b200 as mcp
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


@pytest.mark.parametrize("n,p,r,d", [
    (512, 300_000, 64, 6),    # c3 shape (K1X strided: 148 CTAs / 4 blocks)
    (512, 300_000, 96, 3),    # 3 blocks: block-major ranges
    (512, 5_000, 64, 4),      # p < grid tiles: clusters without tiles, zero-filled slots
    (512, 2_000, 16, 3),      # one column block, p < grid (K1X strided with idle CTAs)
    (400, 30_000, 20, 5),     # K1X ragged n and r, ranges split (148 % 2 == 0 -> strided)
    (512, 60_000, 48, 6),     # K1X: 3 column blocks over 148 CTAs -> block-major ranges
    (500, 40_000, 40, 2),     # ragged n and r (last block partly padding), d = 2
    (256, 50_000, 32, 5),     # CPW = 1
    (1024, 60_000, 256, 3),   # c5 shape: 2-CTA cluster, 8 blocks over 74 clusters
    (900, 20_000, 33, 4),     # cluster, ragged
])
def test_k1w_vs_oracle(n, p, r, d):
    V, nu, lam, A = _case(n, p, r, d, seed=n + p + r)
    obs = mcp.ObservationSet(V, nu)
    res = mcp.fg_implicit(obs, lam, A, d, 0.3)
    assert obs.device_context().last_variant.startswith(("k1w_fg_dmma", "k1x_fg_dmma")), \
        obs.device_context().last_variant
    V64 = V.astype(np.float64)
    nu64 = np.full(p, 1.0 / p) if nu is None else nu
    f, gl, gA = om.fg_implicit(V64, nu64, lam, A, d, 0.3)
    fs, gls, gAs, _ = om.term_scales(V64, nu64, lam, A, d, 0.3)
    e = max(om.term_rel_err(res.f, f, fs), om.term_rel_err(res.g_lam, gl, gls),
            om.term_rel_err(res.g_A, gA, gAs))
    print(f"n={n} p={p} r={r} d={d}: {obs.device_context().last_variant} term-scale {e:.2e}")
    assert e <= 1e-10


def test_k1w_deterministic_and_linear_in_nu():
    n, p, r, d = 512, 40_000, 64, 4
    V, _, lam, A = _case(n, p, r, d, seed=3)
    nu = np.random.default_rng(4).uniform(0.5, 2.0, p) / p
    Y1 = mcp.ttsv_batch(mcp.ObservationSet(V, nu), A, d)
    Y1b = mcp.ttsv_batch(mcp.ObservationSet(V, nu), A, d)
    Y2 = mcp.ttsv_batch(mcp.ObservationSet(V, 2.0 * nu), A, d)
    assert np.array_equal(Y1, Y1b)
    assert np.array_equal(2.0 * Y1, Y2)


def test_k1w_zero_lambda_exact():
    V, _, _, A = _case(1024, 9_000, 64, 3, seed=5)
    res = mcp.fg_implicit(mcp.ObservationSet(V), np.zeros(64), A, 3, 0.0)
    assert res.f == 0.0 and np.array_equal(res.g_A, np.zeros_like(A))
