"""Single-process multi-GPU evaluation (MultiDeviceObservationSet) on a B200.

Only one GPU is reachable from this build, so the shards share device 0 (separate contexts,
separate streams -- the same code path as one shard per GPU, minus the NVLink copies).  Checks:
f+grad equal to the single-set evaluation (the shard sum is a fixed-order reassociation) and to
the CPU oracle; ||X||^2 from shard triangles + cross rectangles; a host-driven L-BFGS fit whose
every iterate the oracle re-evaluates (SURVEY.md 8c replay protocol).
"""

import numpy as np
import pytest

import paper_1911_03813_b200 as mcp
from oracle import lbfgs_oracle as lo
from oracle import momentcp_oracle as om

pytestmark = pytest.mark.gpu


def _data(n=40, p=9001, r=6, seed=3):
    rng = np.random.default_rng(seed)
    mu = rng.standard_normal((n, r))
    mu /= np.linalg.norm(mu, axis=0)
    V = mu[:, rng.integers(0, r, p)] + 0.1 * rng.standard_normal((n, p))
    A = rng.standard_normal((n, r))
    A /= np.linalg.norm(A, axis=0)
    return V, np.full(r, 1.0 / r), A


@pytest.mark.parametrize("weights", [False, True])
def test_multidevice_fg_matches_single_and_oracle(weights):
    V, lam, A = _data()
    p = V.shape[1]
    nu = np.random.default_rng(1).uniform(0.5, 1.5, p) / p if weights else None
    md = mcp.MultiDeviceObservationSet.from_host(V, [0, 0, 0], nu)
    res = md.fg(lam, A, 3, 0.2)
    one = mcp.fg_implicit(mcp.ObservationSet(V, nu), lam, A, 3, 0.2)
    assert abs(res.f - one.f) <= 1e-13 * abs(one.f)
    assert np.allclose(res.g_A, one.g_A, rtol=1e-12, atol=1e-15)
    nu64 = np.full(p, 1.0 / p) if nu is None else nu
    f, gl, gA = om.fg_implicit(V, nu64, lam, A, 3, 0.2)
    fs, gls, gAs, _ = om.term_scales(V, nu64, lam, A, 3, 0.2)
    assert max(om.term_rel_err(res.f, f, fs), om.term_rel_err(res.g_lam, gl, gls),
               om.term_rel_err(res.g_A, gA, gAs)) <= 1e-10
    # repeatable bitwise (fixed shard order)
    res2 = md.fg(lam, A, 3, 0.2)
    assert res2.f == res.f and np.array_equal(res2.g_A, res.g_A)


def test_multidevice_data_norm():
    rng = np.random.default_rng(5)
    V = rng.standard_normal((48, 7000)) / 7
    md = mcp.MultiDeviceObservationSet.from_host(V, [0, 0, 0, 0])
    got = md.data_norm_sq(4)
    want = mcp.data_norm_sq(mcp.ObservationSet(V), 4)
    assert got == pytest.approx(want, rel=1e-12)


def test_multidevice_lbfgs_replay():
    """lbfgs_minimize on the multi-device fg (host solver): every accepted iterate agrees with the
    CPU oracle to 1e-10 term-scale, and the restated reference solver driven by the oracle takes
    the same opening steps."""
    V, lam, A = _data(n=20, p=6000, r=5, seed=9)
    n, r, d = 20, 5, 3
    p = V.shape[1]
    nu = np.full(p, 1.0 / p)
    md = mcp.MultiDeviceObservationSet.from_host(V, [0, 0])
    fg = md.packed_fg(d, r)
    iterates = []
    rep = mcp.lbfgs_minimize(fg, mcp.pack(lam, A), mcp.OptConfig(max_iters=25),
                             shape=(n, r), iterate_hook=iterates.append)
    assert rep.n_steps >= 5
    for x in iterates:
        lam_i, A_i = om.unpack(x, n, r)
        f, gl, gA = om.fg_implicit(V, nu, lam_i, A_i, d, 0.0)
        fs, gls, gAs, _ = om.term_scales(V, nu, lam_i, A_i, d, 0.0)
        g = fg(x)
        assert om.term_rel_err(g[0], f, fs) <= 1e-10
        assert om.term_rel_err(g[1], om.pack(gl, gA), om.pack(gls, gAs)) <= 1e-10
    ref = lo.lbfgs(om.packed_fg(V, nu, d, r), mcp.pack(lam, A), max_iters=5)
    assert np.allclose(ref["x"], iterates[5], rtol=1e-8, atol=1e-10)
