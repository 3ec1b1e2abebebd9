"""The CPU oracle restatement pinned against the reference's golden vectors (no GPU)."""

import numpy as np
import pytest

import instances
from oracle import lbfgs_oracle as lo
from oracle import momentcp_oracle as om


def _nu(V, nu):
    return np.full(V.shape[1], 1.0 / V.shape[1]) if nu is None else nu


def _inputs_sha(V, nu, lam, A):
    return instances.sha(V, lam, A) if nu is None else instances.sha(V, nu, lam, A)


def test_kats(golden):
    k = golden["kat"]
    V = np.array([[1.0], [2.0]])
    Y = om.ttsv_batch(V, np.array([1.0]), np.array([[1.0], [1.0]]), 3)
    assert np.allclose(Y, [[9.0], [18.0]], rtol=1e-14)
    assert np.array_equal(Y, k["ttsv_9_18"])
    assert om.data_norm_sq(np.array([[2.0]]), np.array([1.0]), 3) == float(k["dnorm_64"]) == 64.0
    _, _, _, w = om.gram_tail(np.array([1.0]), np.array([[1.0], [1.0]]), 3,
                              np.array([[9.0], [18.0]]))
    assert np.array_equal(w, k["w_27"])
    v = np.array([0.6, 0.8])
    f, _, _ = om.fg_implicit(v[:, None], np.array([1.0]), np.array([1.0]), v[:, None], 3, 1.0)
    assert abs(f) <= 1e-14 and f == float(k["exact_fit_f"])
    assert om.kruskal_norm_sq(np.array([2.0]), np.array([[1.0], [1.0]]), 3) == float(k["kruskal_32"])


@pytest.mark.parametrize("kind,count,make", [("t", instances.TINY_COUNT, instances.tiny_instance),
                                             ("e", instances.EXT_COUNT, instances.ext_instance)])
def test_sweep_matches_reference(golden, kind, count, make):
    g = golden["sweep"]
    for k in range(count):
        V, nu, lam, A, d, alpha = make(k)
        key = f"{kind}{k}_"
        assert str(g[key + "sha"]) == _inputs_sha(V, nu, lam, A), f"input drift at {key}"
        Vf = np.asarray(V, dtype=float)
        nuv = _nu(Vf, nu)
        f, gl, gA = om.fg_implicit(Vf, nuv, lam, A, d, alpha)
        # same numpy calls in the same order as the reference -> bitwise identical here
        assert f == float(g[key + "f"]), key
        assert np.array_equal(gl, g[key + "g_lam"]), key
        assert np.array_equal(gA, g[key + "g_A"]), key
        assert np.array_equal(om.ttsv_batch(Vf, nuv, A, d), g[key + "Y"]), key
        assert om.data_norm_sq(Vf, nuv, d) == float(g[key + "dnorm"]), key
        if key + "f_explicit" in g:
            # the dense (explicit) route of the oracle agrees with the reference's explicit f
            X = om.dense_moment(Vf, nuv, d)
            Yd = np.column_stack([om.dense_ttsv(X, A[:, j]) for j in range(A.shape[1])])
            fe, _, _ = om.finish(Yd, lam, A, d, alpha)
            fs = float(g[key + "f_scale"])
            assert abs(fe - float(g[key + "f_explicit"])) <= 1e-12 * (fs + abs(fe)), key


def test_term_scales_match_reference(golden):
    g = golden["sweep"]
    for k in range(0, instances.TINY_COUNT, 7):
        V, nu, lam, A, d, alpha = instances.tiny_instance(k)
        f_s, gl_s, gA_s, _ = om.term_scales(V, _nu(V, nu), lam, A, d, alpha)
        key = f"t{k}_"
        assert f_s == float(g[key + "f_scale"])
        assert np.array_equal(gl_s, g[key + "gl_scale"])
        assert np.allclose(gA_s, g[key + "gA_scale"], rtol=1e-6)


def test_partial_split_is_additive():
    rng = np.random.default_rng(5)
    V = rng.standard_normal((7, 40))
    nu = rng.random(40) + 0.5
    lam = rng.standard_normal(3)
    A = rng.standard_normal((7, 3))
    f, gl, gA = om.fg_implicit(V, nu, lam, A, 4, 0.3)
    Y1, w1 = om.fg_partial(V[:, :13], nu[:13], A, 4)
    Y2, w2 = om.fg_partial(V[:, 13:], nu[13:], A, 4)
    f2, gl2, gA2 = om.finish_from_partial(Y1 + Y2, w1 + w2, lam, A, 4, 0.3)
    assert abs(f - f2) <= 1e-12 * max(1.0, abs(f))
    assert np.allclose(gl, gl2, rtol=1e-12, atol=1e-13)
    assert np.allclose(gA, gA2, rtol=1e-12, atol=1e-13)


def test_blocked_data_norm_matches_full(golden):
    cfg, V, _, _ = instances.config_instance("c4")
    nu = np.full(V.shape[1], 1.0 / V.shape[1])
    full = float(golden["configs"]["c4_dnorm"])
    blocked = om.data_norm_sq_blocked(V, nu, cfg.d, block=1000)
    assert abs(blocked - full) <= 1e-12 * float(golden["configs"]["c4_dnorm_scale"])


@pytest.mark.parametrize("name", list(instances.CONFIG_CASES))
def test_configs_match_reference(golden, name):
    g = golden["configs"]
    cfg, V, lam, A = instances.config_instance(name)
    key = name + "_"
    assert str(g[key + "sha"]) == (instances.sha(V) if lam is None else instances.sha(V, lam, A))
    if name in ("c3", "c5"):
        return  # large fp64 oracle GEMMs: covered by test_sweep + the GPU parity tests
    Vf = np.asarray(V, dtype=float)
    nu = np.full(Vf.shape[1], 1.0 / Vf.shape[1])
    if lam is not None:
        f, gl, gA = om.fg_implicit(Vf, nu, lam, A, cfg.d, 0.0)
        assert f == float(g[key + "f"])
        assert np.array_equal(gl, g[key + "g_lam"])
        assert np.array_equal(gA, g[key + "g_A"])


def test_lbfgs_replays_reference_trajectory(golden):
    """The restated L-BFGS + oracle fg reproduce the reference's 100-step c1 fit bitwise."""
    g = golden["lbfgs_c1"]
    cfg, V, lam, A = instances.config_instance("c1")
    nu = np.full(V.shape[1], 1.0 / V.shape[1])
    fg = om.packed_fg(V, nu, cfg.d, cfg.r)
    its = []
    rep = lo.lbfgs(fg, om.pack(lam, A), max_iters=100, iterate_hook=its.append)
    assert rep["n_steps"] == int(g["n_steps"]) and rep["n_fg"] == int(g["n_fg"])
    assert rep["reason"] == str(g["reason"])
    assert np.array_equal(np.stack(its), g["iterates"])
    assert rep["f"] == float(g["final_f"])


def test_validation_errors():
    V = np.ones((2, 3))
    nu = np.full(3, 1 / 3)
    with pytest.raises(ValueError):
        om.ttsv_batch(V, nu, np.ones((3, 2)), 3)
    with pytest.raises(ValueError):
        om.ttsv_batch(V, nu, np.ones((2, 2)), 1)
    with pytest.raises(ValueError):
        om.fg_implicit(V, nu, np.array([np.nan]), np.ones((2, 1)), 3)
    with pytest.raises(ValueError):
        om.fg_implicit(V, nu, np.ones(1), np.ones((2, 1)), 3, np.inf)


def test_adam_restatement_reproduces_reference_run(golden):
    """oracle/adam_oracle.py vs the reference adam_minimize (tests/golden/adam_c1.npz)."""
    from oracle import adam_oracle as ao

    g = golden["adam_c1"]
    cfg, V, lam, A = instances.config_instance("c1")
    out = ao.adam(V, cfg.d, cfg.r, om.pack(lam, A), np.random.default_rng(instances.ADAM_SEED),
                  **instances.ADAM_C1)
    assert np.array_equal(np.array(out["trace_f"]), g["trace_f"])
    assert out["reason"] == str(g["reason"]) and out["n_iter"] == int(g["n_fg"])
    lam_b, A_b = om.unpack(out["x"], cfg.n, cfg.r)
    assert np.array_equal(lam_b, g["final_lam"]) and np.array_equal(A_b, g["final_A"])
    assert out["grad_inf"] == float(g["grad_inf"])
