"""Host-side logic of the drop-in API (no GPU): validation, packing, no CPU fallback."""

import ast
import os

import numpy as np
import pytest

import paper_1911_03813_b200 as mcp
from conftest import ROOT, gpu_available
from paper_1911_03813_b200 import synth


def test_pack_layout_matches_reference():
    lam = np.array([1.0, 2.0])
    A = np.array([[3.0, 5.0], [4.0, 6.0]])
    x = mcp.pack(lam, A)
    assert np.array_equal(x, [1, 2, 3, 4, 5, 6])          # optimize.py:104-110 (column-major)
    l2, A2 = mcp.unpack(x, 2, 2)
    assert np.array_equal(l2, lam) and np.array_equal(A2, A)
    with pytest.raises(ValueError):
        mcp.unpack(x[:-1], 2, 2)


def test_observation_set_validation():
    with pytest.raises(ValueError):
        mcp.ObservationSet(np.ones(3))
    with pytest.raises(ValueError):
        mcp.ObservationSet(np.ones((0, 3)))
    V = np.ones((2, 3))
    V[0, 0] = np.nan
    with pytest.raises(ValueError):
        mcp.ObservationSet(V)
    with pytest.raises(ValueError):
        mcp.ObservationSet(np.ones((2, 3)), np.array([1.0, -1.0, 1.0]))
    with pytest.raises(ValueError):
        mcp.ObservationSet(np.ones((2, 3)), np.ones(2))
    obs = mcp.ObservationSet(np.ones((2, 3)))
    assert obs.n == 2 and obs.p == 3 and obs.has_uniform_weights()
    assert np.array_equal(obs.nu, np.full(3, 1.0 / 3))
    o32 = mcp.ObservationSet(np.ones((2, 3), dtype=np.float32))
    assert o32.V.dtype == np.float64   # the reference surface stays float64


def test_argument_errors_precede_device_work():
    obs = mcp.ObservationSet(np.ones((2, 3)))
    with pytest.raises(ValueError):
        mcp.fg_implicit(obs, np.ones(2), np.ones((3, 2)), 3)
    with pytest.raises(ValueError):
        mcp.fg_implicit(obs, np.array([np.inf]), np.ones((2, 1)), 3)
    with pytest.raises(ValueError):
        mcp.fg_implicit(obs, np.ones(1), np.ones((2, 1)), 3, alpha=np.nan)
    with pytest.raises(ValueError):
        mcp.ttsv_batch(obs, np.ones((2, 1)), 1)
    with pytest.raises(ValueError):
        mcp.data_norm_sq(obs, 1)


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback():
    obs = mcp.ObservationSet(np.ones((2, 3)))
    with pytest.raises(RuntimeError):
        mcp.fg_implicit(obs, np.ones(1), np.ones((2, 1)), 3)


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_1911_03813_b200")
    for fn in os.listdir(pkg):
        if not fn.endswith(".py"):
            continue
        tree = ast.parse(open(os.path.join(pkg, fn)).read())
        for node in ast.walk(tree):
            if isinstance(node, ast.Import):
                names = [a.name for a in node.names]
            elif isinstance(node, ast.ImportFrom):
                names = [node.module or ""]
            else:
                continue
            assert not any(n.split(".")[0] == "oracle" for n in names), fn


def test_synth_host_generation_is_deterministic():
    cfg = synth.CONFIGS["c1"]
    a = synth.host_observations(cfg, 3, p=500)
    b = synth.host_observations(cfg, 3, p=500)
    assert a.shape == (20, 500) and np.array_equal(a, b)
    lam, A = synth.initial_point(cfg, 3)
    assert np.allclose(np.linalg.norm(A, axis=0), 1.0) and np.all(lam == 1.0 / cfg.r)
    c3 = synth.host_observations(synth.CONFIGS["c3"], 1, p=100)
    assert c3.dtype == np.float32 and c3.shape == (512, 100)


def test_lbfgs_minimize_accepts_any_callback():
    """A plain fg(x) callback (no device problem) runs on the host solver, which follows the
    reference's decisions: on a quadratic it reaches the tolerance, and it reproduces the
    restated reference solver's iterates bitwise."""
    import paper_1911_03813_b200 as mcp
    from oracle import lbfgs_oracle as lo

    D = np.diag(np.arange(1.0, 6.0))
    b = np.array([1.0, -2.0, 0.5, 3.0, -1.0])

    def fg(x):
        return 0.5 * float(x @ D @ x) - float(b @ x), D @ x - b

    rep = mcp.lbfgs_minimize(fg, np.zeros(5), mcp.OptConfig(pgtol=1e-7))
    assert rep.reason == "tolerance"
    assert np.allclose(rep.lam, np.linalg.solve(D, b), atol=1e-6)
    with pytest.raises(ValueError):
        mcp.lbfgs_minimize(lambda x: (np.nan, x), np.zeros(3), mcp.OptConfig())
    # a nonconvex objective: the same trajectory as the restated reference solver
    rng = np.random.default_rng(4)
    Q = rng.standard_normal((6, 6))

    def fg2(x):
        z = Q @ x
        return float(np.sum(z ** 4) - np.sum(z ** 2)), Q.T @ (4 * z ** 3 - 2 * z)

    x0 = rng.standard_normal(6)
    rep2 = mcp.lbfgs_minimize(fg2, x0, mcp.OptConfig(max_iters=40))
    ref = lo.lbfgs(fg2, x0, memory=5, max_iters=40)
    assert rep2.n_fg == ref["n_fg"] and rep2.n_steps == ref["n_steps"]
    assert np.array_equal(rep2.lam, ref["x"]) and rep2.f == ref["f"]


def test_lbfgs_config_checks():
    import paper_1911_03813_b200 as mcp

    with pytest.raises(ValueError):
        mcp.OptConfig(pgtol=0)
    with pytest.raises(ValueError):
        mcp.OptConfig(memory=0)


def test_adam_config_checks():
    import paper_1911_03813_b200 as mcp

    with pytest.raises(ValueError):
        mcp.AdamConfig(epoch_len=0)
    with pytest.raises(ValueError):
        mcp.AdamConfig(batch=0)
    assert mcp.AdamConfig().estimate_samples == 1000
