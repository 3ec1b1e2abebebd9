"""Stochastic path on the device against the restated reference.

* sample_observations draws the reference's indices and gathers exactly those rows on the GPU.
* adam_minimize (mcp_adam, device-resident) reproduces, BITWISE, the restated reference Adam
  (oracle/adam_oracle.py, itself pinned bitwise to the reference run in adam_c1.npz) when that
  restatement takes its mini-batch gradients from the same GPU f+grad: same draws, same Adam
  arithmetic order, same kernels on the same rows.
* against the all-CPU restatement the epoch estimates agree to 1e-9 (fp64 reassociation only).
"""

import numpy as np
import pytest

import instances
import paper_1911_03813_b200 as mcp
from oracle import adam_oracle as ao
from oracle import momentcp_oracle as om

pytestmark = pytest.mark.gpu


def _gpu_fg(Vs, lam, A, d):
    res = mcp.fg_implicit(mcp.ObservationSet(Vs), lam, A, d)
    return res.f, res.g_lam, res.g_A


def test_sample_observations_gathers_reference_rows():
    rng = np.random.default_rng(3)
    V = rng.standard_normal((7, 500))
    obs = mcp.ObservationSet(V)
    s = mcp.sample_observations(obs, 64, np.random.default_rng(11))
    idx = np.random.default_rng(11).integers(0, 500, size=64)
    assert s.p == 64 and np.array_equal(s.V, V[:, idx])
    assert np.allclose(s.weights(), 1 / 64, rtol=0, atol=0)
    lam, A = rng.standard_normal(3), rng.standard_normal((7, 3))
    a = mcp.fg_implicit(s, lam, A, 3)
    b = mcp.fg_implicit(mcp.ObservationSet(V[:, idx]), lam, A, 3)
    assert a.f == b.f and np.array_equal(a.g_A, b.g_A)
    with pytest.raises(ValueError):
        mcp.sample_observations(obs, 0, rng)
    with pytest.raises(ValueError):
        mcp.sample_observations(mcp.ObservationSet(V, rng.random(500) + 0.5), 4, rng)


def test_device_adam_bitwise_vs_restated_reference_with_gpu_gradients(golden):
    cfg, V, lam, A = instances.config_instance("c1")
    x0 = om.pack(lam, A)
    obs = mcp.ObservationSet(V)
    rng_dev = np.random.default_rng(instances.ADAM_SEED)
    rng_host = np.random.default_rng(instances.ADAM_SEED)
    dev = mcp.adam_minimize(obs, cfg.d, cfg.r, x0, mcp.AdamConfig(**instances.ADAM_C1), rng_dev)
    host = ao.adam(V, cfg.d, cfg.r, x0, rng_host, fg_fn=_gpu_fg, **instances.ADAM_C1)
    # the epoch drawn ahead of a stopping decision is rewound: same generator state as the reference
    assert rng_dev.bit_generator.state == rng_host.bit_generator.state
    assert dev.reason == host["reason"] == str(golden["adam_c1"]["reason"])
    assert dev.n_fg == host["n_iter"] == int(golden["adam_c1"]["n_fg"])
    assert np.array_equal(np.array([t[0] for t in dev.trace]), np.array(host["trace_f"]))
    assert np.array_equal(mcp.pack(dev.lam, dev.A), host["x"])
    assert dev.f == host["f"] and dev.grad_inf_norm == host["grad_inf"]


def test_device_adam_vs_cpu_reference_run(golden):
    g = golden["adam_c1"]
    cfg, V, lam, A = instances.config_instance("c1")
    dev = mcp.adam_minimize(mcp.ObservationSet(V), cfg.d, cfg.r, om.pack(lam, A),
                            mcp.AdamConfig(**instances.ADAM_C1),
                            np.random.default_rng(instances.ADAM_SEED))
    tf = np.array([t[0] for t in dev.trace])
    assert tf.shape == g["trace_f"].shape
    assert np.allclose(tf, g["trace_f"], rtol=1e-9, atol=1e-12)
    assert np.allclose(dev.A, g["final_A"], rtol=1e-7, atol=1e-9)


def test_device_adam_fp32_set_fast_mode_and_errors():
    cfg, V, lam, A = instances.config_instance("c1")
    x0 = om.pack(lam, A)
    obs32 = mcp.ObservationSet(V.astype(np.float32))
    small = dict(epoch_len=10, batch=32, estimate_samples=100, max_epochs=3)
    for mode in (None, "tf32x3"):
        rep = mcp.adam_minimize(obs32, cfg.d, cfg.r, x0, mcp.AdamConfig(**small),
                                np.random.default_rng(5), mode=mode)
        assert rep.n_fg == 30 and len(rep.trace) == 4 and np.isfinite(rep.f)
    with pytest.raises(ValueError):
        mcp.adam_minimize(mcp.ObservationSet(V, np.random.default_rng(0).random(V.shape[1]) + 1),
                          cfg.d, cfg.r, x0, mcp.AdamConfig(**small), np.random.default_rng(5))
    with pytest.raises(ValueError):
        mcp.adam_minimize(obs32, cfg.d, cfg.r, x0[:-1], mcp.AdamConfig(**small),
                          np.random.default_rng(5))


def test_device_adam_bitwise_on_the_single_launch_path():
    """n > 128: the mini-batch and estimate evaluations run as the single-launch K1Z, the
    mini-batch rows read in place through the epoch's index list (no gathered copy).  The run
    must still equal, bitwise, the restated reference Adam fed with GPU evaluations of UPLOADED
    copies of the same rows (K1Z's summation order depends on the shape only)."""
    rng = np.random.default_rng(41)
    n, p, r, d = 200, 3000, 4, 3
    V = rng.standard_normal((n, p)) / np.sqrt(n)
    lam, A = np.full(r, 1.0 / r), rng.standard_normal((n, r)) / np.sqrt(n)
    x0 = om.pack(lam, A)
    cfg = dict(epoch_len=12, batch=40, estimate_samples=150, max_epochs=4)
    obs = mcp.ObservationSet(V)
    rng_dev, rng_host = np.random.default_rng(9), np.random.default_rng(9)
    dev = mcp.adam_minimize(obs, d, r, x0, mcp.AdamConfig(**cfg), rng_dev)
    sub = mcp.ObservationSet(V[:, :40])
    mcp.fg_implicit(sub, lam, A, d)
    assert sub.device_context().last_variant.startswith("k1z_fg_small")
    host = ao.adam(V, d, r, x0, rng_host, fg_fn=_gpu_fg, **cfg)
    assert rng_dev.bit_generator.state == rng_host.bit_generator.state
    assert dev.n_fg == host["n_iter"] and dev.reason == host["reason"]
    assert np.array_equal(np.array([t[0] for t in dev.trace]), np.array(host["trace_f"]))
    assert np.array_equal(mcp.pack(dev.lam, dev.A), host["x"])
    assert dev.f == host["f"] and dev.grad_inf_norm == host["grad_inf"]
