"""Parity of the CUDA path (through the C ABI) with the reference, on a B200.

Tolerances (BASELINE.json north_star):
  FP64 mode  f, g_lam, g_A: <= 1e-10 in the reference's term-scale metric
             (pkg/tests/test_acceptance.py:5-11,65-74); kernels (Y, ||X||^2): <= 1e-12.
  Bitwise    lambda = 0 gives f = alpha and g_A = 0 exactly (test_objective.py:101-106);
             gradients independent of alpha (:114-121); Y exactly linear in nu
             (test_implicit.py:53-57); repeated evaluations bit-identical (fixed-order reductions).
"""

import numpy as np
import pytest

import instances
import paper_1911_03813_b200 as mcp
from oracle import lbfgs_oracle as lo
from oracle import momentcp_oracle as om

pytestmark = pytest.mark.gpu

FG_TOL = 1e-10
KERNEL_TOL = 1e-12


def _nu(V, nu):
    return np.full(V.shape[1], 1.0 / V.shape[1]) if nu is None else nu


def _err(got, want, scale):
    return om.term_rel_err(got, want, scale)


def test_kats():
    obs = mcp.ObservationSet(np.array([[1.0], [2.0]]), np.array([1.0]))
    Y = mcp.ttsv_batch(obs, np.array([[1.0], [1.0]]), 3)
    assert np.allclose(Y, [[9.0], [18.0]], rtol=1e-14)
    assert mcp.data_norm_sq(mcp.ObservationSet(np.array([[2.0]]), np.array([1.0])), 3) == 64.0
    v = np.array([0.6, 0.8])
    res = mcp.fg_implicit(mcp.ObservationSet(v[:, None], np.array([1.0])), np.array([1.0]),
                          v[:, None], 3, alpha=1.0)
    assert abs(res.f) <= 1e-14
    z = mcp.ttsv_batch(mcp.ObservationSet(np.random.default_rng(0).standard_normal((3, 4))),
                       np.zeros((3, 2)), 3)
    assert np.array_equal(z, np.zeros((3, 2)))


@pytest.mark.parametrize("kind,count,make", [("t", instances.TINY_COUNT, instances.tiny_instance),
                                             ("e", instances.EXT_COUNT, instances.ext_instance)])
def test_sweep_vs_reference_golden(golden, kind, count, make):
    g = golden["sweep"]
    worst_fg = worst_k = 0.0
    for k in range(count):
        V, nu, lam, A, d, alpha = make(k)
        key = f"{kind}{k}_"
        obs = mcp.ObservationSet(V, nu)
        res = mcp.fg_implicit(obs, lam, A, d, alpha)
        e = max(_err(res.f, g[key + "f"], g[key + "f_scale"]),
                _err(res.g_lam, g[key + "g_lam"], g[key + "gl_scale"]),
                _err(res.g_A, g[key + "g_A"], g[key + "gA_scale"]))
        assert e <= FG_TOL, (key, e)
        worst_fg = max(worst_fg, e)
        Y = mcp.ttsv_batch(obs, A, d)
        ek = _err(Y, g[key + "Y"], g[key + "Y_scale"])
        dn = mcp.data_norm_sq(obs, d)
        ek = max(ek, _err(dn, g[key + "dnorm"], g[key + "dnorm_scale"]))
        assert ek <= KERNEL_TOL, (key, ek)
        worst_k = max(worst_k, ek)
    print(f"{kind}: worst fg {worst_fg:.2e}, kernels {worst_k:.2e}")


def test_zero_weights_exact():
    rng = np.random.default_rng(24)
    for n, p, r, d in [(3, 5, 2, 3), (100, 700, 10, 4), (17, 64, 9, 2)]:
        obs = mcp.ObservationSet(rng.standard_normal((n, p)))
        A = rng.standard_normal((n, r))
        res = mcp.fg_implicit(obs, np.zeros(r), A, d, 0.0)
        assert res.f == 0.0
        assert np.array_equal(res.g_A, np.zeros_like(A))


def test_alpha_shift_bitwise():
    rng = np.random.default_rng(25)
    obs = mcp.ObservationSet(rng.standard_normal((30, 500)))
    lam, A = rng.standard_normal(6), rng.standard_normal((30, 6))
    r0 = mcp.fg_implicit(obs, lam, A, 3, 0.0)
    r1 = mcp.fg_implicit(obs, lam, A, 3, 7.25)
    assert r1.f - r0.f == pytest.approx(7.25, rel=1e-12, abs=1e-12 * max(1.0, abs(r0.f)))
    assert np.array_equal(r0.g_lam, r1.g_lam) and np.array_equal(r0.g_A, r1.g_A)


def test_linear_in_weights_bitwise_and_deterministic():
    rng = np.random.default_rng(11)
    V = rng.standard_normal((70, 1000))
    nu = rng.random(1000) + 0.5
    A = rng.standard_normal((70, 12))
    o1 = mcp.ObservationSet(V, nu)
    o2 = mcp.ObservationSet(V, 2.0 * nu)
    Y1 = mcp.ttsv_batch(o1, A, 4)
    assert np.array_equal(mcp.ttsv_batch(o2, A, 4), 2.0 * Y1)
    assert np.array_equal(mcp.ttsv_batch(o1, A, 4), Y1)
    lam = rng.standard_normal(12)
    a, b = mcp.fg_implicit(o1, lam, A, 4), mcp.fg_implicit(o1, lam, A, 4)
    assert a.f == b.f and np.array_equal(a.g_A, b.g_A) and np.array_equal(a.g_lam, b.g_lam)


def test_permutation_invariance():
    rng = np.random.default_rng(12)
    V = rng.standard_normal((40, 3000))
    nu = rng.random(3000) + 0.5
    A = rng.standard_normal((40, 7))
    perm = rng.permutation(3000)
    Y0 = mcp.ttsv_batch(mcp.ObservationSet(V, nu), A, 3)
    Y1 = mcp.ttsv_batch(mcp.ObservationSet(V[:, perm], nu[perm]), A, 3)
    _, _, _, Ya = om.term_scales(V, nu, np.ones(7), A, 3, 0.0)
    assert _err(Y1, Y0, Ya) <= 1e-14
    d0 = mcp.data_norm_sq(mcp.ObservationSet(V, nu), 4)
    d1 = mcp.data_norm_sq(mcp.ObservationSet(V[:, perm], nu[perm]), 4)
    assert d1 == pytest.approx(d0, rel=1e-13)


@pytest.mark.parametrize("name", list(instances.CONFIG_CASES))
def test_configs_vs_reference_golden(golden, name):
    g = golden["configs"]
    cfg, V, lam, A = instances.config_instance(name)
    key = name + "_"
    obs = mcp.ObservationSet(V)
    if lam is not None:
        res = mcp.fg_implicit(obs, lam, A, cfg.d, 0.0)
        e = max(_err(res.f, g[key + "f"], g[key + "f_scale"]),
                _err(res.g_lam, g[key + "g_lam"], g[key + "gl_scale"]),
                _err(res.g_A, g[key + "g_A"], g[key + "gA_scale"]))
        print(f"{name}: fg term-scale err {e:.2e} via {obs.device_context().last_variant}")
        assert e <= FG_TOL
    dn = mcp.data_norm_sq(obs, cfg.d)
    e = _err(dn, g[key + "dnorm"], g[key + "dnorm_scale"])
    print(f"{name}: ||X||^2 term-scale err {e:.2e}")
    assert e <= KERNEL_TOL


def test_finite_differences():
    rng = np.random.default_rng(27)
    h = 1e-6
    for _ in range(8):
        n, p, r, d = int(rng.integers(2, 7)), int(rng.integers(2, 9)), int(rng.integers(1, 4)), \
            int(rng.choice([2, 3, 4]))
        obs = mcp.ObservationSet(rng.standard_normal((n, p)))
        lam = rng.uniform(0.5, 1.5, r) * rng.choice([-1.0, 1.0], r)
        A = rng.standard_normal((n, r))
        A /= np.linalg.norm(A, axis=0)
        fg = mcp.packed_fg_implicit(obs, d, r)
        x = mcp.pack(lam, A)
        _, g = fg(x)
        fd = np.empty_like(x)
        for i in range(x.size):
            e = np.zeros_like(x)
            e[i] = h
            fd[i] = (fg(x + e)[0] - fg(x - e)[0]) / (2.0 * h)
        scale = np.maximum(np.abs(g), np.abs(g).max())
        assert np.all(np.abs(fd - g) <= 1e-5 * np.maximum(scale, 1e-12))


def test_packed_matches_unpacked():
    rng = np.random.default_rng(3)
    obs = mcp.ObservationSet(rng.standard_normal((20, 900)))
    lam, A = rng.standard_normal(5), rng.standard_normal((20, 5))
    f, g = mcp.packed_fg_implicit(obs, 3, 5, alpha=0.25)(mcp.pack(lam, A))
    res = mcp.fg_implicit(obs, lam, A, 3, 0.25)
    assert f == res.f and np.array_equal(g, mcp.pack(res.g_lam, res.g_A))


def test_replay_lbfgs_c1(golden):
    """Replay protocol: drive the restated reference L-BFGS with the GPU fg;
    at every GPU iterate the CPU oracle must agree to 1e-10; the trajectory matches the
    reference's own for the opening steps (chaotic later)."""
    g = golden["lbfgs_c1"]
    cfg, V, lam, A = instances.config_instance("c1")
    nu = np.full(V.shape[1], 1.0 / V.shape[1])
    fg_gpu = mcp.packed_fg_implicit(mcp.ObservationSet(V), cfg.d, cfg.r)
    fg_cpu = om.packed_fg(V, nu, cfg.d, cfg.r)
    its = []
    rep = lo.lbfgs(fg_gpu, om.pack(lam, A), max_iters=100, iterate_hook=its.append)
    assert rep["n_steps"] == 100
    worst = 0.0
    for x in its:
        fc, gc = fg_cpu(x)
        fgp, gg = fg_gpu(x)
        worst = max(worst, abs(fgp - fc) / max(1.0, abs(fc)),
                    float(np.max(np.abs(gg - gc)) / max(1.0, np.max(np.abs(gc)))))
    assert worst <= 1e-10, worst
    ref_its = g["iterates"]
    for k in range(10):
        assert np.allclose(its[k], ref_its[k], rtol=1e-10, atol=1e-12), k
    print(f"replay: worst per-iterate rel {worst:.2e}; final f gpu {rep['f']:.10e} "
          f"ref {float(g['final_f']):.10e}")


def test_c2_full_size_vs_oracle():
    """BASELINE configs[1] at full size (p = 1e6): one evaluation against the CPU oracle."""
    from paper_1911_03813_b200 import synth

    cfg = synth.CONFIGS["c2"]
    V = synth.host_observations(cfg, 2, p=cfg.p)
    lam, A = synth.initial_point(cfg, 2)
    obs = mcp.ObservationSet(V)
    res = mcp.fg_implicit(obs, lam, A, cfg.d, 0.0)
    nu = np.full(cfg.p, 1.0 / cfg.p)
    f, gl, gA = om.fg_implicit(V, nu, lam, A, cfg.d, 0.0)
    f_s, gl_s, gA_s, _ = om.term_scales(V, nu, lam, A, cfg.d, 0.0)
    e = max(_err(res.f, f, f_s), _err(res.g_lam, gl, gl_s), _err(res.g_A, gA, gA_s))
    print(f"c2 full: term-scale err {e:.2e}, plain rel f {abs(res.f - f) / abs(f):.2e}")
    assert e <= FG_TOL


def test_row_shards_sum_to_full():
    """The additive [Y | w] split the multi-GPU path all-reduces, on one GPU (no waiting
    kernels: each shard's partial runs to completion, the sum is done by torch)."""
    import torch

    from paper_1911_03813_b200 import distributed as dist_mod

    rng = np.random.default_rng(8)
    n, p, r, d = 64, 5000, 16, 3
    V = rng.standard_normal((n, p))
    lam, A = rng.standard_normal(r), rng.standard_normal((n, r))
    full = mcp.fg_implicit(mcp.ObservationSet(V), lam, A, d, 0.1)
    Vt = torch.as_tensor(V.T.copy(), device="cuda")
    parts = []
    for rank in range(3):
        lo_, hi_ = dist_mod.shard_bounds(p, 3, rank)
        sobs = mcp.ObservationSet.from_device(Vt[lo_:hi_], p_total=p)
        parts.append(dist_mod.device_partial(sobs, lam, A, d))
    Yw = sum(parts)
    f, gl, gA = dist_mod.device_finish(mcp.ObservationSet.from_device(Vt, p_total=p),
                                       lam, A, d, 0.1, Yw)
    nu = np.full(p, 1.0 / p)
    f_s, gl_s, gA_s, _ = om.term_scales(V, nu, lam, A, d, 0.1)
    assert _err(f, full.f, f_s) <= 1e-13
    assert _err(gl, full.g_lam, gl_s) <= 1e-13
    assert _err(gA, full.g_A, gA_s) <= 1e-13


def test_data_norm_parts_sum_to_full():
    rng = np.random.default_rng(9)
    V = rng.standard_normal((48, 1500)) / 7
    obs = mcp.ObservationSet(V)
    full = mcp.data_norm_sq(obs, 4)
    ctx = obs.device_context()
    parts = [ctx.data_norm_sq(4, None, k, 4) for k in range(4)]
    assert sum(parts) == pytest.approx(full, rel=1e-13)


def test_device_errors_are_value_errors():
    obs = mcp.ObservationSet(np.ones((2, 3)))
    ctx = obs.device_context()
    with pytest.raises(ValueError):
        ctx.fg_packed(np.ones(3), 2, 1, 1, 0.0, None)   # d < 2 checked in the library too
    with pytest.raises(ValueError):
        mcp.fg_implicit(obs, np.ones(1), np.ones((2, 1)), 3, mode="bogus")


# ----------------------------- fast mode (tcgen05 3xTF32) -----------------------------
FAST_TOL = 1e-4   # the stated bound of the fast mode (BASELINE north_star)


def _fast_errs(res, f, gl, gA, scales):
    f_s, gl_s, gA_s = scales
    term = max(_err(res.f, f, f_s), _err(res.g_lam, gl, gl_s), _err(res.g_A, gA, gA_s))
    norm = max(abs(res.f - f) / max(abs(f), 1e-300),
               float(np.linalg.norm(res.g_lam - gl) / max(np.linalg.norm(gl), 1e-300)),
               float(np.linalg.norm(res.g_A - gA) / max(np.linalg.norm(gA), 1e-300)))
    return term, norm


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c5"])
def test_fast_mode_configs(golden, name):
    g = golden["configs"]
    cfg, V, lam, A = instances.config_instance(name)
    key = name + "_"
    obs = mcp.ObservationSet(V)
    res = mcp.fg_implicit(obs, lam, A, cfg.d, 0.0, mode="tf32x3")
    term, norm = _fast_errs(res, float(g[key + "f"]), g[key + "g_lam"], g[key + "g_A"],
                            (g[key + "f_scale"], g[key + "gl_scale"], g[key + "gA_scale"]))
    print(f"{name} tf32x3 via {obs.device_context().last_variant}: term-scale {term:.2e}, "
          f"normwise {norm:.2e}")
    assert term <= FAST_TOL and norm <= FAST_TOL


def test_fast_mode_ext_sweep(golden):
    g = golden["sweep"]
    worst = 0.0
    for k in range(instances.EXT_COUNT):
        V, nu, lam, A, d, alpha = instances.ext_instance(k)
        key = f"e{k}_"
        res = mcp.fg_implicit(mcp.ObservationSet(V, nu), lam, A, d, alpha, mode="tf32x3")
        e = max(_err(res.f, g[key + "f"], g[key + "f_scale"]),
                _err(res.g_lam, g[key + "g_lam"], g[key + "gl_scale"]),
                _err(res.g_A, g[key + "g_A"], g[key + "gA_scale"]))
        assert e <= FAST_TOL, (key, e)
        worst = max(worst, e)
    print(f"fast-mode ext sweep: worst term-scale {worst:.2e}")


def test_fast_mode_zero_weights_and_determinism():
    rng = np.random.default_rng(31)
    obs = mcp.ObservationSet(rng.standard_normal((200, 5000)).astype(np.float32))
    A = rng.standard_normal((200, 24))
    res = mcp.fg_implicit(obs, np.zeros(24), A, 3, 0.0, mode="tf32x3")
    assert res.f == 0.0 and np.array_equal(res.g_A, np.zeros_like(A))
    lam = rng.standard_normal(24)
    a = mcp.fg_implicit(obs, lam, A, 3, mode="tf32x3")
    b = mcp.fg_implicit(obs, lam, A, 3, mode="tf32x3")
    assert a.f == b.f and np.array_equal(a.g_A, b.g_A)


# ----------------------------- batched multistart -----------------------------
@pytest.mark.parametrize("n,p,r,d,k", [(20, 3000, 5, 3, 4), (100, 20000, 10, 4, 8), (7, 50, 3, 2, 3)])
def test_batched_matches_single_starts(n, p, r, d, k):
    rng = np.random.default_rng(n + k)
    V = rng.standard_normal((n, p))
    obs = mcp.ObservationSet(V)
    X = np.stack([mcp.pack(rng.standard_normal(r), rng.standard_normal((n, r)))
                  for _ in range(k)])
    F, G = mcp.packed_fg_implicit_batched(obs, d, r, alpha=0.5)(X)
    fg1 = mcp.packed_fg_implicit(obs, d, r, alpha=0.5)
    nu = np.full(p, 1.0 / p)
    for s in range(k):
        f1, g1 = fg1(X[s])
        lam, A = mcp.unpack(X[s], n, r)
        f_s, gl_s, gA_s, _ = om.term_scales(V, nu, lam, A, d, 0.5)
        scale = np.concatenate([gl_s, gA_s.ravel(order="F")])
        assert _err(F[s], f1, f_s) <= 1e-13 and _err(G[s], g1, scale) <= 1e-13
        fo, go = om.packed_fg(V, nu, d, r, 0.5)(X[s])
        assert _err(F[s], fo, f_s) <= FG_TOL and _err(G[s], go, scale) <= FG_TOL


def test_partial_then_finish_equals_single_evaluation_bitwise():
    """The sharded building blocks on one rank: partial (K1 + reduce) then finish (K4) must
    reproduce the single-call evaluation bitwise, with and without the fused reduce + finish
    (K3F forms G, C, M, u in-kernel in the same expression order as K4), over orders d and
    ranks up to K3F's limit r = 32.  The single-launch small-problem kernel (K1Z) is switched
    off for the bitwise part: it sums in its own fixed order and is compared to 1e-13."""

    import torch

    from paper_1911_03813_b200 import _native

    rng = np.random.default_rng(21)
    for n, r, d in ((20, 5, 3), (100, 10, 4), (64, 16, 6), (30, 20, 3), (128, 32, 2),
                    (100, 32, 5)):
        V = rng.standard_normal((n, 3000))
        lam, A = rng.standard_normal(r), rng.standard_normal((n, r))
        obs = mcp.ObservationSet(V)
        ctx = obs.device_context()
        x = torch.as_tensor(mcp.pack(lam, A), device="cuda")
        s = _native.stream_handle(torch.cuda.current_stream())
        outs = []
        o_small = torch.empty(1 + r + n * r, dtype=torch.float64, device="cuda")
        ctx.fg_device(d, r, x.data_ptr(), 0.25, None, o_small.data_ptr(), s)
        small = ctx.last_variant.startswith("k1z")
        res = mcp.fg_implicit(obs, lam, A, d, 0.25)
        assert float(o_small[0]) == res.f
        ctx.set_option(_native.MCP_OPT_SMALL_KERNEL, 0)
        for fused in (True, False):
            ctx.set_option(_native.MCP_OPT_FUSED_TAIL, 1 if fused else 0)
            try:
                Yw = torch.empty(n * r + r, dtype=torch.float64, device="cuda")
                o1 = torch.empty(1 + r + n * r, dtype=torch.float64, device="cuda")
                o2 = torch.empty_like(o1)
                ctx.fg_partial_device(d, r, x.data_ptr(), None, Yw.data_ptr(), s)
                ctx.fg_finish_device(d, r, x.data_ptr(), Yw.data_ptr(), 0.25, o1.data_ptr(), s)
                ctx.fg_device(d, r, x.data_ptr(), 0.25, None, o2.data_ptr(), s)
                torch.cuda.synchronize()
                assert torch.equal(o1, o2), (n, r, d, fused)
                outs.append(o1.cpu())
            finally:
                ctx.set_option(_native.MCP_OPT_FUSED_TAIL, 1)
        ctx.set_option(_native.MCP_OPT_SMALL_KERNEL, 1)
        assert torch.equal(outs[0], outs[1]), (n, r, d)
        res = mcp.fg_implicit(obs, lam, A, d, 0.25)
        if small:
            f_s, gl_s, gA_s, _ = om.term_scales(V, _nu(V, None), lam, A, d, 0.25)
            got, want = o_small.cpu().numpy(), outs[0].numpy()
            assert _err(got[0], want[0], f_s) <= 1e-13
            assert _err(got[1:1 + r], want[1:1 + r], gl_s) <= 1e-13
            assert _err(got[1 + r:], want[1 + r:], gA_s.reshape(-1, order="F")) <= 1e-13
        else:
            assert float(outs[0][0]) == res.f


def test_peer_exchange_kernels_two_virtual_ranks():
    """csrc/peer.cu on ONE GPU with two virtual ranks run strictly in sequence (both partials and
    signals complete before either reduce starts -- no kernel waits on another): the peer
    reduce + fused finish equals the single-device evaluation of the union of the rows to the
    fp64 reassociation of the 2-way row split, bitwise identical on both ranks, and matches
    the all-reduce + finish path bitwise (same rank-order sum)."""
    import torch

    from paper_1911_03813_b200 import _native
    from paper_1911_03813_b200 import distributed as D

    rng = np.random.default_rng(33)
    n, p, r, d = 100, 6000, 10, 4
    V = rng.standard_normal((n, p)) / 10
    lam, A = rng.standard_normal(r), rng.standard_normal((n, r)) / 10
    Vt = torch.as_tensor(V.T.copy(), device="cuda")
    L = n * r + r
    bufs = [torch.zeros(2 * L, dtype=torch.float64, device="cuda") for _ in range(2)]
    flags = [torch.zeros(2, dtype=torch.int64, device="cuda") for _ in range(2)]
    buf_ptrs = [b.data_ptr() for b in bufs]
    flag_ptrs = [f.data_ptr() for f in flags]
    ranks = []
    for k in range(2):
        lo, hi = D.shard_bounds(p, 2, k)
        sobs = mcp.ObservationSet.from_device(Vt[lo:hi], p_total=p)
        ranks.append(D.PeerExchange(sobs.device_context(), n, r, k, 2,
                                    buffers=(bufs[k], flags[k], buf_ptrs, flag_ptrs)))
    x = torch.as_tensor(mcp.pack(lam, A), device="cuda")
    s = _native.stream_handle(torch.cuda.current_stream())
    outs = [torch.empty(1 + L, dtype=torch.float64, device="cuda") for _ in range(2)]
    for epoch in (1, 2, 3):                      # both slots, and a slot reused
        for k in range(2):
            ranks[k].partial(d, x.data_ptr(), None, s, epoch)
        for k in range(2):
            ranks[k].reduce_finish(d, x.data_ptr(), 0.5, outs[k].data_ptr(), s, epoch)
        torch.cuda.synchronize()
        assert not ranks[0].failed() and not ranks[1].failed()
        assert torch.equal(outs[0], outs[1])
    # the NCCL-path equivalent: sum of the two partials in rank order, then the finish
    Yw = bufs[0][L:2 * L] + bufs[1][L:2 * L]      # epoch 3 lives in slot 1
    ref = torch.empty_like(outs[0])
    ranks[0].ctx.fg_partial_device(d, r, x.data_ptr(), None, bufs[0][L:].data_ptr(), s)
    ranks[0].ctx.fg_finish_device(d, r, x.data_ptr(), Yw.data_ptr(), 0.5, ref.data_ptr(), s)
    torch.cuda.synchronize()
    assert torch.equal(ref, outs[0])
    full = mcp.fg_implicit(mcp.ObservationSet(V), lam, A, d, 0.5)
    f_s, gl_s, gA_s, _ = om.term_scales(V, np.full(p, 1 / p), lam, A, d, 0.5)
    h = outs[0].cpu().numpy()
    assert _err(h[0], full.f, f_s) <= 1e-13
    assert _err(h[1:1 + r], full.g_lam, gl_s) <= 1e-13
    assert _err(h[1 + r:].reshape((n, r), order="F"), full.g_A, gA_s) <= 1e-13


def test_large_n_beyond_register_tiled_kernels():
    """n = 2500 > the register-tiled K1 limit (2048): K1G keeps Y in L2 and handles any n."""
    rng = np.random.default_rng(44)
    n, p, r, d = 2500, 700, 6, 3
    V = rng.standard_normal((n, p)) / np.sqrt(n)
    lam, A = rng.standard_normal(r), rng.standard_normal((n, r)) / np.sqrt(n)
    res = mcp.fg_implicit(mcp.ObservationSet(V), lam, A, d, 0.3)
    nu = np.full(p, 1.0 / p)
    f, gl, gA = om.fg_implicit(V, nu, lam, A, d, 0.3)
    f_s, gl_s, gA_s, _ = om.term_scales(V, nu, lam, A, d, 0.3)
    assert _err(res.f, f, f_s) <= FG_TOL
    assert _err(res.g_lam, gl, gl_s) <= FG_TOL
    assert _err(res.g_A, gA, gA_s) <= FG_TOL


@pytest.mark.parametrize("n,r,d", [(160, 20, 3), (288, 40, 4), (384, 72, 3), (64, 70, 5)])
def test_fast_mode_tile_shapes_vs_oracle(n, r, d):
    """tcgen05 fast mode over the shapes that switch its tiling: GEMM2's 3-D TMA boxes with
    out-of-range column chunks (n % 128 != 0, n % 32 == 0), several factor column blocks
    (r > 64), and the 2-D path (n < 128); against the CPU oracle within the stated bound."""
    rng = np.random.default_rng(n + r)
    p = 9000
    V = (rng.standard_normal((n, p)) / np.sqrt(n)).astype(np.float32)
    lam, A = rng.standard_normal(r), rng.standard_normal((n, r)) / np.sqrt(n)
    res = mcp.fg_implicit(mcp.ObservationSet(V), lam, A, d, 0.1, mode="tf32x3")
    V64 = V.astype(np.float64)
    nu = np.full(p, 1.0 / p)
    f, gl, gA = om.fg_implicit(V64, nu, lam, A, d, 0.1)
    f_s, gl_s, gA_s, _ = om.term_scales(V64, nu, lam, A, d, 0.1)
    e = max(_err(res.f, f, f_s), _err(res.g_lam, gl, gl_s), _err(res.g_A, gA, gA_s))
    assert e <= FAST_TOL, e


@pytest.mark.parametrize("n,r", [(1024, 256), (900, 200)])
def test_fast_mode_transient_tiles_deterministic(n, r):
    """Fast mode with transient GEMM2 m-tiles (c5 shape: two per tile, RB = 64) drained by bulk
    tensor reduce-adds: repeated evaluations are bitwise identical (each tile's
    reduce-adds complete before the next tile's are issued, so the add order is fixed), and the
    result stays within the stated bound of FP64."""
    rng = np.random.default_rng(n + r)
    p = 20_000
    V = (rng.standard_normal((n, p)) / np.sqrt(n)).astype(np.float32)
    lam = rng.standard_normal(r)
    A = rng.standard_normal((n, r)) / np.sqrt(n)
    obs = mcp.ObservationSet(V)
    a = mcp.fg_implicit(obs, lam, A, 3, 0.0, mode="tf32x3")
    assert "transient" in obs.device_context().last_variant, obs.device_context().last_variant
    b = mcp.fg_implicit(obs, lam, A, 3, 0.0, mode="tf32x3")
    assert a.f == b.f and np.array_equal(a.g_lam, b.g_lam) and np.array_equal(a.g_A, b.g_A)
    ref = mcp.fg_implicit(obs, lam, A, 3, 0.0)
    e = max(abs(a.f - ref.f) / abs(ref.f),
            np.linalg.norm(a.g_A - ref.g_A) / np.linalg.norm(ref.g_A),
            np.linalg.norm(a.g_lam - ref.g_lam) / np.linalg.norm(ref.g_lam))
    assert e <= 1e-4, e
