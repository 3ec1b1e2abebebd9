"""K1Z, the single-launch small-problem f+grad (csrc/k1z_small.cuh), through the C ABI.

* against the CPU oracle over shapes that cover the 8 / 16 / 32-row GEMM1 passes, both column
  paddings (r <= 8, 16, 32), n not a multiple of 4 or 8, one and many CTAs, ragged last CTAs
  and passes, several slabs per CTA, fp32 and fp64 rows, explicit weights, d = 2..6 -- term-scale <= 1e-10 (pkg/tests/test_acceptance.py:65-74);
* against the general K1 -> reduce+finish chain (MCP_OPT_SMALL_KERNEL = 0) to 1e-13;
* repeated evaluations bit-identical, gradients bitwise independent of alpha, lambda = 0 exact
  (test_objective.py:101-121);
* a sampled set evaluates to the bits of an uploaded copy of the same rows (the split depends
  on the shape only); the device Adam reads its mini-batch rows through the index list, which
  tests/test_gpu_stochastic.py pins bitwise against evaluations of uploaded copies.
"""

import numpy as np
import pytest

import paper_1911_03813_b200 as mcp
from paper_1911_03813_b200 import _native
from oracle import momentcp_oracle as om

pytestmark = pytest.mark.gpu

SHAPES = [
    # n, r, d, p, dtype, weighted
    (500, 10, 3, 1_000, np.float64, False),   # the paper's Table 2 mini-batch: 8-row passes
    (500, 10, 3, 10, np.float64, False),      # two CTAs
    (200, 5, 2, 7, np.float64, False),        # one CTA (no grid barrier), ragged pass
    (300, 12, 4, 150, np.float64, True),      # 19 CTAs, the last ragged, explicit weights
    (130, 16, 6, 2_000, np.float64, False),   # 16-row passes, all 16 columns, d = 6
    (512, 16, 3, 1_900, np.float64, True),    # largest n and r
    (512, 6, 3, 5_000, np.float64, False),    # 32-row passes, 64 rows per CTA in two slabs
    (257, 3, 5, 700, np.float32, False),      # fp32 rows, n = 1 (mod 4) and (mod 8)
    (33, 8, 4, 18_000, np.float32, True),     # fp32 rows, 128 rows per CTA, 5 variable tiles
    (20, 5, 3, 10_000, np.float32, False),    # config 1's shape on fp32 rows: 3 variable tiles
    (7, 1, 2, 5, np.float32, False),          # one CTA, one column, one variable tile
    (129, 9, 3, 4_736, np.float64, False),    # 32 rows on every CTA of a 148-SM part
    (320, 7, 3, 18_000, np.float64, False),   # 128 rows per CTA: four 32-row passes per slab
    (500, 32, 3, 1_000, np.float64, False),   # 32 columns (four column tiles), 8-row passes
    (300, 20, 4, 2_000, np.float64, True),    # 32-column padding of r = 20, 16-row passes
    (512, 32, 3, 900, np.float64, False),     # largest n and r: the shared-memory limit
    (200, 25, 2, 60, np.float32, False),      # fp32 rows, 32-column padding, 8 CTAs
]


def _instance(k, n, r, d, p, dtype, weighted):
    rng = np.random.default_rng(1000 + k)
    V = (rng.standard_normal((n, p)) / np.sqrt(n)).astype(dtype)
    nu = (rng.random(p) + 0.5) / p if weighted else None
    lam = rng.standard_normal(r)
    A = rng.standard_normal((n, r)) / np.sqrt(n)
    return V, nu, lam, A, 0.375


def _check(res, V, nu, lam, A, d, alpha, tol):
    V64 = V.astype(np.float64)
    nu_ = np.full(V.shape[1], 1.0 / V.shape[1]) if nu is None else nu
    f, gl, gA = om.fg_implicit(V64, nu_, lam, A, d, alpha)
    f_s, gl_s, gA_s, _ = om.term_scales(V64, nu_, lam, A, d, alpha)
    e = max(om.term_rel_err(res.f, f, f_s), om.term_rel_err(res.g_lam, gl, gl_s),
            om.term_rel_err(res.g_A, gA, gA_s))
    assert e <= tol, e


@pytest.mark.parametrize("k", range(len(SHAPES)))
def test_k1z_vs_oracle_and_general_chain(k):
    n, r, d, p, dtype, weighted = SHAPES[k]
    V, nu, lam, A, alpha = _instance(k, *SHAPES[k])
    obs = mcp.ObservationSet(V, nu)
    ctx = obs.device_context()
    res = mcp.fg_implicit(obs, lam, A, d, alpha)
    assert ctx.last_variant.startswith("k1z_fg_small"), ctx.last_variant
    assert ctx.last_launch_count == 1
    _check(res, V, nu, lam, A, d, alpha, 1e-10)
    again = mcp.fg_implicit(obs, lam, A, d, alpha)
    assert again.f == res.f and np.array_equal(again.g_lam, res.g_lam)
    assert np.array_equal(again.g_A, res.g_A)
    shifted = mcp.fg_implicit(obs, lam, A, d, alpha + 3.0)
    assert np.array_equal(shifted.g_lam, res.g_lam) and np.array_equal(shifted.g_A, res.g_A)
    zero = mcp.fg_implicit(obs, np.zeros(r), A, d, alpha)
    assert zero.f == alpha and np.array_equal(zero.g_A, np.zeros_like(A))
    ctx.set_option(_native.MCP_OPT_SMALL_KERNEL, 0)
    try:
        gen = mcp.fg_implicit(obs, lam, A, d, alpha)
        assert not ctx.last_variant.startswith("k1z"), ctx.last_variant
    finally:
        ctx.set_option(_native.MCP_OPT_SMALL_KERNEL, 1)
    V64 = V.astype(np.float64)
    nu_ = np.full(p, 1.0 / p) if nu is None else nu
    f_s, gl_s, gA_s, _ = om.term_scales(V64, nu_, lam, A, d, alpha)
    e = max(om.term_rel_err(res.f, gen.f, f_s), om.term_rel_err(res.g_lam, gen.g_lam, gl_s),
            om.term_rel_err(res.g_A, gen.g_A, gA_s))
    assert e <= 1e-13, e


def test_k1z_limits_fall_back_to_the_general_chain():
    """Outside K1Z's limits (r <= 32, n <= 512, at most 128 rows per SM) and for fp64 sets with
    n <= 128 (where the two-launch K1Q chain measured faster) the general chain runs."""
    rng = np.random.default_rng(5)
    for n, r, p in ((200, 33, 500), (513, 4, 300), (300, 10, 30_000), (100, 10, 3_000)):
        V = rng.standard_normal((n, p)) / np.sqrt(n)
        obs = mcp.ObservationSet(V)
        lam, A = rng.standard_normal(r), rng.standard_normal((n, r)) / np.sqrt(n)
        res = mcp.fg_implicit(obs, lam, A, 3, 0.0)
        assert not obs.device_context().last_variant.startswith("k1z")
        _check(res, V, None, lam, A, 3, 0.0, 1e-10)


def test_k1z_sampled_set_equals_uploaded_copy_bitwise():
    """sample_observations -> fg equals, bitwise, the evaluation of an uploaded copy of the same
    rows (objective.py:97-113): the work split is a function of the shape only."""
    rng = np.random.default_rng(8)
    for n, r, d, p, s in ((200, 5, 3, 4_000, 300), (500, 10, 3, 3_000, 1_000), (264, 8, 4, 900, 7)):
        V = rng.standard_normal((n, p)) / np.sqrt(n)
        obs = mcp.ObservationSet(V)
        lam, A = rng.standard_normal(r), rng.standard_normal((n, r)) / np.sqrt(n)
        sub = mcp.sample_observations(obs, s, np.random.default_rng(77))
        idx = np.random.default_rng(77).integers(0, p, size=s)
        a = mcp.fg_implicit(sub, lam, A, d, 0.5)
        b = mcp.fg_implicit(mcp.ObservationSet(V[:, idx]), lam, A, d, 0.5)
        assert a.f == b.f and np.array_equal(a.g_lam, b.g_lam) and np.array_equal(a.g_A, b.g_A)
        _check(a, V[:, idx], None, lam, A, d, 0.5, 1e-10)


def test_k1z_on_a_row_shard_uses_the_set_weight():
    """A device-resident row shard (weights 1 / p_total, not 1 / rows): K1Z and the general chain
    agree, and both equal the oracle on explicit weights 1 / p_total."""
    import torch

    rng = np.random.default_rng(14)
    n, rows, p_total, r, d = 240, 900, 5_000, 6, 3
    V = rng.standard_normal((n, rows)) / np.sqrt(n)
    lam, A = rng.standard_normal(r), rng.standard_normal((n, r)) / np.sqrt(n)
    obs = mcp.ObservationSet.from_device(torch.as_tensor(V.T.copy(), device="cuda"),
                                         p_total=p_total)
    ctx = obs.device_context()
    x = torch.as_tensor(mcp.pack(lam, A), device="cuda")
    s = _native.stream_handle(torch.cuda.current_stream())
    outs = []
    for small in (1, 0):
        ctx.set_option(_native.MCP_OPT_SMALL_KERNEL, small)
        o = torch.empty(1 + r + n * r, dtype=torch.float64, device="cuda")
        ctx.fg_device(d, r, x.data_ptr(), 0.125, None, o.data_ptr(), s)
        torch.cuda.synchronize()
        assert ctx.last_variant.startswith("k1z") == bool(small), ctx.last_variant
        outs.append(o.cpu().numpy())
    ctx.set_option(_native.MCP_OPT_SMALL_KERNEL, 1)
    nu = np.full(rows, 1.0 / p_total)
    f, gl, gA = om.fg_implicit(V, nu, lam, A, d, 0.125)
    f_s, gl_s, gA_s, _ = om.term_scales(V, nu, lam, A, d, 0.125)
    for got, tol in ((outs[0], 1e-10), (outs[1], 1e-10)):
        e = max(om.term_rel_err(got[0], f, f_s), om.term_rel_err(got[1:1 + r], gl, gl_s),
                om.term_rel_err(got[1 + r:], gA.reshape(-1, order="F"),
                                gA_s.reshape(-1, order="F")))
        assert e <= tol, e
    e = max(om.term_rel_err(outs[0][0], outs[1][0], f_s),
            om.term_rel_err(outs[0][1 + r:], outs[1][1 + r:], gA_s.reshape(-1, order="F")))
    assert e <= 1e-13, e


@pytest.mark.parametrize("shape", [(500, 10, 3, 1_000), (20, 5, 3, 10_000)])
def test_device_evaluations_capture_into_a_callers_cuda_graph(shape):
    """fg_device launches on the stream it is given, so a caller may capture evaluations into a
    CUDA graph of its own (the cooperative K1Z launch and the K1Q -> K3F chain under programmatic
    dependent launch both capture); replays reproduce the eager result bitwise."""
    import torch

    n, r, d, p = shape
    rng = np.random.default_rng(p)
    V = rng.standard_normal((n, p)) / np.sqrt(n)
    ctx = mcp.ObservationSet(V).device_context()
    lam, A = rng.standard_normal(r), rng.standard_normal((n, r)) / np.sqrt(n)
    x = torch.as_tensor(mcp.pack(lam, A), device="cuda")
    out = torch.empty(1 + r + n * r, dtype=torch.float64, device="cuda")
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        s = _native.stream_handle(torch.cuda.current_stream())
        ctx.fg_device(d, r, x.data_ptr(), 0.5, None, out.data_ptr(), s)
        torch.cuda.synchronize()
        eager = out.clone()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=side):
            s = _native.stream_handle(torch.cuda.current_stream())
            for _ in range(3):
                ctx.fg_device(d, r, x.data_ptr(), 0.5, None, out.data_ptr(), s)
        out.zero_()
        graph.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, eager)
        x.mul_(1.5)            # the graph reads x in place: a new point, no re-capture
        graph.replay()
        torch.cuda.synchronize()
        replayed = out.clone()
        ctx.fg_device(d, r, x.data_ptr(), 0.5, None, out.data_ptr(), s)
        torch.cuda.synchronize()
        assert torch.equal(out, replayed)
