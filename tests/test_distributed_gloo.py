"""The N>1 host path (shard bounds, all-reduce of [Y|w], tail on every rank) with world_size 2
over gloo on CPU.  The per-shard compute is the CPU oracle standing in for the CUDA partial
(test infrastructure); the product's own collective and tail plumbing is what runs."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import momentcp_oracle as om


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class OracleShardBackend:
    def __init__(self, V_rows_nxp, nu_rows):
        self.V, self.nu = V_rows_nxp, nu_rows

    def partial(self, lam, A, d):
        Y, w = om.fg_partial(self.V, self.nu, A, d)
        return torch.as_tensor(np.concatenate([Y.ravel(order="F"), w]))

    def finish(self, lam, A, d, alpha, Yw):
        n, r = A.shape
        h = Yw.numpy()
        return om.finish_from_partial(h[:n * r].reshape((n, r), order="F"), h[n * r:], lam, A,
                                      d, alpha)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1911_03813_b200 import distributed as D
        from paper_1911_03813_b200.dense import ObservationSet

        rng = np.random.default_rng(77)
        n, p, r, d = 9, 301, 4, 3
        V = rng.standard_normal((n, p))
        lam, A = rng.standard_normal(r), rng.standard_normal((n, r))
        lo, hi = D.shard_bounds(p, world, rank)
        nu = np.full(p, 1.0 / p)
        local = ObservationSet(V[:, lo:hi])            # host object; compute via the backend
        sobs = D.ShardedObservationSet(local, p, lo,
                                       backend=OracleShardBackend(V[:, lo:hi], nu[lo:hi]))
        res = D.fg_implicit_sharded(sobs, lam, A, d, 0.5)
        fg = D.packed_fg_sharded(sobs, d, r, 0.5)
        f2, g2 = fg(om.pack(lam, A))
        full = om.fg_implicit(V, nu, lam, A, d, 0.5)
        dn = D.data_norm_sq_split(
            local, 4, part_fn=lambda k, W: _pair_slice(V, nu, 4, k, W))
        q.put((rank, res.f, res.g_lam, res.g_A, f2, g2, full, dn, om.data_norm_sq(V, nu, 4)))
    finally:
        dist.destroy_process_group()


def _pair_slice(V, nu, d, k, W):
    # the same row-major block-pair split the CUDA path uses, at block 50
    p = V.shape[1]
    B = 50
    T = (p + B - 1) // B
    pairs = [(i, j) for i in range(T) for j in range(i, T)]
    lo, hi = len(pairs) * k // W, len(pairs) * (k + 1) // W
    s = 0.0
    for i, j in pairs[lo:hi]:
        G = om.rm_power(V[:, i * B:(i + 1) * B].T @ V[:, j * B:(j + 1) * B], d)
        t = float(nu[i * B:(i + 1) * B] @ G @ nu[j * B:(j + 1) * B])
        s += t if i == j else 2.0 * t
    return s


def test_two_rank_sharded_fg_matches_oracle():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(k, world, port, q)) for k in range(world)]
    for pr in procs:
        pr.start()
    results = [q.get(timeout=180) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    results.sort(key=lambda t: t[0])
    (_, f0, gl0, gA0, f20, g20, full, dn0, dn_ref), (_, f1, gl1, gA1, *_rest) = results
    # every rank holds identical results
    assert f0 == f1 and np.array_equal(gl0, gl1) and np.array_equal(gA0, gA1)
    f, gl, gA = full
    assert abs(f0 - f) <= 1e-12 * max(1.0, abs(f))
    assert np.allclose(gl0, gl, rtol=1e-12, atol=1e-14)
    assert np.allclose(gA0, gA, rtol=1e-12, atol=1e-14)
    assert f20 == f0 and np.array_equal(g20, om.pack(gl0, gA0))
    assert dn0 == pytest.approx(dn_ref, rel=1e-12)
    assert dn0 == results[1][7]


def test_shard_bounds_cover_rows_exactly():
    from paper_1911_03813_b200.distributed import shard_bounds

    for p in (1, 7, 100, 1_000_001):
        for world in (1, 2, 4, 8):
            spans = [shard_bounds(p, world, k) for k in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == p
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1


# ---- sharded ||X||^2: the ring pass over row shards (distributed.data_norm_sq_sharded) ----

class OracleRingBackend:
    """Oracle stand-in for CudaShardBackend's ring interface: shards travel as raw float64
    bytes (p_pad x n rows, zero padded) exactly like the device buffers, and the tile-pair
    partition (16-row tiles, row-/column-major halves) follows the kernel's."""

    TILE = 16

    def __init__(self, V_rows_nxp, nu_rows, explicit_nu):
        n, p = V_rows_nxp.shape
        self.n = n
        self.p_pad = -(-p // self.TILE) * self.TILE
        R = np.zeros((self.p_pad, n))
        R[:p] = V_rows_nxp.T
        self.R = R
        self.nu = np.zeros(self.p_pad)
        self.nu[:p] = nu_rows
        self.explicit = explicit_nu
        self.nu_const = float(nu_rows[0])

    def shard(self):
        rows = torch.from_numpy(self.R.copy()).view(torch.uint8).reshape(-1)
        nu = torch.from_numpy(self.nu.copy()).view(torch.uint8) if self.explicit else None
        return rows, self.p_pad, nu, self.nu_const

    def row_bytes(self):
        return self.n * 8

    def buffer(self, nbytes):
        return torch.empty(int(nbytes), dtype=torch.uint8)

    def _nu_of(self, nu_bytes, nu_const, p_pad, R):
        if nu_bytes is not None:
            return nu_bytes.view(torch.float64).numpy()
        # uniform weights: nu_const on every row, padding rows are zero and contribute 0
        return np.full(p_pad, nu_const)

    def self_sum(self, d):
        B, T = self.TILE, self.p_pad // self.TILE
        nu = self.nu if self.explicit else np.full(self.p_pad, self.nu_const)
        s = 0.0
        for i in range(T):
            for j in range(i, T):
                G = om.rm_power(self.R[i * B:(i + 1) * B] @ self.R[j * B:(j + 1) * B].T, d)
                t = float(nu[i * B:(i + 1) * B] @ G @ nu[j * B:(j + 1) * B])
                s += t if i == j else 2.0 * t
        return s

    def cross_sum(self, rows, p_pad, nu_bytes, nu_const, d, part, nparts, order):
        B = self.TILE
        RJ = rows.view(torch.float64).numpy().reshape(p_pad, self.n)
        nuJ = self._nu_of(nu_bytes, nu_const, p_pad, RJ)
        nuI = self.nu if self.explicit else np.full(self.p_pad, self.nu_const)
        TI, TJ = self.p_pad // B, p_pad // B
        pairs = TI * TJ
        lo, hi = pairs * part // nparts, pairs * (part + 1) // nparts
        s = 0.0
        for k in range(lo, hi):
            i, j = (k // TJ, k % TJ) if order == 0 else (k % TI, k // TI)
            G = om.rm_power(self.R[i * B:(i + 1) * B] @ RJ[j * B:(j + 1) * B].T, d)
            s += 2.0 * float(nuI[i * B:(i + 1) * B] @ G @ nuJ[j * B:(j + 1) * B])
        return s


def _ring_worker(rank, world, port, q, explicit_nu):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1911_03813_b200 import distributed as D
        from paper_1911_03813_b200.dense import ObservationSet

        rng = np.random.default_rng(5)
        n, p, d = 6, 157, 4
        V = rng.standard_normal((n, p))
        nu = rng.uniform(0.5, 1.5, p) / p if explicit_nu else np.full(p, 1.0 / p)
        lo, hi = D.shard_bounds(p, world, rank)
        sobs = D.ShardedObservationSet(ObservationSet(V[:, lo:hi]), p, lo)
        be = OracleRingBackend(V[:, lo:hi], nu[lo:hi], explicit_nu)
        val = D.data_norm_sq_sharded(sobs, d, backend=be)
        q.put((rank, val, om.data_norm_sq(V, nu, d)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,explicit_nu", [(2, False), (3, True), (4, False)])
def test_sharded_data_norm_ring_matches_oracle(world, explicit_nu):
    """Every unordered shard pair is reduced exactly once (odd W: floor(W/2) ring steps; even W:
    the last pair split between its two ranks) and all ranks agree bitwise."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ring_worker, args=(k, world, port, q, explicit_nu))
             for k in range(world)]
    for pr in procs:
        pr.start()
    results = [q.get(timeout=240) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    vals = {r[1] for r in results}
    assert len(vals) == 1, results
    got, want = results[0][1], results[0][2]
    assert got == pytest.approx(want, rel=1e-12)
