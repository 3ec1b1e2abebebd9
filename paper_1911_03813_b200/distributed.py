"""Row-sharded evaluation over 1/2/4/8 GPUs (one process per GPU, torch.distributed / NCCL).

The reference is single-process.  Observations are independent, so
Y = sum_l nu_l z_l^(d-1) v_l and w = sum_l nu_l z_l^d are sums over rows of V: each rank holds a
contiguous row block, computes its additive piece [vec_F(Y) | w] on the device (prep -> K1 -> K3,
mcp_fg_partial_device), one all-reduce(sum) of that n*r + r vector is the only exchange, and
every rank runs the O(n r^2) tail (mcp_fg_finish_device) on the reduced piece, so all ranks hold
identical f and gradients.  Uniform weights are 1/p_total on every shard (dense.py:90-91 over
the whole set).

||X||^2 (implicit.py:116-121) couples every pair of observations.  ``data_norm_sq_sharded``
works on the row shards themselves (no rank ever holds the whole V): rank k computes its own
shard's triangle, then the shards travel one hop per step around a ring (NCCL send/recv over
NVLink, the next hop in flight while the current shard's rectangle is reduced), and at step s
rank k reduces the rectangle (k, k+s) -- floor(W/2) steps cover every unordered shard pair once
(for even W the last pair is split in half between its two ranks).  The W partial sums are
all-gathered and added in rank order (deterministic, identical on every rank).
``data_norm_sq_split`` is the replicated variant (every rank holds all of V).

The per-shard compute is pluggable only so the host-side logic (shard bounds, collective,
tail) can be exercised on CPU with gloo in tests; the product path is the CUDA backend, which
raises if the native library or GPU is missing.
"""

from __future__ import annotations

import time

import numpy as np

from ._native import stream_handle
from .dense import ObservationSet
from .objective import FgResult, validate_variables
from .optimize import pack


def shard_bounds(p: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row block [lo, hi) of rank `rank` out of `world` (sizes differ by <= 1)."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of size {world}")
    return p * rank // world, p * (rank + 1) // world


def _torch():
    import torch

    return torch


def device_partial(obs: ObservationSet, lam, A, d: int, mode: str | None = None):
    """[vec_F(Y) | w] of this shard as a CUDA float64 tensor, on the current stream."""
    torch = _torch()
    ctx = obs.device_context()
    n, r = A.shape
    dev = torch.device("cuda", ctx.device)
    x = torch.as_tensor(pack(lam, A), dtype=torch.float64, device=dev)
    Yw = torch.empty(n * r + r, dtype=torch.float64, device=dev)
    stream = stream_handle(torch.cuda.current_stream(dev))
    ctx.fg_partial_device(d, r, x.data_ptr(), mode, Yw.data_ptr(), stream)
    Yw._mcp_x = x  # keep x alive until the stream has consumed it
    return Yw


def device_finish(obs: ObservationSet, lam, A, d: int, alpha: float, Yw):
    """Tail on the reduced piece -> (f, g_lam, g_A) on the host."""
    torch = _torch()
    ctx = obs.device_context()
    n, r = A.shape
    dev = torch.device("cuda", ctx.device)
    x = torch.as_tensor(pack(lam, A), dtype=torch.float64, device=dev)
    out = torch.empty(1 + r + n * r, dtype=torch.float64, device=dev)
    stream = stream_handle(torch.cuda.current_stream(dev))
    ctx.fg_finish_device(d, r, x.data_ptr(), Yw.data_ptr(), float(alpha), out.data_ptr(), stream)
    h = out.cpu().numpy()
    return float(h[0]), h[1:1 + r].copy(), h[1 + r:].reshape((n, r), order="F").copy()


class _CudaBytes:
    """Zero-copy torch view (uint8) of device memory owned by the native context."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (int(nbytes),), "typestr": "|u1",
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None}


class CudaShardBackend:
    """Per-shard compute on this rank's GPU through the C ABI."""

    def __init__(self, obs: ObservationSet, mode: str | None = None):
        self.obs = obs
        self.mode = mode

    def partial(self, lam, A, d):
        return device_partial(self.obs, lam, A, d, self.mode)

    def finish(self, lam, A, d, alpha, Yw):
        return device_finish(self.obs, lam, A, d, alpha, Yw)

    # -- sharded ||X||^2 (ring pass) -------------------------------------------------------
    def shard(self):
        """(rows bytes tensor, padded rows, weights bytes tensor or None, uniform weight)."""
        torch = _torch()
        ctx = self.obs.device_context()
        v = ctx.obs_device_view()
        elem = 8 if v["dtype"] == 0 else 4
        dev = torch.device("cuda", ctx.device)
        rows = torch.as_tensor(_CudaBytes(v["ptr"], v["p_pad"] * v["ldv"] * elem), device=dev)
        nu = (torch.as_tensor(_CudaBytes(v["nu"], v["p_pad"] * 8), device=dev)
              if v["nu"] else None)
        self._row_bytes = v["ldv"] * elem
        return rows, v["p_pad"], nu, v["nu_const"]

    def row_bytes(self) -> int:
        return self._row_bytes

    def buffer(self, nbytes: int):
        torch = _torch()
        ctx = self.obs.device_context()
        return torch.empty(int(nbytes), dtype=torch.uint8, device=torch.device("cuda", ctx.device))

    def self_sum(self, d) -> float:
        return self.obs.device_context().data_norm_sq(d, self.mode)

    def cross_sum(self, rows, p_pad, nu, nu_const, d, part, nparts, order) -> float:
        torch = _torch()
        ctx = self.obs.device_context()
        # the library's stream is not ordered after the receive on torch's stream
        torch.cuda.current_stream(torch.device("cuda", ctx.device)).synchronize()
        return ctx.data_norm_sq_cross(rows.data_ptr(), p_pad, nu.data_ptr() if nu is not None
                                      else None, nu_const, d, self.mode, part, nparts,
                                      order)


class ShardedObservationSet:
    """This rank's row block of a p_total-observation set, plus the process group."""

    def __init__(self, local: ObservationSet, p_total: int, row_offset: int, group=None,
                 backend=None):
        self.local = local
        self.n = local.n
        self.p = int(p_total)
        self.row_offset = int(row_offset)
        self.group = group
        self.backend = backend if backend is not None else CudaShardBackend(local)

    @classmethod
    def from_device_rows(cls, V_rows, p_total: int, row_offset: int, group=None):
        """Wrap this rank's rows (rows x n CUDA tensor, observation-major)."""
        local = ObservationSet.from_device(V_rows, p_total=p_total)
        return cls(local, p_total, row_offset, group)


def _all_reduce_sum(t, group):
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def fg_implicit_sharded(sobs: ShardedObservationSet, lam, A, d: int, alpha: float = 0.0,
                        eval_kind: str = "implicit") -> FgResult:
    """fg_implicit over a row-sharded set: partial -> all-reduce([Y|w]) -> tail, all ranks."""
    lam, A = validate_variables(lam, A, sobs.n, alpha)
    if d < 2:
        raise ValueError(f"order must be >= 2, got {d}")
    start = time.perf_counter()
    Yw = sobs.backend.partial(lam, A, d)
    _all_reduce_sum(Yw, sobs.group)
    f, g_lam, g_A = sobs.backend.finish(lam, A, d, alpha, Yw)
    return FgResult(f, g_lam, g_A, time.perf_counter() - start, eval_kind)


def packed_fg_sharded(sobs: ShardedObservationSet, d: int, r: int, alpha: float = 0.0,
                      mode: str | None = None):
    """packed_fg_implicit for a sharded set (every rank calls it with the same x)."""
    n = sobs.n
    if mode is not None and isinstance(sobs.backend, CudaShardBackend):
        sobs.backend.mode = mode

    def fg(x):
        x = np.asarray(x, dtype=float)
        lam, A = x[:r].copy(), x[r:].reshape((n, r), order="F").copy()
        res = fg_implicit_sharded(sobs, lam, A, d, alpha)
        return res.f, pack(res.g_lam, res.g_A)

    return fg


class PeerExchangeError(RuntimeError):
    """A peer's partial never arrived (lost rank or > 30 s skew); see PeerExchange.step."""


class PeerExchange:
    """[vec_F(Y) | w] exchange over NVLink peer memory, fused with the finish (replaces the
    all-reduce + tail of the row-sharded evaluation; csrc/peer.cu).

    Each rank owns two symmetric partial slots (epoch parity) and a flag array; one evaluation is
    ``partial -> signal -> reduce_finish`` on the rank's stream, with no host round trip and no
    NCCL call, and every rank sums the partials in rank order (bitwise identical results on all
    ranks).  ``buffers`` (tests) injects plain device buffers instead of symmetric memory.
    """

    def __init__(self, ctx, n: int, r: int, rank: int, world: int, group=None, buffers=None):
        torch = _torch()
        self.ctx, self.n, self.r, self.rank, self.world = ctx, int(n), int(r), int(rank), int(world)
        dev = torch.device("cuda", ctx.device)
        self.L = self.n * self.r + self.r
        if buffers is None:
            import torch.distributed as dist
            import torch.distributed._symmetric_memory as symm

            self.buf = symm.empty(2 * self.L, dtype=torch.float64, device=dev)
            self.flags = symm.empty(self.world, dtype=torch.int64, device=dev)
            self.flags.zero_()
            torch.cuda.synchronize(dev)
            grp = group if group is not None else dist.group.WORLD
            hb = symm.rendezvous(self.buf, grp)
            hf = symm.rendezvous(self.flags, grp)
            buf_ptrs, flag_ptrs = list(hb.buffer_ptrs), list(hf.buffer_ptrs)
            dist.barrier(group)
        else:
            self.buf, self.flags, buf_ptrs, flag_ptrs = buffers
        self.parts = [torch.tensor([b + slot * self.L * 8 for b in buf_ptrs], dtype=torch.int64,
                                   device=dev) for slot in (0, 1)]
        self.flag_ptrs = torch.tensor(flag_ptrs, dtype=torch.int64, device=dev)
        self.err = torch.zeros(1, dtype=torch.int32, device=dev)
        self.epoch = 0

    def slot_ptr(self, epoch: int) -> int:
        return self.buf.data_ptr() + (epoch % 2) * self.L * 8

    def partial(self, d, x_ptr, mode, stream, epoch):
        # the partial's reduce kernel publishes the epoch itself (no separate signal launch)
        self.ctx.fg_partial_signal_device(d, self.r, x_ptr, mode, self.slot_ptr(epoch),
                                          self.flag_ptrs.data_ptr(), self.rank, self.world,
                                          epoch, stream)

    def reduce_finish(self, d, x_ptr, alpha, out_ptr, stream, epoch):
        self.ctx.peer_reduce_finish(d, self.r, x_ptr, self.parts[epoch % 2].data_ptr(),
                                    self.flags.data_ptr(), self.world, epoch, alpha, out_ptr,
                                    self.err.data_ptr(), stream)

    def step(self, d, x_ptr, mode, alpha, out_ptr, stream, check: bool = True):
        """One sharded evaluation x -> out = [f ; g_lam ; vec_F(g_A)] on every rank.

        A peer that never publishes its partial (csrc/peer.cu: 30 s bound) makes the kernel
        write NaN into every output and set the error flag.  With ``check`` (default) the step
        waits for the stream and raises ``PeerExchangeError``; timed loops pass
        ``check=False`` and call :meth:`raise_if_failed` once afterwards (outputs of a failed
        step are NaN either way, never a stale sum)."""
        self.epoch += 1
        self.partial(d, x_ptr, mode, stream, self.epoch)
        self.reduce_finish(d, x_ptr, alpha, out_ptr, stream, self.epoch)
        if check:
            self.raise_if_failed()

    def failed(self) -> bool:
        """True once any reduce of this exchange timed out waiting for a peer (syncs)."""
        return bool(self.err.item())

    def raise_if_failed(self) -> None:
        if self.failed():
            raise PeerExchangeError(
                f"rank {self.rank}: a peer's partial did not arrive within the exchange's wait "
                f"bound (epoch <= {self.epoch}); outputs were poisoned with NaN")


def data_norm_sq_sharded(sobs: ShardedObservationSet, d: int, group=None,
                         mode: str | None = None, backend=None) -> float:
    """||X||^2 of a row-sharded set (implicit.py:116-121), shards passed around a ring.

    Every rank calls it; all ranks return the same value (partials summed in rank order).
    The rounding differs from the single-GPU reduction only by the association of the tile
    sums (fixed for a given world size).
    """
    torch = _torch()
    import torch.distributed as dist

    if d < 2:
        raise ValueError(f"order must be >= 2, got {d}")
    group = group if group is not None else sobs.group
    world, rank = 1, 0
    if dist.is_available() and dist.is_initialized():
        world, rank = dist.get_world_size(group), dist.get_rank(group)
    be = backend if backend is not None else CudaShardBackend(sobs.local, mode)
    if world == 1:
        return float(be.self_sum(d))
    rows, p_pad, nu, nu_const = be.shard()
    rb = be.row_bytes()
    dev = rows.device
    # every rank's padded row count, weights flag and uniform weight
    meta = torch.tensor([float(p_pad), 1.0 if nu is not None else 0.0, nu_const],
                        dtype=torch.float64, device=dev)
    metas = [torch.zeros_like(meta) for _ in range(world)]
    dist.all_gather(metas, meta, group=group)
    metas = [m.cpu().tolist() for m in metas]
    if len({m[1] for m in metas}) != 1:
        raise ValueError("every shard must have explicit weights, or none")
    with_nu = metas[0][1] != 0.0
    pmax = int(max(m[0] for m in metas))
    gr = (lambda k: dist.get_global_rank(group, k)) if group is not None else (lambda k: k)
    left, right = gr((rank - 1) % world), gr((rank + 1) % world)
    bufs = [be.buffer(pmax * rb) for _ in range(2)]
    nubufs = [be.buffer(pmax * 8) for _ in range(2)] if with_nu else [None, None]
    steps = world // 2

    # gloo moves only host tensors point to point: device shards are staged through host
    # copies there (the multi-rank-on-one-GPU test mode); NCCL sends HBM directly
    staged = dev.type == "cuda" and dist.get_backend(group) == "gloo"

    def exchange(cur_rows, cur_nu, src_shard, slot):
        # send the shard we hold to the left neighbour, receive the next one from the right
        nb = int(metas[src_shard][0])
        pairs = [(cur_rows, bufs[slot][:nb * rb])]
        if with_nu:
            pairs.append((cur_nu, nubufs[slot][:nb * 8]))
        ops, landing = [], []
        for snd, rcv in pairs:
            if staged:
                snd = snd.cpu()
                host = torch.empty(rcv.shape, dtype=rcv.dtype)
                landing.append((host, rcv))
                rcv = host
            ops += [dist.P2POp(dist.isend, snd, left, group),
                    dist.P2POp(dist.irecv, rcv, right, group)]
        return dist.batch_isend_irecv(ops), landing

    total = float(be.self_sum(d))
    cur_rows, cur_nu = rows, nu
    reqs, landing = exchange(cur_rows, cur_nu, (rank + 1) % world, 0)
    for s in range(1, steps + 1):
        for q in reqs:
            q.wait()
        for host, rcv in landing:
            rcv.copy_(host)
        src = (rank + s) % world
        nb = int(metas[src][0])
        slot = (s - 1) % 2
        cur_rows = bufs[slot][:nb * rb]
        cur_nu = nubufs[slot][:nb * 8] if with_nu else None
        if s < steps:   # next hop in flight while this rectangle is reduced
            reqs, landing = exchange(cur_rows, cur_nu, (rank + s + 1) % world, s % 2)
        part, nparts, order = 0, 1, 0
        if world % 2 == 0 and s == steps:
            # shards k and k + W/2 meet from both sides: the lower rank takes the first half of
            # the rectangle with its own tiles outer, the upper rank the second half with the
            # lower rank's tiles outer -- together every tile pair exactly once
            part, nparts, order = (0, 2, 0) if rank < world // 2 else (1, 2, 1)
        total += float(be.cross_sum(cur_rows, nb, cur_nu, metas[src][2], d, part, nparts,
                                    order))
    mine = torch.tensor([total], dtype=torch.float64, device=dev)
    parts = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine, group=group)
    out = 0.0
    for t in parts:
        out += float(t.item())
    return out


def data_norm_sq_split(obs_full: ObservationSet, d: int, group=None, mode: str | None = None,
                       part_fn=None) -> float:
    """||X||^2 with the tile-pair list split over the ranks of `group`.

    Every rank holds the full set; rank k computes pair slice k of W, the W partial sums are
    all-gathered and added in rank order (deterministic, identical on every rank).
    """
    import torch
    import torch.distributed as dist

    if d < 2:
        raise ValueError(f"order must be >= 2, got {d}")
    world, rank = 1, 0
    if dist.is_available() and dist.is_initialized():
        world, rank = dist.get_world_size(group), dist.get_rank(group)
    if part_fn is None:
        ctx = obs_full.device_context()
        part = ctx.data_norm_sq(d, mode, rank, world) if world > 1 else ctx.data_norm_sq(d, mode)
        dev = torch.device("cuda", ctx.device)
    else:
        part = part_fn(rank, world)
        dev = torch.device("cpu")
    if world == 1:
        return float(part)
    mine = torch.tensor([part], dtype=torch.float64, device=dev)
    parts = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine, group=group)
    total = 0.0
    for t in parts:
        total += float(t.item())
    return total
