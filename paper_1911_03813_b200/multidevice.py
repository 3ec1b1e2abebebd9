"""One observation set spread over several GPUs, driven from ONE process.

The reference drives f+grad from a single process (pkg/src/momentcp/optimize.py:255-355, with
threads for multistart at :484-493).  ``MultiDeviceObservationSet`` keeps that programming model
on a multi-GPU node: the rows of V are split into contiguous shards, one per device (each a
regular device-resident :class:`ObservationSet` with uniform weight 1/p_total or its slice of
nu), and one evaluation

  1. enqueues every shard's additive piece [vec_F(Y) | w] (K1 -> K3, ``mcp_fg_partial_device``)
     on its own device's stream -- all GPUs compute concurrently;
  2. adds the pieces on the first device in shard order (peer copies over NVLink, a fixed-order
     sum, so results are deterministic and independent of timing);
  3. runs the O(n r^2) tail once (``mcp_fg_finish_device``) and returns f, g_lam, g_A.

``packed_fg(d, r)`` is a plain ``fg(x) -> (f, g)`` callback, so ``lbfgs_minimize`` drives it with
the host solver (the reference's decisions, :mod:`.host_solver`) -- the headline user flow, a
full c5 fit, runs on every GPU of the node from one Python process.  ``data_norm_sq`` sums each
shard's own Gram triangle and every shard pair's rectangle (``mcp_data_norm_sq_cross``, the pair's
second shard copied to the first's device), in a fixed order.

Several shards may share one device (the tests do this on a one-GPU box); the arithmetic is the
same.
"""

from __future__ import annotations

import time

import numpy as np

from ._native import stream_handle
from .dense import ObservationSet
from .objective import FgResult, validate_variables
from .optimize import pack


def _torch():
    import torch

    return torch


class MultiDeviceObservationSet:
    """Row shards of one set of p observations in R^n, shard k on ``devices[k]``."""

    def __init__(self, shards: list[ObservationSet], devices: list[int], p_total: int,
                 row_offsets: list[int]):
        if not shards or len(shards) != len(devices) or len(shards) != len(row_offsets):
            raise ValueError("one device and one row offset per shard")
        n = shards[0].n
        if any(s.n != n for s in shards):
            raise ValueError("every shard must have the same number of variables")
        self.shards, self.devices = list(shards), [int(d) for d in devices]
        self.n, self.p = n, int(p_total)
        self.row_offsets = [int(o) for o in row_offsets]

    # -- construction -----------------------------------------------------------------------
    @classmethod
    def from_host(cls, V, devices, nu=None):
        """Split the (n, p) host matrix V (reference ObservationSet layout) by rows of the
        observation-major view over ``devices`` (one contiguous shard per entry)."""
        from .distributed import shard_bounds

        V = np.asarray(V)
        if V.ndim != 2:
            raise ValueError(f"V must be a 2-D matrix, got ndim={V.ndim}")
        n, p = V.shape
        if n < 1 or p < 1:
            raise ValueError(f"V must be at least 1x1, got shape {V.shape}")
        if not np.isfinite(V).all():
            raise ValueError("V contains non-finite entries")
        if nu is not None:
            nu = np.asarray(nu, dtype=float)
            if nu.shape != (p,):
                raise ValueError(f"nu must have length p={p}, got shape {nu.shape}")
            if not np.isfinite(nu).all() or np.any(nu <= 0.0):
                raise ValueError("nu entries must be finite and strictly positive")
        devices = list(devices)
        W = len(devices)
        shards, offs = [], []
        Vt = np.ascontiguousarray(V.T) if V.dtype in (np.float32, np.float64) else \
            np.ascontiguousarray(V.T, dtype=float)
        for k, dev in enumerate(devices):
            lo, hi = shard_bounds(p, W, k)
            shards.append(ObservationSet.from_obs_major_host(
                Vt[lo:hi], None if nu is None else nu[lo:hi], p_total=p, device=dev))
            offs.append(lo)
        return cls(shards, devices, p, offs)

    @classmethod
    def from_device_rows(cls, rows: list, p_total: int):
        """Wrap per-device CUDA tensors of observations (rows_k x n each), in row order."""
        shards, devs, offs, off = [], [], [], 0
        for t in rows:
            shards.append(ObservationSet.from_device(t, p_total=p_total, release=True))
            devs.append(t.device.index or 0)
            offs.append(off)
            off += t.shape[0]
        if off != p_total:
            raise ValueError(f"the shards hold {off} rows, expected p_total={p_total}")
        return cls(shards, devs, p_total, offs)

    # -- f + grad ---------------------------------------------------------------------------
    def _partials(self, x_host: np.ndarray, d: int, r: int, mode):
        torch = _torch()
        parts = []
        for s, dev in zip(self.shards, self.devices):
            ctx = s.device_context()
            tdev = torch.device("cuda", dev)
            x = torch.as_tensor(x_host, dtype=torch.float64).to(tdev, non_blocking=False)
            Yw = torch.empty(self.n * r + r, dtype=torch.float64, device=tdev)
            ctx.fg_partial_device(d, r, x.data_ptr(), mode, Yw.data_ptr(),
                                  stream_handle(torch.cuda.current_stream(tdev)))
            parts.append((Yw, x))   # x stays alive until its stream has consumed it
        return parts

    def fg(self, lam, A, d: int, alpha: float = 0.0, mode: str | None = None) -> FgResult:
        """fg_implicit over all shards (reference objective.py:77-94)."""
        torch = _torch()
        lam, A = validate_variables(lam, A, self.n, alpha)
        if d < 2:
            raise ValueError(f"order must be >= 2, got {d}")
        start = time.perf_counter()
        n, r = self.n, A.shape[1]
        x_host = pack(lam, A)
        parts = self._partials(x_host, d, r, mode)
        dev0 = torch.device("cuda", self.devices[0])
        total = parts[0][0].clone()
        for Yw, _ in parts[1:]:
            total += Yw.to(dev0)          # shard order: a fixed summation order
        ctx0 = self.shards[0].device_context()
        x0 = parts[0][1]
        out = torch.empty(1 + r + n * r, dtype=torch.float64, device=dev0)
        ctx0.fg_finish_device(d, r, x0.data_ptr(), total.data_ptr(), float(alpha), out.data_ptr(),
                              stream_handle(torch.cuda.current_stream(dev0)))
        h = out.cpu().numpy()
        return FgResult(float(h[0]), h[1:1 + r].copy(), h[1 + r:].reshape((n, r), order="F").copy(),
                        time.perf_counter() - start, "implicit")

    def packed_fg(self, d: int, r: int, alpha: float = 0.0, mode: str | None = None):
        """``fg(x) -> (f, g)`` on packed variables (reference optimize.py:123-134)."""
        n = self.n
        if d < 2:
            raise ValueError(f"order must be >= 2, got {d}")

        def fg(x):
            x = np.asarray(x, dtype=float)
            if x.shape != (r + n * r,):
                raise ValueError(f"expected packed length {r + n * r}, got {x.shape}")
            res = self.fg(x[:r].copy(), x[r:].reshape((n, r), order="F").copy(), d, alpha, mode)
            return res.f, pack(res.g_lam, res.g_A)

        return fg

    # -- ||X||^2 ------------------------------------------------------------------------------
    def data_norm_sq(self, d: int, mode: str | None = None) -> float:
        """||X||^2 of the whole set (implicit.py:116-121): shard triangles plus every shard
        pair's rectangle, added in a fixed order."""
        torch = _torch()
        if d < 2:
            raise ValueError(f"order must be >= 2, got {d}")
        total = 0.0
        W = len(self.shards)
        for k in range(W):
            total += self.shards[k].device_context().data_norm_sq(d, mode)
        for i in range(W):
            ci = self.shards[i].device_context()
            di = torch.device("cuda", self.devices[i])
            for j in range(i + 1, W):
                vj = self.shards[j].device_context().obs_device_view()
                elem = 8 if vj["dtype"] == 0 else 4
                if self.devices[j] == self.devices[i]:
                    ptr, nu_ptr, keep = vj["ptr"], vj["nu"], None
                else:
                    from .distributed import _CudaBytes

                    dj = torch.device("cuda", self.devices[j])
                    rows = torch.as_tensor(_CudaBytes(vj["ptr"], vj["p_pad"] * vj["ldv"] * elem),
                                           device=dj).to(di)
                    nuc = (torch.as_tensor(_CudaBytes(vj["nu"], vj["p_pad"] * 8), device=dj).to(di)
                           if vj["nu"] else None)
                    torch.cuda.synchronize(di)
                    ptr, nu_ptr, keep = rows.data_ptr(), (nuc.data_ptr() if nuc is not None
                                                          else 0), (rows, nuc)
                total += ci.data_norm_sq_cross(ptr, vj["p_pad"], nu_ptr or None, vj["nu_const"],
                                               d, mode)
                del keep
        return total
