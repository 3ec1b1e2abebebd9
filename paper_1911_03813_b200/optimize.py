"""Packed-variable adapter handing the B200 f+grad to a quasi-Newton driver.

Same layout as the reference (pkg/src/momentcp/optimize.py:104-134): x = [lam; vec_F(A)],
gradient packed the same way.  ``packed_fg_implicit`` returns the ``fg(x) -> (f, g)`` closure
that ``lbfgs_minimize`` (optimize.py:255-355) and ``multistart`` (:454-508) consume; each call
is one C-ABI call (``mcp_fg_packed``): H2D of x, one CUDA-graph replay, D2H of [f; g].
"""

from __future__ import annotations

from typing import Callable

import numpy as np

from .dense import ObservationSet

FgCallback = Callable[[np.ndarray], tuple[float, np.ndarray]]


def pack(lam, A) -> np.ndarray:
    """Flatten (lam, A): lam first, then A column-major (reference optimize.py:104-110)."""
    lam = np.asarray(lam, dtype=float)
    A = np.asarray(A, dtype=float)
    if A.ndim != 2 or lam.ndim != 1 or A.shape[1] != lam.size:
        raise ValueError(f"inconsistent shapes: lam {lam.shape}, A {A.shape}")
    return np.concatenate([lam, A.ravel(order="F")])


def unpack(x, n: int, r: int) -> tuple[np.ndarray, np.ndarray]:
    """Invert :func:`pack` for an n x r factor matrix (reference optimize.py:113-120)."""
    x = np.asarray(x, dtype=float)
    if x.shape != (r + n * r,):
        raise ValueError(f"expected packed length {r + n * r}, got {x.shape}")
    return x[:r].copy(), x[r:].reshape((n, r), order="F").copy()


def packed_fg_implicit(obs: ObservationSet, d: int, r: int, alpha: float = 0.0, *,
                       mode: str | None = None) -> FgCallback:
    """Matrix-free objective on packed variables, evaluated on the B200."""
    n = obs.n
    if d < 2:
        raise ValueError(f"order must be >= 2, got {d}")
    ctx = obs.device_context()

    def fg(x: np.ndarray) -> tuple[float, np.ndarray]:
        x = np.asarray(x, dtype=float)
        if x.shape != (r + n * r,):
            raise ValueError(f"expected packed length {r + n * r}, got {x.shape}")
        if not np.isfinite(x).all():
            raise ValueError("model variables and alpha must be finite")
        return ctx.fg_packed(x, n, d, r, alpha, mode)

    return fg


def packed_fg_implicit_batched(obs: ObservationSet, d: int, r: int, alpha: float = 0.0, *,
                               mode: str | None = None):
    """fg over a batch of packed points X (k x (r + n r)) -> (f[k], G[k x (r + n r)]).

    The k starts share one pass over V (batched multistart); each row equals
    ``packed_fg_implicit(obs, d, r, alpha)(X[s])`` up to fp64 reassociation of the column blocks.
    """
    n = obs.n
    if d < 2:
        raise ValueError(f"order must be >= 2, got {d}")
    ctx = obs.device_context()

    def fg(X: np.ndarray):
        X = np.asarray(X, dtype=float)
        if X.ndim != 2 or X.shape[1] != r + n * r:
            raise ValueError(f"expected a (k, {r + n * r}) batch, got {X.shape}")
        if not np.isfinite(X).all():
            raise ValueError("model variables and alpha must be finite")
        return ctx.fg_batch(X, n, d, r, alpha, mode)

    return fg
