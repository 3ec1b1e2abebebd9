"""Function and gradient evaluation of the symmetric CP fit, on the B200.

``fg_implicit`` keeps the reference contract (pkg/src/momentcp/objective.py:77-94): validate
(objective.py:38-48, ValueError on bad shapes or non-finite input), evaluate, return
``FgResult(f, g_lam, g_A, eval_time, eval_kind)``.  The whole evaluation -- TTSVs, w, the
Gram tail and both gradients (implicit.py:94-107,143-151; objective.py:51-56) -- runs on the
device in one CUDA-graph replay; only lam, A go in and f, g come out.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from .dense import ObservationSet


@dataclass
class FgResult:
    """Objective value and gradients at one point (lam, A) (reference objective.py:27-35)."""

    f: float
    g_lam: np.ndarray
    g_A: np.ndarray
    eval_time: float
    eval_kind: str


def validate_variables(lam, A, n: int, alpha: float):
    """Shape and finiteness checks of reference objective.py:38-48."""
    lam = np.asarray(lam, dtype=float)
    A = np.asarray(A, dtype=float)
    if lam.ndim != 1 or A.ndim != 2:
        raise ValueError("lam must be a vector and A a matrix")
    if A.shape != (n, lam.size):
        raise ValueError(f"A must be {n} x {lam.size}, got shape {A.shape}")
    if not (np.isfinite(lam).all() and np.isfinite(A).all() and np.isfinite(alpha)):
        raise ValueError("model variables and alpha must be finite")
    return lam, A


def fg_implicit(obs: ObservationSet, lam, A, d: int, alpha: float = 0.0,
                eval_kind: str = "implicit", *, mode: str | None = None) -> FgResult:
    """f, grad_lam, grad_A from (V, nu) alone, O(p n r + n r^2), on the GPU."""
    lam, A = validate_variables(lam, A, obs.n, alpha)
    if d < 2:
        raise ValueError(f"order must be >= 2, got {d}")
    ctx = obs.device_context()
    start = time.perf_counter()
    f, g_lam, g_A = ctx.fg(lam, np.asfortranarray(A), d, float(alpha), mode)
    return FgResult(f, g_lam, np.ascontiguousarray(g_A), time.perf_counter() - start, eval_kind)
