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


def sample_observations(obs: ObservationSet, s: int, rng: np.random.Generator) -> ObservationSet:
    """Draw ``s`` observations uniformly with replacement, weights 1/s (objective.py:97-113).

    Same draws as the reference (``rng.integers(0, p, size=s)``); the rows are gathered on the
    device from the resident set (``mcp_gather_rows``), so the sample never visits the host.
    """
    import torch

    from . import _native

    if s < 1:
        raise ValueError(f"sample size must be >= 1, got {s}")
    if not obs.has_uniform_weights():
        raise ValueError("sampling requires uniform observation weights")
    idx = rng.integers(0, obs.p, size=s)
    labels = obs.labels[idx] if obs.labels is not None else None
    ctx = obs.device_context()
    dt = torch.float32 if ctx.dtype_code == _native.MCP_F32 else torch.float64
    rows = torch.empty((s, obs.n), dtype=dt, device=f"cuda:{ctx.device}")
    ctx.gather_rows(idx, rows.data_ptr(), obs.n, ctx.dtype_code)
    return ObservationSet.from_device(rows, labels=labels)
