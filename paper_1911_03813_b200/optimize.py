"""Packed-variable adapter handing the B200 f+grad to a quasi-Newton driver.

Same layout as the reference (pkg/src/momentcp/optimize.py:104-134): x = [lam; vec_F(A)],
gradient packed the same way.  ``packed_fg_implicit`` returns the ``fg(x) -> (f, g)`` closure
that ``lbfgs_minimize`` (optimize.py:255-355) and ``multistart`` (:454-508) consume; each call
is one C-ABI call (``mcp_fg_packed``): H2D of x, one CUDA-graph replay, D2H of [f; g].
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from .dense import ObservationSet

FgCallback = Callable[[np.ndarray], tuple[float, np.ndarray]]


@dataclass
class OptConfig:
    """L-BFGS settings (reference optimize.py:31-48, same defaults and checks)."""

    memory: int = 5
    pgtol: float = 1e-4
    max_iters: int = 10_000
    max_total_iters: int = 50_000
    sufficient_decrease: float = 1e-4
    curvature: float = 0.9
    max_line_steps: int = 20
    seed: int = 0

    def __post_init__(self) -> None:
        if self.pgtol <= 0:
            raise ValueError(f"pgtol must be > 0, got {self.pgtol}")
        if self.memory < 1:
            raise ValueError(f"memory must be >= 1, got {self.memory}")


@dataclass
class AdamConfig:
    """Epoch-based Adam settings (reference optimize.py:51-75, same defaults and checks)."""

    step_size: float = 0.01
    reduced_step_size: float = 0.001
    epoch_len: int = 100
    batch: int = 100
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    estimate_samples: int = 1000
    max_epochs: int = 1000

    def __post_init__(self) -> None:
        if self.epoch_len < 1:
            raise ValueError(f"epoch_len must be >= 1, got {self.epoch_len}")
        if self.batch < 1:
            raise ValueError(f"batch must be >= 1, got {self.batch}")


@dataclass
class RunReport:
    """Outcome of one optimization run (reference optimize.py:78-101)."""

    lam: np.ndarray
    A: np.ndarray
    f: float
    grad_inf_norm: float
    n_fg: int
    n_steps: int
    wall_time: float
    reason: str
    seed: int | None = None
    trace: list[tuple[float, float]] = field(default_factory=list)
    run_index: int | None = None
    runs: list["RunReport"] | None = None
    failures: list[str] = field(default_factory=list)


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

    d, r, alpha = int(d), int(r), float(alpha)
    if not np.isfinite(alpha):
        raise ValueError("model variables and alpha must be finite")

    def fg(x: np.ndarray) -> tuple[float, np.ndarray]:
        x = np.asarray(x, dtype=float)
        if x.shape != (r + n * r,):
            raise ValueError(f"expected packed length {r + n * r}, got {x.shape}")
        return ctx.fg_packed(x, n, d, r, alpha, mode)   # finiteness checked in the library

    fg.device_problem = (obs, int(d), int(r), float(alpha), mode)  # read by lbfgs_minimize
    return fg


def lbfgs_minimize(fg: FgCallback, x0: np.ndarray, cfg: OptConfig,
                   shape: tuple[int, int] | None = None,
                   iterate_hook: Callable[[np.ndarray], None] | None = None) -> RunReport:
    """L-BFGS with strong-Wolfe line search (reference optimize.py:255-355).

    When ``fg`` comes from :func:`packed_fg_implicit` the whole solve (two-loop recursion,
    trial points, (s, y) history, every f+grad) runs on the GPU through ``mcp_lbfgs`` and the
    host only steers the line search on scalars.  Any other callback (wrapped closures, custom
    objectives, the sharded / multi-GPU ``fg``) is driven by the host solver
    (:mod:`.host_solver`) with the same decisions.  Stopping rules, step logic and the report
    match the reference; ``trace`` rows are ``(f, seconds since start)``.
    """
    import time

    problem = getattr(fg, "device_problem", None)
    if problem is None:
        from .host_solver import lbfgs_host

        start = time.perf_counter()
        out = lbfgs_host(fg, x0, cfg, iterate_hook)
        x = out["x"]
        lam, A = (x.copy(), np.empty((0, 0))) if shape is None else unpack(x, *shape)
        return RunReport(lam=lam, A=A, f=out["f"], grad_inf_norm=float(np.abs(out["g"]).max()),
                         n_fg=out["n_fg"], n_steps=out["n_steps"],
                         wall_time=time.perf_counter() - start, reason=out["reason"],
                         seed=cfg.seed, trace=out["trace"])
    obs, d, r, alpha, mode = problem
    start = time.perf_counter()
    x0 = np.asarray(x0, dtype=float)
    if x0.shape != (r + obs.n * r,):
        raise ValueError(f"expected packed length {r + obs.n * r}, got {x0.shape}")
    if not np.isfinite(x0).all():
        raise ValueError("model variables and alpha must be finite")
    ctx = obs.device_context()
    opts = (cfg.memory, cfg.pgtol, cfg.max_iters, cfg.max_total_iters, cfg.sufficient_decrease,
            cfg.curvature, cfg.max_line_steps)
    out = ctx.lbfgs(x0, obs.n, d, r, alpha, mode, opts, iterate_hook)
    x = out["x"]
    if shape is None:
        lam, A = x.copy(), np.empty((0, 0))
    else:
        lam, A = unpack(x, *shape)
    return RunReport(lam=lam, A=A, f=out["f"], grad_inf_norm=float(np.abs(out["g"]).max()),
                     n_fg=out["n_fg"], n_steps=out["n_steps"],
                     wall_time=time.perf_counter() - start, reason=out["reason"], seed=cfg.seed,
                     trace=out["trace"])


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


def adam_minimize(obs: ObservationSet, d: int, r_hat: int, x0: np.ndarray, cfg: AdamConfig,
                  rng: np.random.Generator, *, mode: str | None = None) -> RunReport:
    """Stochastic minimization with epoch-based Adam, device-resident (optimize.py:365-451).

    Same draws from ``rng`` in the same order as the reference (the estimate subset, then
    ``rng.integers(0, p, size=batch)`` per inner iteration); mini-batches are gathered from the
    resident observations and the Adam state never leaves the GPU (``mcp_adam``).
    """
    import time

    start = time.perf_counter()
    n, p = obs.n, obs.p
    if not obs.has_uniform_weights():
        raise ValueError("stochastic optimization requires uniform weights")
    x = np.asarray(x0, dtype=float).copy()
    if x.shape != (r_hat + n * r_hat,):
        raise ValueError(f"x0 has length {x.size}, expected {r_hat + n * r_hat}")
    if d < 2:
        raise ValueError(f"order must be >= 2, got {d}")
    if not np.isfinite(x).all():
        raise ValueError("model variables and alpha must be finite")
    est_idx = rng.choice(p, size=min(cfg.estimate_samples, p), replace=False)

    before_last_draw: list[dict] = []

    def sample(count: int) -> np.ndarray:
        # the library draws the next epoch while the GPU runs the current one; if the run then
        # stops, that epoch was never needed and the generator is rewound below
        before_last_draw[:] = [rng.bit_generator.state]
        out = np.empty(count, dtype=np.int64)
        for k in range(count // cfg.batch):
            out[k * cfg.batch:(k + 1) * cfg.batch] = rng.integers(0, p, size=cfg.batch)
        return out

    ctx = obs.device_context()
    opts = (cfg.step_size, cfg.reduced_step_size, cfg.epoch_len, cfg.batch, cfg.beta1,
            cfg.beta2, cfg.eps, cfg.max_epochs)
    out = ctx.adam(x, n, d, r_hat, mode, opts, est_idx, sample)
    if out["unused_draws"] and before_last_draw:
        rng.bit_generator.state = before_last_draw[0]   # leave rng where the reference leaves it
    lam, A = unpack(out["x"], n, r_hat)
    return RunReport(lam=lam, A=A, f=out["f"], grad_inf_norm=float(np.abs(out["g"]).max()),
                     n_fg=out["n_iter"], n_steps=out["n_iter"],
                     wall_time=time.perf_counter() - start, reason=out["reason"],
                     trace=out["trace"])


def lbfgs_minimize_batched(fg: FgCallback, X0, cfg: OptConfig,
                           shape: tuple[int, int] | None = None) -> list[RunReport | Exception]:
    """k L-BFGS solves in lock step on the device.

    Row s of ``X0`` is start s.  Each round evaluates one trial point per unfinished run, all of
    them in ONE pass over V (k r factor columns), so k starts cost about one start's latency per
    round.  Every run takes the reference's decisions (optimize.py:255-355) on its own scalars;
    its result equals ``lbfgs_minimize(fg, X0[s], cfg)`` up to the fp64 reassociation of the
    shared pass.  Runs that fail (non-finite start) come back as ValueError instances.
    """
    import time

    problem = getattr(fg, "device_problem", None)
    if problem is None:
        raise TypeError("lbfgs_minimize_batched runs on the device: pass the fg returned by "
                        "packed_fg_implicit(obs, d, r, alpha)")
    obs, d, r, alpha, mode = problem
    X0 = np.asarray(X0, dtype=float)
    if X0.ndim != 2 or X0.shape[1] != r + obs.n * r:
        raise ValueError(f"expected a (k, {r + obs.n * r}) batch of starts, got {X0.shape}")
    start = time.perf_counter()
    opts = (cfg.memory, cfg.pgtol, cfg.max_iters, cfg.max_total_iters, cfg.sufficient_decrease,
            cfg.curvature, cfg.max_line_steps)
    outs = obs.device_context().lbfgs_batch(X0, obs.n, d, r, alpha, mode, opts)
    wall = time.perf_counter() - start
    reports: list[RunReport | Exception] = []
    for out in outs:
        if out["reason"] == "error":
            reports.append(ValueError(out["error"]))
            continue
        x = out["x"]
        lam, A = (x.copy(), np.empty((0, 0))) if shape is None else unpack(x, *shape)
        reports.append(RunReport(lam=lam, A=A, f=out["f"],
                                 grad_inf_norm=float(np.abs(out["g"]).max()), n_fg=out["n_fg"],
                                 n_steps=out["n_steps"], wall_time=wall, reason=out["reason"],
                                 seed=cfg.seed, trace=out["trace"]))
    return reports


def multistart_lbfgs(k: int, init: Callable[[np.random.Generator], np.ndarray],
                     fg: FgCallback, cfg: OptConfig, seed: int,
                     shape: tuple[int, int] | None = None) -> RunReport:
    """multistart (optimize.py:454-508) of device L-BFGS runs, all k in lock step.

    Seeding and selection are the reference's: start i is ``init(default_rng(SeedSequence(seed)
    .spawn(k)[i]))``; the lowest final f wins (ties by run index); failures are collected and an
    all-failed batch raises RuntimeError.
    """
    if k < 1:
        raise ValueError(f"number of starts must be >= 1, got {k}")
    root = seed if isinstance(seed, np.random.SeedSequence) else np.random.SeedSequence(seed)
    children = root.spawn(k)
    X0 = np.stack([np.asarray(init(np.random.default_rng(children[i])), dtype=float)
                   for i in range(k)])
    reports = lbfgs_minimize_batched(fg, X0, cfg, shape)
    successes, errors = [], []
    for i, rep in enumerate(reports):
        if isinstance(rep, Exception):
            errors.append(f"run {i}: {rep}")
        else:
            rep.run_index = i
            successes.append(rep)
    if not successes:
        raise RuntimeError("all multistart runs failed: " + "; ".join(errors))
    best = min(successes, key=lambda rp: (rp.f, rp.run_index))
    best.runs = successes
    best.failures = errors
    best.seed = seed if isinstance(seed, int) else None
    return best
