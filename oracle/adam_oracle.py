"""Stochastic path restated for parity -- TEST INFRASTRUCTURE ONLY.

Restates the reference's row sampling (pkg/src/momentcp/objective.py:97-113) and epoch-based
Adam (pkg/src/momentcp/optimize.py:365-451) on top of the CPU oracle f+grad, drawing from the
generator in the same order, so that with the same seed it reproduces the reference run
bitwise (pinned by tests/golden/adam_c1.npz).  ``grad_fn`` lets tests swap the f+grad used for
the mini-batches (e.g. the GPU one) while keeping every other decision identical.  The product
never imports this module.
"""

from __future__ import annotations

import numpy as np

from . import momentcp_oracle as om


def sample_rows(p: int, s: int, rng: np.random.Generator) -> np.ndarray:
    """The indices sample_observations draws (objective.py:109)."""
    return rng.integers(0, p, size=s)


def _fg_uniform(Vs, lam, A, d):
    return om.fg_implicit(Vs, np.full(Vs.shape[1], 1.0 / Vs.shape[1]), lam, A, d, 0.0)


def adam(V, d: int, r: int, x0, rng: np.random.Generator, *, step_size=0.01,
         reduced_step_size=0.001, epoch_len=100, batch=100, beta1=0.9, beta2=0.999, eps=1e-8,
         estimate_samples=1000, max_epochs=1000, fg_fn=_fg_uniform):
    """Returns dict(x_best, f, grad_inf, n_iter, reason, trace_f).

    ``fg_fn(V_subset, lam, A, d) -> (f, g_lam, g_A)`` evaluates a uniformly weighted subset
    (default: the CPU oracle)."""
    n, p = V.shape
    x = np.asarray(x0, dtype=float).copy()
    est_idx = rng.choice(p, size=min(estimate_samples, p), replace=False)
    Ve = V[:, est_idx]

    def estimate(xv):
        lam, A = om.unpack(xv, n, r)
        f, gl, gA = fg_fn(Ve, lam, A, d)
        return f, om.pack(gl, gA)

    f_best, _ = estimate(x)
    x_best = x.copy()
    trace = [f_best]
    lr = step_size
    m1 = np.zeros_like(x)
    m2 = np.zeros_like(x)
    t = 0
    n_iter = 0
    increases = 0
    reason = "iteration cap"
    for _ in range(max_epochs):
        for _ in range(epoch_len):
            idx = sample_rows(p, batch, rng)
            lam, A = om.unpack(x, n, r)
            _, gl, gA = fg_fn(V[:, idx], lam, A, d)
            grad = om.pack(gl, gA)
            t += 1
            m1 = beta1 * m1 + (1.0 - beta1) * grad
            m2 = beta2 * m2 + (1.0 - beta2) * grad * grad
            m1_hat = m1 / (1.0 - beta1**t)
            m2_hat = m2 / (1.0 - beta2**t)
            x = x - lr * m1_hat / (np.sqrt(m2_hat) + eps)
            n_iter += 1
        f_est, _ = estimate(x)
        trace.append(f_est)
        if f_est < f_best:
            f_best = f_est
            x_best = x.copy()
        else:
            increases += 1
            x = x_best.copy()
            m1[:] = 0.0
            m2[:] = 0.0
            t = 0
            if increases == 1:
                lr = reduced_step_size
            else:
                reason = "learning-rate exhausted"
                break
    _, g_final = estimate(x_best)
    return {"x": x_best, "f": f_best, "grad_inf": float(np.abs(g_final).max()),
            "n_iter": n_iter, "reason": reason, "trace_f": trace}
