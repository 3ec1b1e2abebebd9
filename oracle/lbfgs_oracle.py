"""L-BFGS driver restated for trajectory (replay) parity -- TEST INFRASTRUCTURE ONLY.

A restatement of the reference solver, pkg/src/momentcp/optimize.py:149-355 (two-loop
recursion :149-168, safeguarded quadratic interpolation :171-176, strong-Wolfe bracket/zoom
line search :179-252, outer loop :255-345), written to take the same decisions in the same
order so that, driven by the same ``fg``, it reproduces the reference's iterates bitwise
(pinned by tests/golden/lbfgs_c1.npz).  The product never imports this; tests use it to drive
the GPU ``packed_fg_implicit`` and the CPU oracle side by side (SURVEY.md section 8c replay
protocol).
"""

from __future__ import annotations

from collections import deque

import numpy as np


def two_loop(g, S, Yh, gamma):
    """-H g for the L-BFGS inverse Hessian on gamma*I (optimize.py:149-168)."""
    q = g.copy()
    m = len(S)
    rho = [1.0 / float(Yh[i] @ S[i]) for i in range(m)]
    alpha = [0.0] * m
    for i in range(m - 1, -1, -1):
        alpha[i] = rho[i] * float(S[i] @ q)
        q -= alpha[i] * Yh[i]
    q *= gamma
    for i in range(m):
        beta = rho[i] * float(Yh[i] @ q)
        q += (alpha[i] - beta) * S[i]
    return -q


def _interp(a_lo, f_lo, d_lo, a_hi, f_hi):
    den = f_hi - f_lo - d_lo * (a_hi - a_lo)
    if den == 0 or not np.isfinite(den):
        return None
    c = a_lo - 0.5 * d_lo * (a_hi - a_lo) ** 2 / den
    return c if np.isfinite(c) else None


def wolfe(fg, x, f0, g0, p, a0, c1, c2, budget):
    """Strong-Wolfe search (optimize.py:179-252); returns (x, f, g, evals) or (None, ...)."""
    slope0 = float(g0 @ p)
    state = {"evals": 0, "best": None}

    def probe(a):
        xa = x + a * p
        fa, ga = fg(xa)
        state["evals"] += 1
        if np.isfinite(fa) and fa <= f0 + c1 * a * slope0:
            b = state["best"]
            if b is None or fa < b[1]:
                state["best"] = (a, fa, ga, xa)
        return fa, ga, xa

    def fallback():
        b = state["best"]
        if b is not None:
            return b[3], b[1], b[2], state["evals"]
        return None, f0, g0, state["evals"]

    prev = (0.0, f0, slope0)
    a = a0
    lo = hi = None
    for _ in range(budget):
        fa, ga, xa = probe(a)
        da = float(ga @ p) if np.isfinite(fa) else np.nan
        bad = (not np.isfinite(fa)) or fa > f0 + c1 * a * slope0 or (prev[0] > 0.0 and fa >= prev[1])
        if bad:
            lo, hi = prev, (a, fa, da)
            break
        if abs(da) <= -c2 * slope0:
            return xa, fa, ga, state["evals"]
        if da >= 0.0:
            lo, hi = (a, fa, da), prev
            break
        prev = (a, fa, da)
        a = min(2.0 * a, 1e20)
    if lo is None:
        return fallback()

    while state["evals"] < budget:
        a_lo, f_lo, d_lo = lo
        a_hi, f_hi = hi[0], hi[1]
        width = a_hi - a_lo
        cand = _interp(a_lo, f_lo, d_lo, a_hi, f_hi) if np.isfinite(f_hi) else None
        lb, ub = a_lo + 0.1 * width, a_hi - 0.1 * width
        if cand is None or not (min(lb, ub) <= cand <= max(lb, ub)):
            cand = a_lo + 0.5 * width
        fa, ga, xa = probe(cand)
        da = float(ga @ p) if np.isfinite(fa) else np.nan
        if (not np.isfinite(fa)) or fa > f0 + c1 * cand * slope0 or fa >= f_lo:
            hi = (cand, fa, da)
        else:
            if abs(da) <= -c2 * slope0:
                return xa, fa, ga, state["evals"]
            if da * (a_hi - a_lo) >= 0.0:
                hi = lo
            lo = (cand, fa, da)
        if abs(hi[0] - lo[0]) < 1e-16 * max(1.0, abs(lo[0])):
            break
    return fallback()


def lbfgs(fg, x0, *, memory=5, pgtol=1e-4, max_iters=10_000, max_total_iters=50_000,
          c1=1e-4, c2=0.9, max_line_steps=20, iterate_hook=None):
    """Outer L-BFGS loop (optimize.py:255-345); returns a dict like RunReport."""
    x = np.asarray(x0, dtype=float).copy()
    f, g = fg(x)
    n_fg = 1
    if not (np.isfinite(f) and np.isfinite(g).all()):
        raise ValueError("objective is not finite at the starting point")
    trace = [f]
    if iterate_hook is not None:
        iterate_hook(x.copy())
    S: deque = deque(maxlen=memory)
    Yh: deque = deque(maxlen=memory)
    steps = 0
    reason = "iteration cap"
    while True:
        if float(np.abs(g).max()) <= pgtol:
            reason = "tolerance"
            break
        if steps >= max_iters or n_fg >= max_total_iters:
            reason = "iteration cap"
            break
        if S:
            gamma = float(S[-1] @ Yh[-1]) / float(Yh[-1] @ Yh[-1])
            p = two_loop(g, list(S), list(Yh), gamma)
            a0 = 1.0
        else:
            p = -g
            a0 = min(1.0, 1.0 / max(float(np.abs(g).sum()), 1e-12))
        if float(p @ g) >= 0.0:
            S.clear()
            Yh.clear()
            p = -g
            a0 = min(1.0, 1.0 / max(float(np.abs(g).sum()), 1e-12))
        budget = min(max_line_steps, max_total_iters - n_fg)
        xn, fn, gn, ev = wolfe(fg, x, f, g, p, a0, c1, c2, budget)
        n_fg += ev
        if xn is None:
            reason = "iteration cap" if n_fg >= max_total_iters else "line-search failure"
            break
        s = xn - x
        y = gn - g
        if float(s @ y) > 1e-12 * float(np.linalg.norm(s)) * float(np.linalg.norm(y)):
            S.append(s)
            Yh.append(y)
        x, f, g = xn, fn, gn
        steps += 1
        trace.append(f)
        if iterate_hook is not None:
            iterate_hook(x.copy())
    return {"x": x, "f": f, "g": g, "n_fg": n_fg, "n_steps": steps, "reason": reason,
            "trace": trace, "grad_inf_norm": float(np.abs(g).max())}
