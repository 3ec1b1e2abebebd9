"""Host-side L-BFGS for arbitrary ``fg(x) -> (f, g)`` callbacks.

``lbfgs_minimize`` runs the whole solve on the device when ``fg`` comes from
``packed_fg_implicit`` (csrc/lbfgs.cu).  Any other callback -- a wrapped closure, a custom
objective, the row-sharded ``packed_fg_sharded``, the single-process multi-GPU
``MultiDeviceObservationSet.packed_fg`` -- is driven from here instead, so the drop-in accepts
everything the reference's ``lbfgs_minimize`` accepts (pkg/src/momentcp/optimize.py:255-355).

The decisions follow the reference in the same order with the same floating-point expressions
(two-loop recursion optimize.py:149-168, safeguarded quadratic interpolation :171-176,
strong-Wolfe bracket + zoom :179-252, outer loop :255-345), so the same ``fg`` yields the same
iterates.  The code is organised as a line-search object whose state (the bracket, the best
sufficient-decrease point, the evaluation count) is explicit, rather than nested closures.
"""

from __future__ import annotations

import time
from collections import deque
from dataclasses import dataclass

import numpy as np


def two_loop_direction(g, s_list, y_list, gamma):
    """-H g for the inverse-Hessian model of the stored (s, y) pairs on gamma I
    (reference optimize.py:149-168: newest pair first, then oldest first)."""
    q = g.copy()
    m = len(s_list)
    rho = [1.0 / float(y_list[i] @ s_list[i]) for i in range(m)]
    coef = [0.0] * m
    for i in reversed(range(m)):
        coef[i] = rho[i] * float(s_list[i] @ q)
        q -= coef[i] * y_list[i]
    q *= gamma
    for i in range(m):
        q += (coef[i] - rho[i] * float(y_list[i] @ q)) * s_list[i]
    return -q


def _safeguarded_quadratic(a_lo, f_lo, d_lo, a_hi, f_hi):
    """Minimiser of the quadratic through (a_lo, f_lo, slope d_lo) and (a_hi, f_hi), or None
    (reference optimize.py:171-176)."""
    den = f_hi - f_lo - d_lo * (a_hi - a_lo)
    if den == 0 or not np.isfinite(den):
        return None
    a = a_lo - 0.5 * d_lo * (a_hi - a_lo) ** 2 / den
    return a if np.isfinite(a) else None


@dataclass
class _Point:
    a: float
    f: float
    slope: float


class _StrongWolfe:
    """One strong-Wolfe line search along ``p`` from ``x`` (reference optimize.py:179-252)."""

    def __init__(self, fg, x, f0, g0, p, c1, c2, budget):
        self.fg, self.x, self.f0, self.g0, self.p = fg, x, f0, g0, p
        self.c1, self.c2, self.budget = c1, c2, budget
        self.slope0 = float(g0 @ p)
        self.evals = 0
        self.best = None          # (a, f, g, x) with the lowest f meeting sufficient decrease

    def _probe(self, a):
        xa = self.x + a * self.p
        fa, ga = self.fg(xa)
        self.evals += 1
        if np.isfinite(fa) and fa <= self.f0 + self.c1 * a * self.slope0:
            if self.best is None or fa < self.best[1]:
                self.best = (a, fa, ga, xa)
        slope = float(ga @ self.p) if np.isfinite(fa) else np.nan
        return fa, ga, xa, slope

    def _curvature_ok(self, slope):
        return abs(slope) <= -self.c2 * self.slope0

    def _fallback(self):
        if self.best is not None:
            return self.best[3], self.best[1], self.best[2]
        return None, self.f0, self.g0

    def run(self, a0):
        prev = _Point(0.0, self.f0, self.slope0)
        a = a0
        lo = hi = None
        for _ in range(self.budget):                      # bracketing phase
            fa, ga, xa, slope = self._probe(a)
            if (not np.isfinite(fa) or fa > self.f0 + self.c1 * a * self.slope0
                    or (prev.a > 0.0 and fa >= prev.f)):
                lo, hi = prev, _Point(a, fa, slope)
                break
            if self._curvature_ok(slope):
                return xa, fa, ga
            if slope >= 0.0:
                lo, hi = _Point(a, fa, slope), prev
                break
            prev = _Point(a, fa, slope)
            a = min(2.0 * a, 1e20)
        if lo is None:
            return self._fallback()
        while self.evals < self.budget:                   # zoom phase
            width = hi.a - lo.a
            cand = (_safeguarded_quadratic(lo.a, lo.f, lo.slope, hi.a, hi.f)
                    if np.isfinite(hi.f) else None)
            b0, b1 = lo.a + 0.1 * width, hi.a - 0.1 * width
            if cand is None or not (min(b0, b1) <= cand <= max(b0, b1)):
                cand = lo.a + 0.5 * width
            fa, ga, xa, slope = self._probe(cand)
            if not np.isfinite(fa) or fa > self.f0 + self.c1 * cand * self.slope0 or fa >= lo.f:
                hi = _Point(cand, fa, slope)
            else:
                if self._curvature_ok(slope):
                    return xa, fa, ga
                if slope * (hi.a - lo.a) >= 0.0:
                    hi = lo
                lo = _Point(cand, fa, slope)
            if abs(hi.a - lo.a) < 1e-16 * max(1.0, abs(lo.a)):
                break
        return self._fallback()


def _steepest_step(g):
    return min(1.0, 1.0 / max(float(np.abs(g).sum()), 1e-12))


def lbfgs_host(fg, x0, cfg, iterate_hook=None):
    """The reference outer loop (optimize.py:255-345) on the host; returns a dict like the
    device solver's: x, g, f, n_fg, n_steps, reason, trace."""
    start = time.perf_counter()
    x = np.asarray(x0, dtype=float).copy()
    f, g = fg(x)
    n_fg = 1
    if not (np.isfinite(f) and np.isfinite(g).all()):
        raise ValueError("objective is not finite at the starting point")
    trace = [(f, time.perf_counter() - start)]
    if iterate_hook is not None:
        iterate_hook(x.copy())
    S: deque = deque(maxlen=cfg.memory)
    Yh: deque = deque(maxlen=cfg.memory)
    n_steps = 0
    while True:
        if float(np.abs(g).max()) <= cfg.pgtol:
            reason = "tolerance"
            break
        if n_steps >= cfg.max_iters or n_fg >= cfg.max_total_iters:
            reason = "iteration cap"
            break
        if S:
            gamma = float(S[-1] @ Yh[-1]) / float(Yh[-1] @ Yh[-1])
            p, a0 = two_loop_direction(g, list(S), list(Yh), gamma), 1.0
        else:
            p, a0 = -g, _steepest_step(g)
        if float(p @ g) >= 0.0:          # rounding gave a non-descent direction: restart
            S.clear()
            Yh.clear()
            p, a0 = -g, _steepest_step(g)
        search = _StrongWolfe(fg, x, f, g, p, cfg.sufficient_decrease, cfg.curvature,
                              min(cfg.max_line_steps, cfg.max_total_iters - n_fg))
        x_new, f_new, g_new = search.run(a0)
        n_fg += search.evals
        if x_new is None:
            reason = "iteration cap" if n_fg >= cfg.max_total_iters else "line-search failure"
            break
        s, y = x_new - x, g_new - g
        if float(s @ y) > 1e-12 * float(np.linalg.norm(s)) * float(np.linalg.norm(y)):
            S.append(s)
            Yh.append(y)
        x, f, g = x_new, f_new, g_new
        n_steps += 1
        trace.append((f, time.perf_counter() - start))
        if iterate_hook is not None:
            iterate_hook(x.copy())
    return {"x": x, "g": g, "f": f, "n_fg": n_fg, "n_steps": n_steps, "reason": reason,
            "trace": trace}
