"""CPU oracle for the implicit moment-tensor CP f+grad path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference ``momentcp`` arithmetic on
the hot path.  It exists to check the B200 product path, never to be it:
only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import it.  The product package
(``paper_1911_03813_b200``) never imports anything under ``oracle/``.

Parity pin: every function here is checked against golden vectors produced by
the *unmodified* reference package (``tests/golden/make_golden.py`` imports it
from ``/root/reference/pkg/src`` in the build container and commits the
vectors as ``tests/golden/*.npz``); ``tests/test_oracle_golden.py`` asserts the
restatement reproduces them (bitwise where the same numpy calls are made,
1e-13 term-scale otherwise).

Reference locations (paths relative to the reference root):

* repeated-multiplication power ....... pkg/src/momentcp/implicit.py:82-91
* batched TTSV  Y = V diag(nu) (V^T A)^(d-1) .. pkg/src/momentcp/implicit.py:94-107
* model norm    lam^T (A^T A)^d lam ... pkg/src/momentcp/implicit.py:110-113
* data norm     nu^T (V^T V)^d nu ..... pkg/src/momentcp/implicit.py:116-121
* w_j = a_j^T y_j ..................... pkg/src/momentcp/implicit.py:124-140
* Gram cache G, C, u, w ............... pkg/src/momentcp/implicit.py:143-151
* f / g_lam / g_A tail ................ pkg/src/momentcp/objective.py:51-56
* argument validation ................. pkg/src/momentcp/objective.py:38-48
* pack / unpack ....................... pkg/src/momentcp/optimize.py:104-120
* term-scale tolerance metric ......... pkg/tests/test_acceptance.py:5-11,65-74

Arrays follow the reference's conventions: ``V`` is n x p (column l is
observation v_l), ``nu`` has length p, ``A`` is n x r, ``lam`` has length r.
"""

from __future__ import annotations

import numpy as np


def rm_power(M: np.ndarray, k: int) -> np.ndarray:
    """Elementwise M**k as a left-to-right product M*M*...*M (implicit.py:82-91).

    k == 0 gives ones; the first factor is a copy, then k-1 in-place multiplies,
    so the rounding sequence is ((M*M)*M)*... exactly as the reference forms it.
    """
    if k < 0:
        raise ValueError(f"power must be >= 0, got {k}")
    if k == 0:
        return np.ones_like(M)
    acc = np.array(M, copy=True)
    for _ in range(1, k):
        np.multiply(acc, M, out=acc)
    return acc


def _check_order(d: int) -> None:
    if d < 2:
        raise ValueError(f"order must be >= 2, got {d}")


def ttsv_batch(V: np.ndarray, nu: np.ndarray, A: np.ndarray, d: int) -> np.ndarray:
    """All-but-one TTSVs of the weighted moment tensor (implicit.py:94-107)."""
    _check_order(d)
    A = np.asarray(A, dtype=float)
    if A.ndim != 2 or A.shape[0] != V.shape[0]:
        raise ValueError(f"A must be {V.shape[0]} x r, got shape {A.shape}")
    Z = V.T @ A                       # p x r projections
    scaled = nu[:, None] * rm_power(Z, d - 1)
    return V @ scaled


def kruskal_norm_sq(lam: np.ndarray, A: np.ndarray, d: int) -> float:
    """||M||^2 = lam^T (A^T A)^d lam (implicit.py:110-113)."""
    return float(lam @ rm_power(A.T @ A, d) @ lam)


def data_norm_sq(V: np.ndarray, nu: np.ndarray, d: int) -> float:
    """||X||^2 = nu^T (V^T V)^d nu with the full p x p Gram (implicit.py:116-121)."""
    _check_order(d)
    return float(nu @ rm_power(V.T @ V, d) @ nu)


def data_norm_sq_blocked(V: np.ndarray, nu: np.ndarray, d: int, block: int = 4096) -> float:
    """Blocked restatement of implicit.py:116-121 for p too large for a p x p Gram.

    Sums nu_I^T (V_I^T V_J)^d nu_J over all block pairs (I, J) in row-major
    block order.  Mathematically identical to :func:`data_norm_sq`; rounding
    differs only by the reassociation of the final two dot products.
    """
    _check_order(d)
    p = V.shape[1]
    total = 0.0
    for i0 in range(0, p, block):
        Vi = V[:, i0:i0 + block]
        ni = nu[i0:i0 + block]
        acc = 0.0
        for j0 in range(0, p, block):
            G = rm_power(Vi.T @ V[:, j0:j0 + block], d)
            acc += float(ni @ (G @ nu[j0:j0 + block]))
        total += acc
    return total


def gram_tail(lam: np.ndarray, A: np.ndarray, d: int, Y: np.ndarray):
    """(G, C, u, w) of one evaluation (implicit.py:143-151, w from :124-140)."""
    G = A.T @ A
    C = rm_power(G, d - 1)
    u = (G * C) @ lam
    w = np.einsum("ij,ij->j", A, Y)
    return G, C, u, w


def finish(Y: np.ndarray, lam: np.ndarray, A: np.ndarray, d: int, alpha: float):
    """f, g_lam, g_A from the TTSV matrix Y (objective.py:51-56)."""
    _, C, u, w = gram_tail(lam, A, d, Y)
    f = alpha + float(lam @ u) - 2.0 * float(w @ lam)
    g_lam = -2.0 * (w - u)
    g_A = -2.0 * d * (Y - (A * lam) @ C) * lam
    return f, g_lam, g_A


def validate(lam, A, n: int, alpha: float):
    """Shape/finiteness checks of objective.py:38-48 (ValueError on failure)."""
    lam = np.asarray(lam, dtype=float)
    A = np.asarray(A, dtype=float)
    if lam.ndim != 1 or A.ndim != 2:
        raise ValueError("lam must be a vector and A a matrix")
    if A.shape != (n, lam.size):
        raise ValueError(f"A must be {n} x {lam.size}, got shape {A.shape}")
    if not (np.isfinite(lam).all() and np.isfinite(A).all() and np.isfinite(alpha)):
        raise ValueError("model variables and alpha must be finite")
    return lam, A


def fg_implicit(V, nu, lam, A, d: int, alpha: float = 0.0):
    """(f, g_lam, g_A) of the implicit route (objective.py:77-94)."""
    lam, A = validate(lam, A, V.shape[0], alpha)
    Y = ttsv_batch(V, nu, A, d)
    return finish(Y, lam, A, d, alpha)


def fg_partial(V, nu, A, d: int):
    """Per-shard additive pieces [Y | w] of one evaluation.

    ``Y`` and ``w = sum_l nu_l z_l^d`` are sums over observations, so row
    shards of V contribute additively; summing shard partials and running
    :func:`finish_from_partial` once is exact math.
    Used as the CPU stand-in for the per-rank CUDA partial in the gloo tests.
    """
    _check_order(d)
    Z = V.T @ A
    P = nu[:, None] * rm_power(Z, d - 1)
    Y = V @ P
    w = np.einsum("lj,lj->j", P, Z)
    return Y, w


def finish_from_partial(Y, w, lam, A, d: int, alpha: float):
    """Tail driven by an externally reduced w (same algebra as objective.py:51-56)."""
    G = A.T @ A
    C = rm_power(G, d - 1)
    u = (G * C) @ lam
    f = alpha + float(lam @ u) - 2.0 * float(w @ lam)
    g_lam = -2.0 * (w - u)
    g_A = -2.0 * d * (Y - (A * lam) @ C) * lam
    return f, g_lam, g_A


def pack(lam, A) -> np.ndarray:
    """x = [lam; vec_F(A)] (optimize.py:104-110)."""
    lam = np.asarray(lam, dtype=float)
    A = np.asarray(A, dtype=float)
    return np.concatenate([lam, A.reshape(-1, order="F")])


def unpack(x, n: int, r: int):
    """Inverse of :func:`pack` (optimize.py:113-120); returns fresh copies."""
    x = np.asarray(x, dtype=float)
    if x.shape != (r + n * r,):
        raise ValueError(f"expected packed length {r + n * r}, got {x.shape}")
    return x[:r].copy(), x[r:].reshape((n, r), order="F").copy()


def packed_fg(V, nu, d: int, r: int, alpha: float = 0.0):
    """Packed-variable callback (optimize.py:123-134)."""
    n = V.shape[0]

    def fg(x):
        lam, A = unpack(x, n, r)
        f, gl, gA = fg_implicit(V, nu, lam, A, d, alpha)
        return f, pack(gl, gA)

    return fg


def term_scales(V, nu, lam, A, d: int, alpha: float):
    """Accumulated-term magnitudes (test_acceptance.py:65-74): the kernel on |inputs|."""
    Va, la, Aa = np.abs(V), np.abs(lam), np.abs(A)
    Ya = ttsv_batch(Va, nu, Aa, d)
    _, C, u, w = gram_tail(la, Aa, d, Ya)
    f_s = abs(alpha) + float(la @ u) + 2.0 * float(w @ la)
    gl_s = 2.0 * (w + u)
    gA_s = 2.0 * d * (Ya + (Aa * la) @ C) * la
    return f_s, gl_s, gA_s, Ya


def term_rel_err(got, want, scale) -> float:
    """max |got - want| / (scale + |want|): the reference's term-scale metric."""
    got = np.asarray(got, dtype=float)
    want = np.asarray(want, dtype=float)
    return float(np.max(np.abs(got - want) / (np.asarray(scale) + np.abs(want) + 1e-300)))


# --- dense (explicit) route for desk-scale cross-checks --------------------------------


def dense_moment(V: np.ndarray, nu: np.ndarray, d: int) -> np.ndarray:
    """X = sum_l nu_l v_l^{(x) d} as a full n^d array (tiny n only)."""
    n, p = V.shape
    X = np.zeros((n,) * d)
    for l in range(p):
        t = V[:, l]
        for _ in range(d - 1):
            t = np.multiply.outer(t, V[:, l])
        X += nu[l] * t
    return X


def dense_ttsv(X: np.ndarray, a: np.ndarray) -> np.ndarray:
    """Contract X with a in all modes but the first."""
    out = X
    for _ in range(X.ndim - 1):
        out = out @ a
    return out
