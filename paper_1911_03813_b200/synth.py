"""Seeded synthetic workloads for the BASELINE configurations (BASELINE.json ``configs``).

The reference measures on synthetic data only (uniform(0,1) and Gaussian mixtures; PAPER.md
experiments, pkg/src/momentcp/gmm.py:91-111); these generators produce mixtures with the
configs' shapes, value distributions and initialisations:

  c1  n=20   p=1e4   d=3 r=5    f64  5 unit-norm means, sigma 0.1, uniform mixture
  c2  n=100  p=1e6   d=4 r=10   f64  10 unit-norm means, sigma 0.1, uniform mixture
  c3  n=512  p=4e6   d=6 r=64   f32  64 means N(0,I)/sqrt(n), sigma 0.05, Dirichlet(1) weights
  c4  n=256  p=2e5   d=4        f64  V ~ N(0,1)/sqrt(n)            (||X||^2 only)
  c5  n=1024 p=1.6e7 d=3 r=256  f32  256 unit-norm means, sigma 0.1, uniform mixture

Host generation (numpy ``default_rng``) is bit-reproducible and is what the parity fixtures use;
device generation (torch Philox on the GPU) is used for the full-size benchmark data, which
is too large to synthesise on the host in reasonable time (c5 is 65.5 GB of float32).
Initial point: lam0 = 1/r, A0 ~ N(0,1) with unit-norm columns (gmm.py:141-149 gaussian_init).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    p: int
    d: int
    r: int
    dtype: str          # "f64" | "f32"
    sigma: float
    k: int              # mixture components (0: plain Gaussian V)
    means: str          # "unit" | "scaled"
    weights: str        # "uniform" | "dirichlet"


CONFIGS = {
    "c1": Config("c1", 20, 10_000, 3, 5, "f64", 0.1, 5, "unit", "uniform"),
    "c2": Config("c2", 100, 1_000_000, 4, 10, "f64", 0.1, 10, "unit", "uniform"),
    "c3": Config("c3", 512, 4_000_000, 6, 64, "f32", 0.05, 64, "scaled", "dirichlet"),
    "c4": Config("c4", 256, 200_000, 4, 0, "f64", 1.0, 0, "none", "none"),
    "c5": Config("c5", 1024, 16_000_000, 3, 256, "f32", 0.1, 256, "unit", "uniform"),
    # the paper's stochastic example (Table 2): Adam with s = 10/100/1000
    "t2": Config("t2", 500, 500_000, 3, 10, "f64", 0.1, 10, "unit", "uniform"),
}


def _means(cfg: Config, rng: np.random.Generator) -> np.ndarray:
    mu = rng.standard_normal((cfg.n, cfg.k))
    if cfg.means == "unit":
        mu /= np.linalg.norm(mu, axis=0)
    else:
        mu /= np.sqrt(cfg.n)
    return mu


def _counts(cfg: Config, p: int, rng: np.random.Generator) -> np.ndarray:
    if cfg.weights == "uniform":
        counts = np.full(cfg.k, p // cfg.k)
        counts[: p % cfg.k] += 1
        return counts
    w = rng.dirichlet(np.ones(cfg.k))
    return rng.multinomial(p, w)


def host_observations(cfg: Config, seed: int, p: int | None = None) -> np.ndarray:
    """V (n x p) on the host, the reference's ObservationSet layout."""
    rng = np.random.default_rng(seed)
    p = cfg.p if p is None else int(p)
    dt = np.float32 if cfg.dtype == "f32" else np.float64
    if cfg.k == 0:
        V = rng.standard_normal((cfg.n, p)) / np.sqrt(cfg.n)
        return V.astype(dt, copy=False)
    mu = _means(cfg, rng)
    labels = np.repeat(np.arange(cfg.k), _counts(cfg, p, rng))
    V = mu[:, labels] + cfg.sigma * rng.standard_normal((cfg.n, p))
    return V.astype(dt, copy=False)


def initial_point(cfg: Config, seed: int) -> tuple[np.ndarray, np.ndarray]:
    """lam0 = 1/r, A0 ~ N(0,1) column-normalised (reference gmm.py:141-149)."""
    rng = np.random.default_rng(seed + 7919)
    A = rng.standard_normal((cfg.n, cfg.r))
    A /= np.linalg.norm(A, axis=0)
    return np.full(cfg.r, 1.0 / cfg.r), A


def device_observations(cfg: Config, seed: int, p: int | None = None, *, device=None,
                        row_offset: int = 0, rows: int | None = None):
    """Observation-major (rows x n) CUDA tensor of the config's mixture, generated on the GPU.

    Rows [row_offset, row_offset + rows) of a p-observation set.  Components are assigned in
    contiguous runs (as :func:`host_observations` does) and the noise is drawn per fixed global
    chunk of rows, so any row shard is bit-identical to the same rows of the full set.
    """
    import torch

    p = cfg.p if p is None else int(p)
    rows = p - row_offset if rows is None else int(rows)
    dt = torch.float32 if cfg.dtype == "f32" else torch.float64
    dev = torch.device(device if device is not None else "cuda")
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    mu = bounds = None
    if cfg.k:
        mu = torch.randn(cfg.k, cfg.n, generator=gen, device=dev, dtype=torch.float64)
        if cfg.means == "unit":
            mu /= mu.norm(dim=1, keepdim=True)
        else:
            mu /= cfg.n ** 0.5
        counts = _counts(cfg, p, np.random.default_rng(seed + 1))
        bounds = torch.as_tensor(np.cumsum(counts), device=dev)
    out = torch.empty(rows, cfg.n, dtype=dt, device=dev)
    chunk = max(1, (1 << 26) // cfg.n)
    lo, hi = row_offset, row_offset + rows
    for gc in range(lo // chunk, (hi + chunk - 1) // chunk):
        g0, g1 = gc * chunk, min(p, (gc + 1) * chunk)
        cgen = torch.Generator(device=dev)
        cgen.manual_seed(seed * 1_000_003 + gc)
        noise = torch.randn(g1 - g0, cfg.n, generator=cgen, device=dev, dtype=torch.float32)
        a, b = max(g0, lo), min(g1, hi)
        noise = noise[a - g0:b - g0]
        if mu is None:
            out[a - lo:b - lo] = (noise.double() / cfg.n ** 0.5).to(dt)
        else:
            idx = torch.arange(a, b, device=dev)
            lab = torch.searchsorted(bounds, idx, right=True)
            out[a - lo:b - lo] = (mu[lab] + cfg.sigma * noise.double()).to(dt)
    return out
