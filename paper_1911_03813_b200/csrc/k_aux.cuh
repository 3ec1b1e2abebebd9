// Auxiliary kernels of one evaluation: factor-fragment prep, deterministic partial reduction
// (K3) and the O(n r^2) device tail (K4).
#pragma once

#include "mcp_common.cuh"

namespace mcp {

// Build the B-fragment ordered factor blocks K1 stages into shared memory:
// Afrag[rb][ks][nt][lane] = A[4ks + t][rb*RB + 8nt + g]  (lane = 4g + t), zero outside n x r.
// A is n x r column-major, i.e. x + r of the packed variable vector (optimize.py:104-110).
__global__ void k_prep_afrag(const double* __restrict__ A, int n, int r, int RB, int rbs, int kst,
                             double* __restrict__ Afrag) {
  const int NT = RB / 8;
  const int64_t total = (int64_t)rbs * kst * NT * 32;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int lane = idx % 32;
    int64_t rest = idx / 32;
    const int nt = rest % NT;
    rest /= NT;
    const int ks = rest % kst;
    const int rb = rest / kst;
    const int i = 4 * ks + (lane & 3);
    const int j = rb * RB + 8 * nt + (lane >> 2);
    Afrag[idx] = (i < n && j < r) ? A[(int64_t)j * n + i] : 0.0;
  }
}

// K3: Y[i][j] = sum over persistent CTAs (fixed order) of the per-CTA partials; w likewise.
// Output Yw = [vec_F(Y) (n*r) ; w (r)], the additive piece all-reduced across ranks.
__global__ void k_reduce_partials(const double* __restrict__ Ypart, const double* __restrict__ wpart,
                                  int n, int r, int n_pad, int RB, int rbs, int gp,
                                  double* __restrict__ Yw) {
  const int64_t ny = (int64_t)rbs * n * RB;
  const int64_t total = ny + (int64_t)rbs * RB;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    if (idx < ny) {
      const int jl = idx % RB;
      const int64_t rest = idx / RB;
      const int i = rest % n;
      const int rb = rest / n;
      const int j = rb * RB + jl;
      if (j >= r) continue;
      const double* src = Ypart + ((size_t)rb * gp * n_pad + i) * RB + jl;
      double s = 0.0;
      for (int q = 0; q < gp; ++q) s += src[(size_t)q * n_pad * RB];
      Yw[(int64_t)j * n + i] = s;
    } else {
      const int64_t k = idx - ny;
      const int jl = k % RB;
      const int rb = k / RB;
      const int j = rb * RB + jl;
      if (j >= r) continue;
      const double* src = wpart + (size_t)rb * gp * RB + jl;
      double s = 0.0;
      for (int q = 0; q < gp; ++q) s += src[(size_t)q * RB];
      Yw[(int64_t)n * r + j] = s;
    }
  }
}

// K4a: G = A^T A and C = G^(d-1) (implicit.py:147-148), row-major r x r.
__global__ void k_tail_gram(const double* __restrict__ x, int n, int r, int d,
                            double* __restrict__ G, double* __restrict__ C) {
  const double* A = x + r;
  const int64_t total = (int64_t)r * r;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int j = idx / r, k = idx % r;
    const double* aj = A + (int64_t)j * n;
    const double* ak = A + (int64_t)k * n;
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += aj[i] * ak[i];
    G[idx] = s;
    C[idx] = rm_pow(s, d - 1);
  }
}

// K4b (one CTA): u = (G o C) lam, g_lam = -2 (w - u), f = alpha + lam.u - 2 w.lam
// (implicit.py:149, objective.py:53-54).  out = [f ; g_lam ; g_A].
__global__ void k_tail_vec(const double* __restrict__ x, const double* __restrict__ Yw,
                           const double* __restrict__ G, const double* __restrict__ C, int n, int r,
                           const double* __restrict__ alpha_dev, double alpha_host,
                           double* __restrict__ out) {
  extern __shared__ double s_u[];
  const double* lam = x;
  const double* w = Yw + (int64_t)n * r;
  for (int j = threadIdx.x; j < r; j += blockDim.x) {
    double u = 0.0;
    for (int k = 0; k < r; ++k) u += (G[(int64_t)j * r + k] * C[(int64_t)j * r + k]) * lam[k];
    s_u[j] = u;
    out[1 + j] = -2.0 * (w[j] - u);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double lu = 0.0, wl = 0.0;
    for (int j = 0; j < r; ++j) lu += lam[j] * s_u[j];
    for (int j = 0; j < r; ++j) wl += w[j] * lam[j];
    const double alpha = alpha_dev ? *alpha_dev : alpha_host;
    out[0] = alpha + lu - 2.0 * wl;
  }
}

// K4c: g_A = -2d (Y - (A o lam) C) o lam (objective.py:55), column-major into out + 1 + r.
__global__ void k_tail_ga(const double* __restrict__ x, const double* __restrict__ Yw,
                          const double* __restrict__ C, int n, int r, int d,
                          double* __restrict__ out) {
  const double* lam = x;
  const double* A = x + r;
  const int64_t total = (int64_t)n * r;
  const double s = -2.0 * d;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int j = idx / n, i = idx % n;
    double m = 0.0;
    for (int k = 0; k < r; ++k) m += (A[(int64_t)k * n + i] * lam[k]) * C[(int64_t)k * r + j];
    out[1 + r + idx] = (s * (Yw[idx] - m)) * lam[j];
  }
}

}  // namespace mcp
