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

// K3: Y[i][j] = sum over the persistent CTAs' partials, in a fixed order; w likewise.
// Output Yw = [vec_F(Y) (n*r) ; w (r)], the additive piece all-reduced across ranks.
// Block = 32 consecutive outputs x 8 partial-groups: thread (tx, ty) sums partials
// q = ty, ty+8, ... (coalesced 256-byte rows), then ty = 0 adds the 8 group sums in order.
constexpr int K3_X = 32, K3_Y = 32;
__global__ void __launch_bounds__(K3_X * K3_Y)
    k_reduce_partials(const double* __restrict__ Ypart, const double* __restrict__ wpart, int n,
                      int r, int n_pad, int RB, int rbs, int gp, double* __restrict__ Yw) {
  __shared__ double s_acc[K3_Y][K3_X];
  const int tx = threadIdx.x % K3_X, ty = threadIdx.x / K3_X;
  const int per_rb = n * RB;                          // Y outputs of one column block
  const int yblocks = (per_rb + K3_X - 1) / K3_X;     // blocks per column block
  const int64_t total_blocks =
      (int64_t)rbs * yblocks + (wpart ? (rbs * RB + K3_X - 1) / K3_X : 0);
  for (int64_t blk = blockIdx.x; blk < total_blocks; blk += gridDim.x) {
    double s = 0.0;
    int64_t dst = -1;
    if (blk < (int64_t)rbs * yblocks) {
      const int rb = blk / yblocks;
      const int e = (blk % yblocks) * K3_X + tx;       // e = i * RB + jl
      if (e < per_rb) {
        const int i = e / RB, jl = e % RB, j = rb * RB + jl;
        const double* src = Ypart + ((size_t)rb * gp * n_pad + i) * RB + jl;
#pragma unroll 4
        for (int q = ty; q < gp; q += K3_Y) s += src[(size_t)q * n_pad * RB];
        if (j < r) dst = (int64_t)j * n + i;
      }
    } else {
      const int k = (blk - (int64_t)rbs * yblocks) * K3_X + tx;   // k = rb * RB + jl
      if (k < rbs * RB) {
        const int rb = k / RB, jl = k % RB, j = rb * RB + jl;
        const double* src = wpart + (size_t)rb * gp * RB + jl;
#pragma unroll 4
        for (int q = ty; q < gp; q += K3_Y) s += src[(size_t)q * RB];
        if (j < r) dst = (int64_t)n * r + j;
      }
    }
    s_acc[ty][tx] = s;
    __syncthreads();
    if (ty == 0 && dst >= 0) {
      double t = 0.0;
#pragma unroll
      for (int y = 0; y < K3_Y; ++y) t += s_acc[y][tx];
      Yw[dst] = t;
    }
    __syncthreads();
  }
}

// K3F: the fixed-order partial reduce of K3 fused with the finish (objective.py:51-56) when
// K1P already produced M = (A o lam) C and u = (G o C) lam: g_A = -2d (Y - M) o lam is
// elementwise on the reduced Y, g_lam = -2 (w - u), and f = alpha + lam.u - 2 w.lam (r <= 32:
// one block holds every w).  out = [f ; g_lam ; vec_F(g_A)], bitwise the k_tail_fused result.
__global__ void __launch_bounds__(K3_X * K3_Y)
    k_reduce_finish(const double* __restrict__ Ypart, const double* __restrict__ wpart, int n,
                    int r, int n_pad, int RB, int rbs, int gp, const double* __restrict__ x,
                    const double* __restrict__ M, const double* __restrict__ u, int d,
                    const double* __restrict__ alpha_dev, double alpha_host,
                    double* __restrict__ out) {
  __shared__ double s_acc[K3_Y][K3_X];
  __shared__ double s_w[K3_X];
  const int tx = threadIdx.x % K3_X, ty = threadIdx.x / K3_X;
  const double* lam = x;
  const int per_rb = n * RB;
  const int yblocks = (per_rb + K3_X - 1) / K3_X;
  const int64_t total_blocks = (int64_t)rbs * yblocks + 1;   // + the w / f block
  const double s2d = -2.0 * d;
  for (int64_t blk = blockIdx.x; blk < total_blocks; blk += gridDim.x) {
    double s = 0.0;
    if (blk < (int64_t)rbs * yblocks) {
      const int rb = blk / yblocks;
      const int e = (blk % yblocks) * K3_X + tx;
      int64_t dst = -1;
      int j = 0;
      if (e < per_rb) {
        const int i = e / RB, jl = e % RB;
        j = rb * RB + jl;
        const double* src = Ypart + ((size_t)rb * gp * n_pad + i) * RB + jl;
#pragma unroll 4
        for (int q = ty; q < gp; q += K3_Y) s += src[(size_t)q * n_pad * RB];
        if (j < r) dst = (int64_t)j * n + i;
      }
      s_acc[ty][tx] = s;
      __syncthreads();
      if (ty == 0 && dst >= 0) {
        double t = 0.0;
#pragma unroll
        for (int y = 0; y < K3_Y; ++y) t += s_acc[y][tx];
        out[1 + r + dst] = (s2d * (t - M[dst])) * lam[j];
      }
      __syncthreads();
    } else {
      // w (r <= 32 < K3_X): reduce, then g_lam and f
      const int k = tx;   // k = rb * RB + jl
      int j = r;
      if (k < rbs * RB) {
        const int rb = k / RB, jl = k % RB;
        j = rb * RB + jl;
        const double* src = wpart + (size_t)rb * gp * RB + jl;
#pragma unroll 4
        for (int q = ty; q < gp; q += K3_Y) s += src[(size_t)q * RB];
      }
      s_acc[ty][tx] = s;
      __syncthreads();
      if (ty == 0) {
        double t = 0.0;
#pragma unroll
        for (int y = 0; y < K3_Y; ++y) t += s_acc[y][tx];
        if (j < r) {
          s_w[j] = t;
          out[1 + j] = -2.0 * (t - u[j]);
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        double lu = 0.0, wl = 0.0;
        for (int jj = 0; jj < r; ++jj) lu += lam[jj] * u[jj];
        for (int jj = 0; jj < r; ++jj) wl += s_w[jj] * lam[jj];
        const double alpha = alpha_dev ? *alpha_dev : alpha_host;
        out[0] = alpha + lu - 2.0 * wl;
      }
      __syncthreads();
    }
  }
}

// K4L: the finish when M = (A o lam) C and u = (G o C) lam are already known (they came with the
// partial): g_A = -2d (Y - M) o lam elementwise, the last block g_lam and f.  Same expressions
// as k_tail_fused / k_reduce_finish.
__global__ void k_finish_light(const double* __restrict__ x, const double* __restrict__ Y,
                               const double* __restrict__ w, const double* __restrict__ M,
                               const double* __restrict__ u, int n, int r, int d,
                               const double* __restrict__ alpha_dev, double alpha_host,
                               double* __restrict__ out) {
  const double* lam = x;
  const int64_t nr = (int64_t)n * r;
  if (blockIdx.x + 1 < gridDim.x) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e < nr) {
      const int j = (int)(e / n);
      out[1 + r + e] = ((-2.0 * d) * (Y[e] - M[e])) * lam[j];
    }
    return;
  }
  for (int j = threadIdx.x; j < r; j += blockDim.x) out[1 + j] = -2.0 * (w[j] - u[j]);
  if (threadIdx.x == 0) {
    double lu = 0.0, wl = 0.0;
    for (int j = 0; j < r; ++j) lu += lam[j] * u[j];
    for (int j = 0; j < r; ++j) wl += w[j] * lam[j];
    const double alpha = alpha_dev ? *alpha_dev : alpha_host;
    out[0] = alpha + lu - 2.0 * wl;
  }
}

// K4a: G = A^T A and C = G^(d-1) (implicit.py:147-148), row-major r x r.  One warp per upper
// triangle entry (j <= k): lanes stride over the n rows of the two columns (coalesced), then a
// fixed butterfly; the value is mirrored so G is exactly symmetric.  Launch with 256-thread
// blocks (K4A_WARPS warps per block).
constexpr int K4A_WARPS = 8;
__global__ void k_tail_gram(const double* __restrict__ x, int n, int r, int d,
                            double* __restrict__ G, double* __restrict__ C) {
  const double* A = x + r;
  const int lane = threadIdx.x & 31;
  const int64_t total = (int64_t)r * r;
  for (int64_t idx = blockIdx.x * (int64_t)K4A_WARPS + (threadIdx.x >> 5); idx < total;
       idx += (int64_t)gridDim.x * K4A_WARPS) {
    const int j = (int)(idx / r), k = (int)(idx % r);
    if (j > k) continue;
    const double* aj = A + (int64_t)j * n;
    const double* ak = A + (int64_t)k * n;
    double s = 0.0;
    for (int i = lane; i < n; i += 32) s += aj[i] * ak[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      const double c = rm_pow(s, d - 1);
      G[(int64_t)j * r + k] = s;
      G[(int64_t)k * r + j] = s;
      C[(int64_t)j * r + k] = c;
      C[(int64_t)k * r + j] = c;
    }
  }
}

// K4b (one CTA): u = (G o C) lam, g_lam = -2 (w - u), f = alpha + lam.u - 2 w.lam
// (implicit.py:149, objective.py:53-54).  out = [f ; g_lam ; g_A].
__global__ void k_tail_vec(const double* __restrict__ x, const double* __restrict__ w,
                           const double* __restrict__ G, const double* __restrict__ C, int n, int r,
                           const double* __restrict__ alpha_dev, double alpha_host,
                           double* __restrict__ out) {
  extern __shared__ double s_u[];
  const double* lam = x;
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
__global__ void k_tail_ga(const double* __restrict__ x, const double* __restrict__ Y,
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
    out[1 + r + idx] = (s * (Y[idx] - m)) * lam[j];
  }
}

// K4 fused (one CTA) for small factor blocks (n*r <= K4S_MAX_NR, r <= K4S_MAX_R): G, C, u, f, g_lam
// and g_A in a single launch, all intermediates in shared memory.  Same algebra and operation
// order as the three-kernel tail above (implicit.py:147-149, objective.py:51-56).
constexpr int K4S_THREADS = 512;
constexpr int K4S_MAX_NR = 4096;
constexpr int K4S_MAX_R = 32;
__global__ void __launch_bounds__(K4S_THREADS)
    k_tail_fused(const double* __restrict__ x, const double* __restrict__ Y,
                 const double* __restrict__ w, int n, int r, int d,
                 const double* __restrict__ alpha_dev, double alpha_host,
                 double* __restrict__ out, int64_t sx = 0, int64_t sy = 0, int64_t sw = 0,
                 int64_t so = 0) {
  // batched launches: CTA b handles start b (strides between consecutive starts' buffers)
  x += blockIdx.x * sx;
  Y += blockIdx.x * sy;
  w += blockIdx.x * sw;
  out += blockIdx.x * so;
  __shared__ double sA[K4S_MAX_NR];
  __shared__ double sC[K4S_MAX_R * K4S_MAX_R];
  __shared__ double sU[K4S_MAX_R];
  const double* lam = x;
  for (int e = threadIdx.x; e < n * r; e += blockDim.x) sA[e] = x[r + e];
  __syncthreads();
  // G_jk = a_j . a_k: one warp per (j, k), lanes stride over i, fixed shuffle order
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int pr = warp; pr < r * r; pr += K4S_THREADS / 32) {
    const int j = pr / r, k = pr % r;
    double s = 0.0;
    for (int i = lane; i < n; i += 32) s += sA[j * n + i] * sA[k * n + i];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) sC[pr] = s;  // G for now
  }
  __syncthreads();
  for (int j = threadIdx.x; j < r; j += blockDim.x) {
    double u = 0.0;
    for (int k = 0; k < r; ++k) {
      const double gjk = sC[j * r + k];
      u += (gjk * rm_pow(gjk, d - 1)) * lam[k];
    }
    sU[j] = u;
    out[1 + j] = -2.0 * (w[j] - u);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) sC[e] = rm_pow(sC[e], d - 1);  // C
  __syncthreads();
  if (threadIdx.x == 0) {
    double lu = 0.0, wl = 0.0;
    for (int j = 0; j < r; ++j) lu += lam[j] * sU[j];
    for (int j = 0; j < r; ++j) wl += w[j] * lam[j];
    const double alpha = alpha_dev ? *alpha_dev : alpha_host;
    out[0] = alpha + lu - 2.0 * wl;
  }
  const double s2d = -2.0 * d;
  for (int e = threadIdx.x; e < n * r; e += blockDim.x) {
    const int j = e / n, i = e % n;
    double m = 0.0;
    for (int k = 0; k < r; ++k) m += (sA[k * n + i] * lam[k]) * sC[k * r + j];
    out[1 + r + e] = (s2d * (Y[e] - m)) * lam[j];
  }
}

}  // namespace mcp
