// Auxiliary kernels of one evaluation: factor-fragment prep, deterministic partial reduction
// (K3) and the O(n r^2) device tail (K4).
#pragma once

#include "mcp_common.cuh"
#include "tail_pieces.cuh"
#include "pdl.h"

namespace mcp {

// Build the B-fragment ordered factor blocks K1 stages into shared memory:
// Afrag[rb][ks][nt][lane] = A[4ks + t][rb*RB + 8nt + g]  (lane = 4g + t), zero outside n x r.
// A is n x r column-major, i.e. x + r of the packed variable vector (optimize.py:104-110).
__global__ void k_prep_afrag(const double* __restrict__ A, int n, int r, int RB, int rbs, int kst,
                             double* __restrict__ Afrag) {
  pdl_enter();
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
// Y blocks: K3_X consecutive outputs x K3_Y partial lanes; lane ty sums partials q = ty,
// ty + K3_Y, ... in order, then a fixed binary tree over the lanes (one or two loads per thread at
// gp = 148: the reduce is latency-, not bandwidth-bound).  The w block uses 32 columns x 32
// lanes the same way.  K3 and K3F share both orders, so partial + finish == fused, bitwise.

template <int X, int Y>
__device__ __forceinline__ double k3_tree(double s, double* sm, int tx, int ty) {
  sm[ty * X + tx] = s;
  __syncthreads();
#pragma unroll
  for (int stride = Y / 2; stride > 0; stride >>= 1) {
    if (ty < stride) sm[ty * X + tx] += sm[(ty + stride) * X + tx];
    __syncthreads();
  }
  const double t = sm[tx];
  __syncthreads();
  return t;
}

// Y entry e = i * RB + jl of column block rb (valid when e < n * RB)
__device__ __forceinline__ double k3_y_lane(const double* __restrict__ Ypart, int n_pad, int RB,
                                            int gp, int rb, int e, int ty) {
  const int i = e / RB, jl = e % RB;
  const double* src = Ypart + ((size_t)rb * gp * n_pad + i) * RB + jl;
  double s = 0.0;
  for (int q = ty; q < gp; q += K3_Y) s += src[(size_t)q * n_pad * RB];
  return s;
}
__device__ __forceinline__ double k3_w_lane(const double* __restrict__ wpart, int RB, int gp,
                                            int k, int ty) {
  const int rb = k / RB, jl = k % RB;
  const double* src = wpart + (size_t)rb * gp * RB + jl;
  double s = 0.0;
  for (int q = ty; q < gp; q += K3W_Y) s += src[(size_t)q * RB];
  return s;
}

// Publication without a reduce (fast mode: its w is formed after K3)
__global__ void k_publish(K3Signal sig) {
  if (threadIdx.x != 0) return;
  __threadfence_system();
  for (int k = 0; k < sig.world; ++k)
    asm volatile("st.release.sys.global.b64 [%0], %1;\n" ::"l"(sig.flags[k] + sig.rank),
                 "l"(sig.epoch)
                 : "memory");
}

__global__ void __launch_bounds__(K3_T)
    k_reduce_partials(const double* __restrict__ Ypart, const double* __restrict__ wpart, int n,
                      int r, int n_pad, int RB, int rbs, int gp, double* __restrict__ Yw,
                      K3Signal sig = K3Signal()) {
  // PDL: launched while K1 drains; its partials are complete only after this wait
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  __shared__ double sm[K3_T];
  const int per_rb = n * RB;
  const int yblocks = (per_rb + K3_X - 1) / K3_X;
  const int wblocks = wpart ? (rbs * RB + K3W_X - 1) / K3W_X : 0;
  const int64_t total_blocks = (int64_t)rbs * yblocks + wblocks;
  for (int64_t blk = blockIdx.x; blk < total_blocks; blk += gridDim.x) {
    if (blk < (int64_t)rbs * yblocks) {
      const int tx = threadIdx.x % K3_X, ty = threadIdx.x / K3_X;
      const int rb = blk / yblocks;
      const int e = (blk % yblocks) * K3_X + tx;
      const double s = e < per_rb ? k3_y_lane(Ypart, n_pad, RB, gp, rb, e, ty) : 0.0;
      const double t = k3_tree<K3_X, K3_Y>(s, sm, tx, ty);
      if (ty == 0 && e < per_rb) {
        const int i = e / RB, j = rb * RB + e % RB;
        if (j < r) Yw[(int64_t)j * n + i] = t;
      }
    } else {
      const int tx = threadIdx.x % K3W_X, ty = threadIdx.x / K3W_X;
      const int k = (int)(blk - (int64_t)rbs * yblocks) * K3W_X + tx;   // k = rb * RB + jl
      const double s = k < rbs * RB ? k3_w_lane(wpart, RB, gp, k, ty) : 0.0;
      const double t = k3_tree<K3W_X, K3W_Y>(s, sm, tx, ty);
      if (ty == 0 && k < rbs * RB) {
        const int j = (k / RB) * RB + k % RB;
        if (j < r) Yw[(int64_t)n * r + j] = t;
      }
    }
  }
  if (sig.flags) {
    __shared__ bool last;
    __threadfence_system();   // this block's outputs, before its ticket
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(sig.ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (last && threadIdx.x == 0) {
      *sig.ticket = 0u;
      __threadfence_system();
      for (int k = 0; k < sig.world; ++k)
        asm volatile("st.release.sys.global.b64 [%0], %1;\n" ::"l"(sig.flags[k] + sig.rank),
                     "l"(sig.epoch)
                     : "memory");
    }
  }
}

// K3F: the fixed-order partial reduce of K3 fused with the whole finish (objective.py:51-56,
// implicit.py:143-151) for r <= 32.  Every block first forms G, C (and the M / u entries it
// needs) from x alone -- under programmatic dependent launch this runs while K1 drains -- then
// waits for K1's partials: g_A = -2d (Y - M) o lam is elementwise on the reduced Y,
// g_lam = -2 (w - u), f = alpha + lam.u - 2 w.lam.  out = [f ; g_lam ; vec_F(g_A)], bitwise the
// K3 + K4 result.
__global__ void __launch_bounds__(K3_T)
    k_reduce_finish(const double* __restrict__ Ypart, const double* __restrict__ wpart, int n,
                    int r, int n_pad, int RB, int rbs, int gp, const double* __restrict__ x, int d,
                    const double* __restrict__ alpha_dev, double alpha_host,
                    double* __restrict__ out) {
  __shared__ double sm[K3_T];
  __shared__ double s_w[K3W_X];
  __shared__ double sG[K3F_MAXR * K3F_MAXR], sC[K3F_MAXR * K3F_MAXR];
  __shared__ double s_u[K3F_MAXR];
  const double* lam = x;
  // x is final here: K1 (launched before us) waited for its producer before triggering us
  tail_gc_block(x, n, r, d, sG, sC);
  __syncthreads();
  // PDL: K1's partials are complete only after this wait; the next kernel may start its V-only
  // prologue right away.
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  const int per_rb = n * RB;
  const int yblocks = (per_rb + K3_X - 1) / K3_X;
  const int64_t total_blocks = (int64_t)rbs * yblocks + 1;   // + the w / f block
  const double s2d = -2.0 * d;
  for (int64_t blk = blockIdx.x; blk < total_blocks; blk += gridDim.x) {
    if (blk < (int64_t)rbs * yblocks) {
      const int tx = threadIdx.x % K3_X, ty = threadIdx.x / K3_X;
      const int rb = blk / yblocks;
      const int e = (blk % yblocks) * K3_X + tx;
      const double s = e < per_rb ? k3_y_lane(Ypart, n_pad, RB, gp, rb, e, ty) : 0.0;
      const double t = k3_tree<K3_X, K3_Y>(s, sm, tx, ty);
      if (ty == 0 && e < per_rb) {
        const int i = e / RB, j = rb * RB + e % RB;
        if (j < r) {
          const double m = tail_m_entry(x, sC, n, r, i, j);
          out[1 + r + (int64_t)j * n + i] = (s2d * (t - m)) * lam[j];
        }
      }
    } else {
      // w (rbs * RB <= 32 columns): reduce, then g_lam and f
      const int tx = threadIdx.x % K3W_X, ty = threadIdx.x / K3W_X;
      const int k = tx;
      const double s = k < rbs * RB ? k3_w_lane(wpart, RB, gp, k, ty) : 0.0;
      const double t = k3_tree<K3W_X, K3W_Y>(s, sm, tx, ty);
      if (ty == 0 && k < rbs * RB) {
        const int j = (k / RB) * RB + k % RB;
        if (j < r) {
          const double u = tail_u_entry(sG, sC, lam, r, j);
          s_w[j] = t;
          s_u[j] = u;
          out[1 + j] = -2.0 * (t - u);
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        double lu = 0.0, wl = 0.0;
        for (int jj = 0; jj < r; ++jj) lu += lam[jj] * s_u[jj];
        for (int jj = 0; jj < r; ++jj) wl += s_w[jj] * lam[jj];
        const double alpha = alpha_dev ? *alpha_dev : alpha_host;
        out[0] = alpha + lu - 2.0 * wl;
      }
      __syncthreads();
    }
  }
}

// K4a: G = A^T A and C = G^(d-1) (implicit.py:147-148), row-major r x r.  One warp per upper
// triangle entry (j <= k): lanes stride over the n rows of the two columns (coalesced), then a
// fixed butterfly; the value is mirrored so G is exactly symmetric.  Launch with 256-thread
// blocks (K4A_WARPS warps per block).
constexpr int K4A_WARPS = 8;
__global__ void k_tail_gram(const double* __restrict__ x, int n, int r, int d,
                            double* __restrict__ G, double* __restrict__ C) {
  pdl_enter();
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
    // unrolled so the loads of several trips are in flight (same sequential sum order)
#pragma unroll 8
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
  pdl_enter();
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
  pdl_enter();
  const double* lam = x;
  const double* A = x + r;
  const int64_t total = (int64_t)n * r;
  const double s = -2.0 * d;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int j = idx / n, i = idx % n;
    double m = 0.0;
#pragma unroll 8
    for (int k = 0; k < r; ++k) m += (A[(int64_t)k * n + i] * lam[k]) * C[(int64_t)k * r + j];
    out[1 + r + idx] = (s * (Y[idx] - m)) * lam[j];
  }
}

// K4 fused (one CTA) for small factor blocks (n*r <= K4S_MAX_NR, r <= K4S_MAX_R): G, C, u, f, g_lam
// and g_A in a single launch, all intermediates in shared memory.  Same algebra and operation
// order as the three-kernel tail above (implicit.py:147-149, objective.py:51-56).
constexpr int K4S_THREADS = 512;
constexpr int K4S_MAX_NR = 4096;    // A staged in (dynamic) shared memory
constexpr int K4S_MAX_R = 32;
__host__ __device__ constexpr size_t k4s_smem_bytes(int64_t nr) {
  return sizeof(double) * ((size_t)nr + (size_t)K4S_MAX_R * K4S_MAX_R + K4S_MAX_R);
}
__global__ void __launch_bounds__(K4S_THREADS)
    k_tail_fused(const double* __restrict__ x, const double* __restrict__ Y,
                 const double* __restrict__ w, int n, int r, int d,
                 const double* __restrict__ alpha_dev, double alpha_host,
                 double* __restrict__ out, int64_t sx = 0, int64_t sy = 0, int64_t sw = 0,
                 int64_t so = 0) {
  pdl_enter();
  // batched launches: CTA b handles start b (strides between consecutive starts' buffers)
  x += blockIdx.x * sx;
  Y += blockIdx.x * sy;
  w += blockIdx.x * sw;
  out += blockIdx.x * so;
  extern __shared__ double k4s_smem[];   // [K4S_MAX_R^2 C][K4S_MAX_R u][n r A]
  double* sC = k4s_smem;
  double* sU = sC + K4S_MAX_R * K4S_MAX_R;
  double* sA = sU + K4S_MAX_R;
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
