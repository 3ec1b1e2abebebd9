// K5 (FP64 mode): ||X||^2 = nu^T (V^T V)^d nu without the p x p Gram.
//
// Replaces pkg/src/momentcp/implicit.py:116-121 (G = V^T V -> G**d elementwise -> nu @ G @ nu),
// whose p x p intermediate is 320 GB at BASELINE config 4.  The Gram is visited as 64 x 64
// tiles (I, J) with I <= J (symmetry: off-diagonal tiles count twice, exact x2); each tile is a
// DMMA.8x8x4 GEMM over n in 64-wide chunks with an in-register epilogue
//   sum += nu_l nu_l' * g_ll'^d    (g^d by repeated multiplication, implicit.py:82-91).
// Tile pairs are split statically over persistent CTAs (and over GPUs via [begin, end)); each
// CTA's sum is written once and reduced in a fixed order, so the result is deterministic.
#pragma once

#include "mcp_common.cuh"

namespace mcp {

constexpr int K5_T = 64;
constexpr int K5_NK = 64;
constexpr int K5_SV = 68;
constexpr int K5_THREADS = 256;

template <typename VT>
__host__ __device__ constexpr size_t k5_smem_bytes() {
  return 4 * (size_t)K5_T * K5_SV * sizeof(VT) + 8 * sizeof(double);
}

// pair index k -> (I, J), I <= J, row-major over the upper triangle of a T x T tile grid.
__device__ __forceinline__ void k5_decode(int64_t k, int64_t T, int64_t& I, int64_t& J) {
  const double b = 2.0 * (double)T + 1.0;
  int64_t i = (int64_t)floor((b - sqrt(b * b - 8.0 * (double)k)) * 0.5);
  if (i < 0) i = 0;
  auto cum = [T](int64_t ii) { return ii * T - ii * (ii - 1) / 2; };
  while (i > 0 && cum(i) > k) --i;
  while (cum(i + 1) <= k) ++i;
  I = i;
  J = i + (k - cum(i));
}

template <typename VT>
__device__ __forceinline__ void k5_load(VT* dst, const VT* __restrict__ V, int64_t ldv,
                                        int64_t row0, int c) {
  constexpr int SEG = 16 / sizeof(VT);
  constexpr int SEGS_ROW = K5_NK / SEG;
  constexpr int TOTAL = K5_T * SEGS_ROW;
#pragma unroll
  for (int s = threadIdx.x; s < TOTAL; s += K5_THREADS) {
    const int row = s / SEGS_ROW, seg = s % SEGS_ROW;
    const int64_t col = (int64_t)c * K5_NK + seg * SEG;
    const bool ok = col < ldv;
    const VT* src = ok ? V + (row0 + row) * ldv + col : V;
    cp_async16(dst + row * K5_SV + seg * SEG, src, ok ? 16 : 0);
  }
}

template <typename VT>
__global__ void __launch_bounds__(K5_THREADS)
    k5_gram_power(const VT* __restrict__ V, int64_t ldv, int n_chunks, const double* __restrict__ nu,
                  double nu_const, int d, int64_t T, int64_t pair_begin, int64_t pair_end,
                  double* __restrict__ part) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  VT* sI[2];
  VT* sJ[2];
  sI[0] = reinterpret_cast<VT*>(smem_raw);
  sI[1] = sI[0] + K5_T * K5_SV;
  sJ[0] = sI[1] + K5_T * K5_SV;
  sJ[1] = sJ[0] + K5_T * K5_SV;
  double* sRed = reinterpret_cast<double*>(sJ[1] + K5_T * K5_SV);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp >> 2;  // 2 x 32 rows
  const int wn = warp & 3;   // 4 x 16 cols
  double tsum = 0.0;

  for (int64_t pair = pair_begin + blockIdx.x; pair < pair_end; pair += gridDim.x) {
    int64_t I, J;
    k5_decode(pair, T, I, J);
    double acc[4][2][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

    k5_load<VT>(sI[0], V, ldv, I * K5_T, 0);
    k5_load<VT>(sJ[0], V, ldv, J * K5_T, 0);
    cp_async_commit();
    for (int c = 0; c < n_chunks; ++c) {
      const int s = c & 1;
      if (c + 1 < n_chunks) {
        k5_load<VT>(s ? sI[0] : sI[1], V, ldv, I * K5_T, c + 1);
        k5_load<VT>(s ? sJ[0] : sJ[1], V, ldv, J * K5_T, c + 1);
        cp_async_commit();
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      const VT* ai = (s ? sI[1] : sI[0]) + (32 * wm + g) * K5_SV + t;
      const VT* bj = (s ? sJ[1] : sJ[0]) + (16 * wn + g) * K5_SV + t;
#pragma unroll 4
      for (int ks = 0; ks < 16; ++ks) {
        double a[4], b[2];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) a[mt] = to_f64(ai[8 * mt * K5_SV + 4 * ks]);
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) b[nt] = to_f64(bj[8 * nt * K5_SV + 4 * ks]);
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) dmma884(acc[mt][nt], a[mt], b[nt]);
      }
      __syncthreads();
    }

    // epilogue: sum nu_l nu_l' g^d over the tile (x2 off the diagonal)
    double tile_sum = 0.0;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      const int64_t l = I * K5_T + 32 * wm + 8 * mt + g;
      const double nl = nu ? nu[l] : nu_const;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t l2 = J * K5_T + 16 * wn + 8 * nt + 2 * t + e;
          const double nl2 = nu ? nu[l2] : nu_const;
          tile_sum += (nl * nl2) * rm_pow(acc[mt][nt][e], d);
        }
    }
    tsum += (I == J) ? tile_sum : 2.0 * tile_sum;
  }

  // fixed-order block reduction
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) tsum += __shfl_xor_sync(0xffffffffu, tsum, off);
  if (lane == 0) sRed[warp] = tsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < K5_THREADS / 32; ++w) s += sRed[w];
    part[blockIdx.x] = s;
  }
}

// ---- K5 v2: 128 x 128 tile pairs, 16 warps (4 x 4 warp grid, 32 x 32 per warp), 32-wide
// n-chunks double buffered.  4 + 4 fragment loads feed 16 DMMAs per k-step (vs 6 per 8 for
// 64 x 64 tiles) and each pair moves half the L2 bytes per flop.
constexpr int K52_T = 128;
constexpr int K52_NK = 32;
constexpr int K52_SV = 36;   // == 4 (mod 16) doubles: conflict-free 8-byte fragment loads
constexpr int K52_THREADS = 512;

template <typename VT>
__host__ __device__ constexpr size_t k52_smem_bytes() {
  return 4 * (size_t)K52_T * K52_SV * sizeof(VT) + 16 * sizeof(double);
}

template <typename VT>
__device__ __forceinline__ void k52_load(VT* dst, const VT* __restrict__ V, int64_t ldv,
                                         int64_t row0, int c) {
  constexpr int SEG = 16 / sizeof(VT);
  constexpr int SEGS_ROW = K52_NK / SEG;
  constexpr int TOTAL = K52_T * SEGS_ROW;
#pragma unroll
  for (int s = threadIdx.x; s < TOTAL; s += K52_THREADS) {
    const int row = s / SEGS_ROW, seg = s % SEGS_ROW;
    const int64_t col = (int64_t)c * K52_NK + seg * SEG;
    const bool ok = col < ldv;
    const VT* src = ok ? V + (row0 + row) * ldv + col : V;
    cp_async16(dst + row * K52_SV + seg * SEG, src, ok ? 16 : 0);
  }
}

// Second operand of a cross-shard reduction (sharded ||X||^2): the J tiles come from another
// row shard VJ (same pitch and dtype), the tile pairs (I, J) cover the whole TI x TJ rectangle
// in row-major order (pair k -> I = k / TJ, J = k % TJ; colmajor: I = k % TI, J = k / TI), every
// tile counts twice (the (J, I) half of the symmetric Gram lives on the other shard's side).
// VJ == nullptr: the upper triangle of one shard's own Gram (off-diagonal tiles x2).
template <typename VT>
struct K52Cross {
  const VT* VJ = nullptr;
  const double* nuJ = nullptr;
  double nu_constJ = 0.0;
  int64_t TJ = 0;
  int colmajor = 0;
};

template <typename VT>
__global__ void __launch_bounds__(K52_THREADS, 1)
    k52_gram_power(const VT* __restrict__ V, int64_t ldv, int n_chunks, const double* __restrict__ nu,
                   double nu_const, int d, int64_t T, int64_t pair_begin, int64_t pair_end,
                   double* __restrict__ part, K52Cross<VT> cross) {
  extern __shared__ __align__(16) unsigned char smem_raw5[];
  VT* sI[2];
  VT* sJ[2];
  sI[0] = reinterpret_cast<VT*>(smem_raw5);
  sI[1] = sI[0] + K52_T * K52_SV;
  sJ[0] = sI[1] + K52_T * K52_SV;
  sJ[1] = sJ[0] + K52_T * K52_SV;
  double* sRed = reinterpret_cast<double*>(sJ[1] + K52_T * K52_SV);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp >> 2, wn = warp & 3;   // 4 x 4 warps, 32 x 32 each
  double tsum = 0.0;
  const bool rect = cross.VJ != nullptr;
  const VT* __restrict__ VJ = rect ? cross.VJ : V;
  const double* __restrict__ nuJ = rect ? cross.nuJ : nu;
  const double nu_cJ = rect ? cross.nu_constJ : nu_const;
  auto decode = [&](int64_t k, int64_t& I_, int64_t& J_) {
    if (rect && cross.colmajor) {
      I_ = k % T;
      J_ = k / T;
    } else if (rect) {
      I_ = k / cross.TJ;
      J_ = k % cross.TJ;
    } else {
      k5_decode(k, T, I_, J_);
    }
  };

  // one cp.async pipeline over the flat (pair, chunk) sequence: the last chunk of a pair
  // prefetches chunk 0 of the CTA's next pair, so no tile pair starts on an exposed load
  int64_t pair = pair_begin + blockIdx.x;
  int64_t I = 0, J = 0;
  if (pair < pair_end) {
    decode(pair, I, J);
    k52_load<VT>(sI[0], V, ldv, I * K52_T, 0);
    k52_load<VT>(sJ[0], VJ, ldv, J * K52_T, 0);
    cp_async_commit();
  }
  int s = 0;   // buffer of the chunk being consumed (continues across pairs)
  for (; pair < pair_end; pair += gridDim.x) {
    const int64_t npair = pair + gridDim.x;
    int64_t nI = 0, nJ = 0;
    if (npair < pair_end) decode(npair, nI, nJ);
    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

    for (int c = 0; c < n_chunks; ++c) {
      const bool more = c + 1 < n_chunks || npair < pair_end;
      if (more) {
        const int64_t li = c + 1 < n_chunks ? I : nI, lj = c + 1 < n_chunks ? J : nJ;
        const int lc = c + 1 < n_chunks ? c + 1 : 0;
        k52_load<VT>(s ? sI[0] : sI[1], V, ldv, li * K52_T, lc);
        k52_load<VT>(s ? sJ[0] : sJ[1], VJ, ldv, lj * K52_T, lc);
        cp_async_commit();
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      const VT* ai = (s ? sI[1] : sI[0]) + (32 * wm + g) * K52_SV + t;
      const VT* bj = (s ? sJ[1] : sJ[0]) + (32 * wn + g) * K52_SV + t;
#pragma unroll
      for (int ks = 0; ks < K52_NK / 4; ++ks) {
        double a[4], b[4];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) a[mt] = to_f64(ai[8 * mt * K52_SV + 4 * ks]);
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) b[nt] = to_f64(bj[8 * nt * K52_SV + 4 * ks]);
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) dmma884(acc[mt][nt], a[mt], b[nt]);
      }
      __syncthreads();
      s ^= 1;
    }

    double tile_sum = 0.0;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      const int64_t l = I * K52_T + 32 * wm + 8 * mt + g;
      const double nl = nu ? nu[l] : nu_const;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t l2 = J * K52_T + 32 * wn + 8 * nt + 2 * t + e;
          const double nl2 = nuJ ? nuJ[l2] : nu_cJ;
          tile_sum += (nl * nl2) * rm_pow(acc[mt][nt][e], d);
        }
    }
    tsum += (I == J && !rect) ? tile_sum : 2.0 * tile_sum;
    I = nI;
    J = nJ;
  }

#pragma unroll
  for (int off = 16; off > 0; off >>= 1) tsum += __shfl_xor_sync(0xffffffffu, tsum, off);
  if (lane == 0) sRed[warp] = tsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    double sum = 0.0;
    for (int w = 0; w < K52_THREADS / 32; ++w) sum += sRed[w];
    part[blockIdx.x] = sum;
  }
}

// Ordered sum of per-CTA partials (single thread: <= a few thousand values).
__global__ void k_ordered_sum(const double* __restrict__ part, int m, double* __restrict__ out) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < m; ++i) s += part[i];
    *out = s;
  }
}

}  // namespace mcp
