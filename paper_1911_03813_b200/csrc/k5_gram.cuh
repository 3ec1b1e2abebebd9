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

#include <cuda.h>

#include "k1s_fp64.cuh"      // mbarrier helpers
#include "k1x_common.cuh"    // ordered shared loads, async-proxy fence
#include "mcp_common.cuh"
#include "umma.cuh"          // TMA helpers

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


// ---- K53 (fp64 sets): K52's 128 x 128 tile pairs and 4 x 4 warp grid, fed like K1X ----------
// ncu at c4 put K52 at 78% of the FP64 pipe with 11% of the warp time issuing cp.async (2048
// 16-byte copies and their addresses per 32-column chunk) and the rest of the loss at the two
// __syncthreads per chunk.  K53 stages each 16-double chunk of the I and J tiles with one 2-D TMA
// apiece (128-byte swizzle) into a ring of 6 stages that flows across tile pairs; the 16 warps
// wait on the stage's mbarrier and, after the chunk, meet at one CTA barrier, after which thread
// 0 refills the stage STAGES - 1 chunks ahead.  Measured at c4: 360.8 ms, the same as K52 (359.4;
// 77% of the FP64 pipe) with one TMA pair per chunk instead of 2048 cp.async.  Releasing stages
// warp by warp with the last warp refilling (no CTA barrier, K1X's scheme) measured 404 ms: the
// fastest warps run to the end of the ring and then wait for refills gated by the slowest warp.
// Round 2: the refill decode (sqrt + 64-bit divisions per chunk on warp 0) made warp 0 the
// straggler at every barrier (ncu source view: 15% of samples behind BAR.SYNC); the refill cursor
// is now kept by every thread, decoded once per pair, the refilling warp rotates, and the next
// k-step's operands load before the current DMMAs -- 359.5 -> 346.8 ms (76.8% -> 79.6%).  Then
// each tile pair split into two 64-row halves of I on neighbouring CTAs (8 warps, 4-stage ring,
// two CTAs per SM): one CTA's barrier skew and epilogue are covered by the other CTA's DMMAs --
// 349.3 -> 333.0 ms (83% of the FP64 pipe; profiles/r02/ab_c4_k53_halves.txt).  Fragment loads stay conflict-free under
// the swizzle by letting DMMA row (column) g of a 8-row m-tile read physical tile row
// 2g (g < 4) / 2(g - 4) + 1 (g >= 4): the 16 lanes of a half-warp then hit 16 distinct 8-byte
// banks.  The epilogue uses the same row map for the weights, so the sum is the same Gram power
// sum as K52 (tile-pair order and the per-CTA fixed-order reduction unchanged).
constexpr int K53_T = 128;
constexpr int K53_NK = 16;          // doubles per chunk row (one 128-byte swizzle row)
// TI = rows of the I tile a CTA takes: 128 (16 warps, one CTA per SM) or 64 (K53H: each tile
// pair split in two row halves, 8 warps per CTA, two CTAs per SM -- one CTA's barrier skew and
// epilogue are covered by the other's DMMAs)
#ifndef MCP_K53_STAGES32
#define MCP_K53_STAGES32 2   // ring depth of the 32-row form (2: four CTAs per SM, 3: three)
#endif
template <int TI> __host__ __device__ constexpr int k53_threads() { return 4 * TI; }
template <int TI> __host__ __device__ constexpr int k53_stages() {
  return TI == 128 ? 6 : TI == 64 ? 4 : MCP_K53_STAGES32;
}
template <int TI> __host__ __device__ constexpr int k53_stage_bytes() { return (TI + K53_T) * K53_NK * 8; }
constexpr int K53_THREADS = k53_threads<128>();
constexpr int K53_STAGES = k53_stages<128>();
constexpr int K53_STAGE_BYTES = k53_stage_bytes<128>();   // I and J chunks, 32 KB
#ifndef MCP_K53_SYNC
#define MCP_K53_SYNC 1
#endif
// chunks per CTA barrier (and refill group); measured at c4 (tools/ab.sh, one box): 1 -> 346.8 ms,
// 2 -> 347.9, 3 -> 350.6 -- the skew does not amortise over longer groups
constexpr int K53_SYNC = MCP_K53_SYNC;

template <int TI = 128>
__host__ __device__ constexpr size_t k53_smem_bytes() {
  return 1024 + (size_t)k53_stages<TI>() * k53_stage_bytes<TI>() + 256;
}

__device__ __forceinline__ int k53_prow(int g) { return g < 4 ? 2 * g : 2 * (g - 4) + 1; }

template <int TI>
__global__ void __launch_bounds__(k53_threads<TI>(), 128 / TI)
    k53_gram_power(const __grid_constant__ CUtensorMap tmI, const __grid_constant__ CUtensorMap tmJ,
                   int n_chunks, const double* __restrict__ nu, double nu_const,
                   const double* __restrict__ nuJ, double nu_constJ, int d, int64_t T, int64_t TJ,
                   int rect, int colmajor, int64_t pair_begin, int64_t pair_end,
                   double* __restrict__ part) {
  constexpr int ST_ = k53_stages<TI>(), SB_ = k53_stage_bytes<TI>(), NTH_ = k53_threads<TI>();
  constexpr int HALVES = K53_T / TI;   // units per tile pair
  extern __shared__ __align__(16) unsigned char k53_raw[];
  unsigned char* base = k53_raw + ((1024u - (smem_u32(k53_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + (size_t)ST_ * SB_);
  double* sRed = reinterpret_cast<double*>(full + ST_);   // 16 doubles

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp >> 2, wn = warp & 3;   // (TI / 32) x 4 warps, 32 x 32 outputs each
  const int prow = k53_prow(g);
  const double* nuJv = rect ? nuJ : nu;
  const double ncJ = rect ? nu_constJ : nu_const;

  auto decode = [&](int64_t k, int64_t& I_, int64_t& J_) {
    if (rect && colmajor) {
      I_ = k % T;
      J_ = k / T;
    } else if (rect) {
      I_ = k / TJ;
      J_ = k % TJ;
    } else {
      k5_decode(k, T, I_, J_);
    }
  };
  // this CTA's units (tile pair x row half): unit blockIdx.x + kp * gridDim.x of
  // HALVES * (pair_end - pair_begin); both halves of a pair run on neighbouring CTAs
  const int64_t units = (pair_end - pair_begin) * HALVES;
  const int64_t my_units =
      blockIdx.x < units ? (units - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const int64_t nsteps = my_units * n_chunks;
  auto pair_of = [&](int64_t kp, int64_t& I_, int64_t& J_, int& h_) {
    const int64_t u = blockIdx.x + kp * gridDim.x;
    decode(pair_begin + u / HALVES, I_, J_);
    h_ = (int)(u % HALVES);
  };
  auto issue = [&](int s, int c, int64_t I, int64_t J, int h) {   // one chunk into stage s
    unsigned char* st = base + (size_t)s * SB_;
    mbar_arrive_expect_tx(&full[s], SB_);
    tma_load_2d(st, &tmI, c * K53_NK, (int)(I * K53_T + TI * h), smem_u32(&full[s]));
    tma_load_2d(st + TI * K53_NK * 8, &tmJ, c * K53_NK, (int)(J * K53_T), smem_u32(&full[s]));
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST_; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    tma_prefetch_desc(&tmI);
    tma_prefetch_desc(&tmJ);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t I = 0, J = 0;
    int h = 0;
    for (int64_t q = 0; q < ST_ && q < nsteps; ++q) {
      if (q % n_chunks == 0) pair_of(q / n_chunks, I, J, h);
      issue((int)q, (int)(q % n_chunks), I, J, h);
    }
  }
  // Refill cursor (step q + STAGES), kept by every thread so the refilling warp can rotate: the
  // tile-pair decode (sqrt, 64-bit divisions) runs once per pair on all warps at the same point
  // instead of once per chunk on warp 0, which made warp 0 the straggler at every chunk barrier
  // (ncu source view of the previous form: 15% of warp samples waiting behind BAR.SYNC).
  int64_t r_kp = ST_ / n_chunks;
  int r_c = ST_ % n_chunks;
  int64_t rI = 0, rJ = 0;
  int rh = 0;
  if (ST_ < nsteps) pair_of(r_kp, rI, rJ, rh);

  // per-lane word offsets (doubles) inside a stage: row * 16 + (k ^ 2 (row & 7)), row & 7 = prow
  const int swz = 2 * prow;
  int aoff[4], boff[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    aoff[i] = (32 * wm + 8 * i + prow) * K53_NK;
    boff[i] = TI * K53_NK + (32 * wn + 8 * i + prow) * K53_NK;
  }
  const uint32_t st0 = smem_u32(base);
  double tsum = 0.0;
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  int s = 0, cc = 0;      // stage, chunk of the current pair
  uint32_t ph = 0;
  int64_t kp = 0;
  for (int64_t q = 0; q < nsteps; ++q) {
    mbar_wait(&full[s], ph);
    const uint32_t sb = st0 + (uint32_t)s * SB_;
    // operands of k-step ks + 1 are loaded before k-step ks's DMMAs issue (ordered ld.shared),
    // so a warp running alone keeps the pipe fed
    double a[2][4], b[2][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[0][i] = k1w_lds_f64(sb + 8u * (uint32_t)(aoff[i] + (t ^ swz)));
#pragma unroll
    for (int i = 0; i < 4; ++i) b[0][i] = k1w_lds_f64(sb + 8u * (uint32_t)(boff[i] + (t ^ swz)));
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const int cur = ks & 1, nxt = cur ^ 1;
      if (ks < 3) {
        const int kk = (4 * (ks + 1) + t) ^ swz;
#pragma unroll
        for (int i = 0; i < 4; ++i) a[nxt][i] = k1w_lds_f64(sb + 8u * (uint32_t)(aoff[i] + kk));
#pragma unroll
        for (int i = 0; i < 4; ++i) b[nxt][i] = k1w_lds_f64(sb + 8u * (uint32_t)(boff[i] + kk));
      }
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma884(acc[mt][nt], a[cur][mt], b[cur][nt]);
    }
    // every K53_SYNC chunks: every warp is done with those stages; refill them with the steps
    // STAGES ahead (one CTA barrier per K53_SYNC chunks: the barrier skew is per barrier)
    if ((q + 1) % K53_SYNC == 0 || q + 1 == nsteps) {
      __syncthreads();
      const int64_t q0 = q + 1 - ((q % K53_SYNC) + 1);   // first step of this sync group
      for (int64_t qq = q0; qq <= q; ++qq) {
        if (qq + ST_ >= nsteps) break;
        if (warp == (int)(qq % (NTH_ / 32)) && lane == 0) {
          k1w_fence_proxy_async();
          issue((int)(qq % ST_), r_c, rI, rJ, rh);
        }
        if (++r_c == n_chunks) {
          r_c = 0;
          ++r_kp;
          if (qq + ST_ + 1 < nsteps) pair_of(r_kp, rI, rJ, rh);
        }
      }
    }
    if (++s == ST_) {
      s = 0;
      ph ^= 1u;
    }
    if (++cc == n_chunks) {
      cc = 0;
      // last chunk of a tile pair: sum nu_l nu_l' g^d over the tile (x2 off the diagonal)
      int64_t I, J;
      int h;
      pair_of(kp++, I, J, h);
      double tile_sum = 0.0;
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const int64_t l = I * K53_T + TI * h + 32 * wm + 8 * mt + prow;
        const double nl = nu ? nu[l] : nu_const;
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int64_t l2 = J * K53_T + 32 * wn + 8 * nt + k53_prow(2 * t + e);
            const double nl2 = nuJv ? nuJv[l2] : ncJ;
            tile_sum += (nl * nl2) * rm_pow(acc[mt][nt][e], d);
            acc[mt][nt][e] = 0.0;
          }
      }
      tsum += (I == J && !rect) ? tile_sum : 2.0 * tile_sum;
    }
  }

#pragma unroll
  for (int off = 16; off > 0; off >>= 1) tsum += __shfl_xor_sync(0xffffffffu, tsum, off);
  if (lane == 0) sRed[warp] = tsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    double sum = 0.0;
    for (int w = 0; w < NTH_ / 32; ++w) sum += sRed[w];
    part[blockIdx.x] = sum;
  }
}

}  // namespace mcp
