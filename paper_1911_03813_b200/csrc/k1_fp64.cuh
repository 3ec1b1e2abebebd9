// K1 (FP64 mode): fused single-pass f+grad partial over a row block of observations.
//
// Replaces, per tile of K1_TP observations and one block of RB factor columns, the reference's
//   Z = V^T A                      pkg/src/momentcp/implicit.py:106   (GEMM1, DMMA.8x8x4)
//   P = nu * Z^(d-1)               pkg/src/momentcp/implicit.py:82-91,106-107 (epilogue, registers)
//   w += sum_l nu_l z_l^d          (= a_j^T y_j, pkg/src/momentcp/implicit.py:139; epilogue)
//   Y += V P                       pkg/src/momentcp/implicit.py:107   (GEMM2, DMMA.8x8x4)
// Z and P live only in registers / shared memory -- the p x r intermediate never reaches HBM.
//
// Layout in HBM: V is observation-major (p_pad x ldv, row l = observation v_l, zero padded to a
// multiple of K1_TP rows and to a 16-byte row pitch).  Each CTA is persistent over a static,
// strided sequence of tiles and owns one RB-column block; its Y partial (n_pad x RB) lives in
// registers across all of its tiles, distributed over 8 warps by 8-row m-tiles of n.  Partials
// are written once per CTA and summed in a fixed order by k_reduce_partials, so results are
// bitwise reproducible and exactly linear in nu (pkg/tests/test_implicit.py:53-57).
#pragma once

#include "mcp_common.cuh"
#include "pdl.h"
#include "k1s_fp64.cuh"   // smem_u32
#include "umma.cuh"       // TMEM helpers
#include "k1x_common.cuh"  // (column block, tile) work split

namespace mcp {

#ifndef MCP_K1_ODD
#define MCP_K1_ODD 0            // 1: GEMM1 even / odd k-step accumulator chains (no gain measured)
#endif

constexpr int K1_TP = 64;       // observations per tile
constexpr int K1_NK = 64;       // n-chunk width staged in shared memory
constexpr int K1_THREADS = 256; // 8 warps
constexpr int K1_SV = 68;       // smem row pitch (elements): 68 = 4 mod 16 -> conflict-free
                                // 8-byte fragment loads for both GEMMs

struct K1Params {
  const void* V;       // p_pad x ldv, observation-major
  int64_t ldv;         // row pitch in elements (multiple of 16 bytes)
  int64_t num_tiles;   // p_pad / K1_TP
  int n;               // variables
  int n_chunks;        // ceil(n / K1_NK)
  int n_pad;           // n_chunks * K1_NK
  const double* nu;    // p_pad weights (zero padded) or nullptr for uniform
  double nu_const;     // uniform weight when nu == nullptr
  const double* Afrag; // [rbs][n_chunks*16][RB/8][32] B-fragment ordered factor blocks
  int d;
  int rbs;             // number of RB-column blocks
  int gp;              // persistent CTAs per column block (K1G: partial slots per block)
  int groups = 0;      // K1G: the k1w_split work split (k1x_common.cuh)
  int64_t t_main = 0;
  double* Ypart;       // [rbs][gp][n_pad][RB]
  double* wpart;       // [rbs][gp][RB]
};

template <typename VT, int RB>
__host__ __device__ constexpr size_t k1_smem_bytes() {
  return 2 * (size_t)K1_TP * K1_SV * sizeof(VT)      // V chunk, double buffered
         + 2 * (size_t)16 * (RB / 8) * 32 * 8        // factor fragments, double buffered
         + (size_t)K1_TP * (RB + 4) * 8              // P tile
         + (size_t)8 * RB * 8;                       // w cross-warp reduction
}

template <typename VT, int THREADS = K1_THREADS>
__device__ __forceinline__ void k1_load_v(VT* dst, const VT* __restrict__ V, int64_t ldv,
                                          int64_t row0, int c) {
  constexpr int SEG = 16 / sizeof(VT);
  constexpr int SEGS_ROW = K1_NK / SEG;
  constexpr int TOTAL = K1_TP * SEGS_ROW;
#pragma unroll
  for (int s = threadIdx.x; s < TOTAL; s += THREADS) {
    const int row = s / SEGS_ROW, seg = s % SEGS_ROW;
    const int64_t col = (int64_t)c * K1_NK + seg * SEG;
    const bool ok = col < ldv;
    const VT* src = ok ? V + (row0 + row) * ldv + col : V;
    cp_async16(dst + row * K1_SV + seg * SEG, src, ok ? 16 : 0);
  }
}

template <typename VT, int THREADS = K1_THREADS>
__device__ __forceinline__ void k1_load_v_hint(VT* dst, const VT* __restrict__ V, int64_t ldv,
                                               int64_t row0, int c, uint64_t policy) {
  constexpr int SEG = 16 / sizeof(VT);
  constexpr int SEGS_ROW = K1_NK / SEG;
  constexpr int TOTAL = K1_TP * SEGS_ROW;
#pragma unroll
  for (int s = threadIdx.x; s < TOTAL; s += THREADS) {
    const int row = s / SEGS_ROW, seg = s % SEGS_ROW;
    const int64_t col = (int64_t)c * K1_NK + seg * SEG;
    const bool ok = col < ldv;
    const VT* src = ok ? V + (row0 + row) * ldv + col : V;
    cp_async16_hint(dst + row * K1_SV + seg * SEG, src, ok ? 16 : 0, policy);
  }
}

template <int NT, int THREADS = K1_THREADS>
__device__ __forceinline__ void k1_load_a(double* dst, const double* __restrict__ src) {
  constexpr int TOTAL = 16 * NT * 32 / 2;
#pragma unroll
  for (int s = threadIdx.x; s < TOTAL; s += THREADS) cp_async16(dst + 2 * s, src + 2 * s, 16);
}

template <typename VT, int RB, int MTW>
__global__ void __launch_bounds__(K1_THREADS) k1_fg_dmma(K1Params prm) {
  pdl_enter();   // the factor fragments come from the preceding prep kernel
  constexpr int NT = RB / 8;
  constexpr int SP = RB + 4;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  VT* sV0 = reinterpret_cast<VT*>(smem_raw);
  VT* sV1 = sV0 + K1_TP * K1_SV;
  double* sA0 = reinterpret_cast<double*>(smem_raw + 2 * (size_t)K1_TP * K1_SV * sizeof(VT));
  double* sA1 = sA0 + 16 * NT * 32;
  double* sP = sA1 + 16 * NT * 32;
  double* sW = sP + K1_TP * SP;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int rb = blockIdx.x % prm.rbs;
  const int pg = blockIdx.x / prm.rbs;
  const int C = prm.n_chunks;
  const int dm1 = prm.d - 1;
  const VT* __restrict__ V = static_cast<const VT*>(prm.V);
  const double* __restrict__ Af = prm.Afrag + (size_t)rb * C * 16 * NT * 32;

  double yacc[MTW][NT][2];
  double wacc[NT][2];
#pragma unroll
  for (int c = 0; c < MTW; ++c)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) yacc[c][nt][0] = yacc[c][nt][1] = 0.0;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) wacc[nt][0] = wacc[nt][1] = 0.0;

  for (int64_t tile = pg; tile < prm.num_tiles; tile += prm.gp) {
    const int64_t row0 = tile * K1_TP;

    // ---------------- GEMM1: Z[64 x RB] = V_tile[64 x n] * A[n x RB] ----------------
    // even / odd k-steps in separate accumulators: 2 NT independent DMMA chains per warp
    double zacc[NT][2], zodd[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) zacc[nt][0] = zacc[nt][1] = zodd[nt][0] = zodd[nt][1] = 0.0;

    k1_load_v<VT>(sV0, V, prm.ldv, row0, 0);
    k1_load_a<NT>(sA0, Af);
    cp_async_commit();
    for (int c = 0; c < C; ++c) {
      VT* sv = (c & 1) ? sV1 : sV0;
      double* sa = (c & 1) ? sA1 : sA0;
      if (c + 1 < C) {
        k1_load_v<VT>((c & 1) ? sV0 : sV1, V, prm.ldv, row0, c + 1);
        k1_load_a<NT>((c & 1) ? sA0 : sA1, Af + (size_t)(c + 1) * 16 * NT * 32);
        cp_async_commit();
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      const VT* vrow = sv + (8 * warp + g) * K1_SV + t;
#pragma unroll
      for (int ks = 0; ks < 16; ks += 2) {
        const double a0 = to_f64(vrow[4 * ks]);
        const double a1 = to_f64(vrow[4 * ks + 4]);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          dmma884(zacc[nt], a0, sa[(ks * NT + nt) * 32 + lane]);
          dmma884(MCP_K1_ODD ? zodd[nt] : zacc[nt], a1, sa[((ks + 1) * NT + nt) * 32 + lane]);
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      zacc[nt][0] += zodd[nt][0];
      zacc[nt][1] += zodd[nt][1];
    }

    // ---------------- epilogue: P = nu * z^(d-1), w += P * z ----------------
    {
      const int lr = 8 * warp + g;
      const double nul = prm.nu ? prm.nu[row0 + lr] : prm.nu_const;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        double pv[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const double z = zacc[nt][e];
          pv[e] = nul * rm_pow(z, dm1);
          wacc[nt][e] += pv[e] * z;
        }
        *reinterpret_cast<double2*>(&sP[lr * SP + 8 * nt + 2 * t]) = make_double2(pv[0], pv[1]);
      }
    }
    __syncthreads();

    // ---------------- GEMM2: Y[n x RB] += V_tile^T[n x 64] * P[64 x RB] ----------------
    // Chunks run last-to-first so the (up to two) chunks still resident from GEMM1 are used
    // before any reload; with n <= 128 the tile is read from HBM exactly once.
#pragma unroll
    for (int cc = 0; cc < MTW; ++cc) {
      const int c = MTW - 1 - cc;
      if (c < C) {
        const VT* sv = (c & 1) ? sV1 : sV0;
        if (c >= 1 && c - 1 <= C - 3) {
          k1_load_v<VT>(((c - 1) & 1) ? sV1 : sV0, V, prm.ldv, row0, c - 1);
          cp_async_commit();
          cp_async_wait<1>();
        } else {
          cp_async_wait<0>();
        }
        __syncthreads();
        const VT* vcol = sv + t * K1_SV + 8 * warp + g;
        const double* prow = sP + t * SP + g;
#pragma unroll 4
        for (int ks = 0; ks < 16; ++ks) {
          const double a = to_f64(vcol[4 * ks * K1_SV]);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) dmma884(yacc[c][nt], a, prow[4 * ks * SP + 8 * nt]);
        }
        __syncthreads();
      }
    }
  }

  // ---------------- write this CTA's partials ----------------
  double* Yp = prm.Ypart + ((size_t)rb * prm.gp + pg) * prm.n_pad * RB;
#pragma unroll
  for (int c = 0; c < MTW; ++c) {
    if (c < C) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
        *reinterpret_cast<double2*>(&Yp[(size_t)(c * K1_NK + 8 * warp + g) * RB + 8 * nt + 2 * t]) =
            make_double2(yacc[c][nt][0], yacc[c][nt][1]);
    }
  }
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      double v = wacc[nt][e];
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      if (g == 0) sW[warp * RB + 8 * nt + 2 * t + e] = v;
    }
  __syncthreads();
  if (threadIdx.x < RB) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < K1_THREADS / 32; ++w) s += sW[w * RB + threadIdx.x];
    prm.wpart[((size_t)rb * prm.gp + pg) * RB + threadIdx.x] = s;
  }
}

// ---------------------------------------------------------------------------------------------
// K1G: the same tile pipeline with the Y partial kept in global memory (L2-resident, one
// n_pad x RB block per CTA, owned element-wise by one thread) instead of registers.  GEMM2
// accumulates each n-chunk of a tile in fresh registers and adds the chunk into the CTA's
// partial right after it (prefetched before the chunk's k-steps), so registers no longer bound
// the column block: RB = 64 for every n (vs RB = 16 at n = 1024 in K1), i.e. 4x fewer passes over
// V for r = 256, and every warp runs NT = RB / 8 independent DMMA chains in both GEMMs.
// The per-tile read-modify-write of the partial is ~1 MB per CTA per tile (~15 GB/s per SM at
// c5), far below L2 bandwidth.  Static tile order per CTA + single-owner elements keep the
// result deterministic.
#ifndef MCP_K1G_HINTS
#define MCP_K1G_HINTS 0   // 1: L2 hints (V evict_first, Y evict_last): -20% DRAM, +3% time
#endif
#ifndef MCP_K1GT_TMEM_CHUNKS
#define MCP_K1GT_TMEM_CHUNKS 64   // cap on K1GT's TMEM-resident chunks (experiments)
#endif
#ifndef MCP_K1G_TMA_RED
#define MCP_K1G_TMA_RED 1   // K1GT's L2 chunks added by bulk tensor reduce-add (0: load + store)
#endif
#ifndef MCP_K1G_G2MAP
#define MCP_K1G_G2MAP 1   // fp32 rows: conflict-free GEMM2 row map (experiment builds: 0)
#endif
#define K1G_LOAD_V(dst, V, ldv, row0, c)                                       \
  (MCP_K1G_HINTS ? k1_load_v_hint<VT, THREADS>(dst, V, ldv, row0, c, pol_v) \
                 : k1_load_v<VT, THREADS>(dst, V, ldv, row0, c))

template <typename VT, int RB>
__host__ __device__ constexpr int k1g_sp() {
  return (MCP_K1G_G2MAP && sizeof(VT) == 4) ? RB + 2 : RB + 4;
}
template <typename VT, int RB, bool TM = false>
__host__ __device__ constexpr size_t k1g_smem_bytes() {
  return 2 * (size_t)K1_TP * K1_SV * sizeof(VT) + 2 * (size_t)16 * (RB / 8) * 32 * 8 +
         (size_t)K1_TP * k1g_sp<VT, RB>() * 8 + (size_t)8 * RB * 8 +
         (TM && MCP_K1G_TMA_RED ? 128 + (size_t)8 * 8 * RB * 8 : 0);   // K1GT L2-chunk staging
}

// bulk tensor reduce-add (TMA, performed at L2) of a shared-memory box into global memory
__device__ __forceinline__ void k1g_bulk_reduce_add_2d(const CUtensorMap* tm, int c0, int c1,
                                                       const void* src) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];\n"
      "cp.async.bulk.commit_group;\n" ::"l"(tm),
      "r"(c0), "r"(c1), "r"((uint32_t)__cvta_generic_to_shared(src))
      : "memory");
}

// K1G with TM = true ("K1GT"): the Y partial lives in tensor memory instead of L2 -- all of it
// when n_chunks * RB <= 512, else (RB = 64 at n = 1024, the c5 default) chunks 0-7 in TMEM and
// the rest in L2: half K1G's L2 working set, which then stays resident.  Measured at c5 (one
// box, back to back): K1G 633 ms / 845 W / DRAM 14.3x V; K1GT RB = 32 657 ms / 669 W / 1.0x;
// K1GT RB = 64 half-and-half 625.5 ms / 741 W / 1.4x (profiles/r02/ab_c5_k1gt_half.txt).  The L2
// chunks are then added by one bulk tensor reduce-add per warp and chunk (the warp's 8 x RB result
// staged in shared memory; the add happens at L2, no load of the previous value): 611.5 ms, 684 W
// (profiles/r02/ab_c5_k1gt_tmared.txt; 0 or 4 TMEM chunks instead of 8 measured 646 / 628 ms).  TMEM is
// used as private per-thread storage (fp64 as two 32-bit columns): thread (warp w, lane L) owns
// TMEM lane 32 (w % 4) + L, columns [256 (w / 4), 256 (w / 4) + 256) -- 128 doubles, i.e. the
// 2 NT doubles of each of the n_chunks GEMM2 accumulators it owns (n_chunks * RB <= 512: c5's
// n = 1024 runs RB = 32).  Per chunk the previous partial is read with one tcgen05.ld before the
// k-steps and written back with one tcgen05.st after them: the read-modify-write that spilled
// from L2 to DRAM at c5 (14x the V bytes, ncu round 1) stays on chip, and the sum order per
// element is K1G's (acc + prev, tile by tile), so the partials are the same arithmetic.
// NW = 8 or 16 warps.  With 16 the warps split the column block in halves: warp w owns row
// block / GEMM2 m-tile w % 8 and the NTW = NT / 2 column tiles starting at 8 NTW (w / 8) in both
// GEMMs (4 warps per sub-partition instead of 2, each with half the DMMA chains).
template <typename VT, int RB, bool TM, int NW = 8>
__global__ void __launch_bounds__(NW * 32, 1) k1g_fg_dmma(K1Params prm,
                                                          const __grid_constant__ CUtensorMap tm_y) {
  pdl_enter();   // the factor fragments come from the preceding prep kernel
  constexpr int THREADS = NW * 32;
  constexpr int NT = RB / 8;
  constexpr int NTW = NT / (NW / 8);     // column tiles per warp
  constexpr int TCOLS = 512 / (NW / 4);  // TMEM columns per thread (K1GT)
  static_assert(NW == 8 || NW == 16, "K1G: 8 or 16 warps");
  static_assert(NTW >= 1, "K1G: column block too narrow for the warp split");
  static_assert(!TM || NTW == 2 || NTW == 4 || NTW == 8, "K1GT: 8 / 16 / 32 TMEM columns per chunk");
  // P row pitch (doubles): == 4 (mod 16) for fp64 rows (GEMM2 k index = tile row 4 ks + t), == 2
  // (mod 16) for fp32 rows, whose GEMM2 k index runs over tile rows 8 (ks >> 1) + 2 t + (ks & 1):
  // the 4-byte V fragment loads then hit bank 8 t + g (+ const), all 32 distinct, where 4 ks + t
  // gave a 2-way conflict on every load (ncu at c5: 150-257M per launch)
  constexpr int SP = k1g_sp<VT, RB>();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  VT* sV0 = reinterpret_cast<VT*>(smem_raw);
  VT* sV1 = sV0 + K1_TP * K1_SV;
  double* sA0 = reinterpret_cast<double*>(smem_raw + 2 * (size_t)K1_TP * K1_SV * sizeof(VT));
  double* sA1 = sA0 + 16 * NT * 32;
  double* sP = sA1 + 16 * NT * 32;
  double* sW = sP + K1_TP * SP;
  // K1GT's L2 chunks: each warp stages its 8 x RB GEMM2 result (fp64) and adds it into the
  // partial with one bulk tensor reduce-add -- no load of the previous value, the add at L2
  constexpr bool kTmaRed = TM && MCP_K1G_TMA_RED && NW == 8;
  double* sStg = reinterpret_cast<double*>(
      (reinterpret_cast<uintptr_t>(sW + 8 * RB) + 127) & ~(uintptr_t)127);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wr = warp & 7;               // row block (GEMM1) / m-tile (GEMM2)
  const int nt0 = NTW * (warp >> 3);     // first column tile of this warp
  const int C = prm.n_chunks;
  const int dm1 = prm.d - 1;
  const VT* __restrict__ V = static_cast<const VT*>(prm.V);
  // the (column block, tile) work split shared with K1X (k1x_common.cuh): groups of one CTA per
  // column block stride the main tiles together, leftover CTAs take block-major tail ranges
  K1WParams wp;
  wp.num_tiles = prm.num_tiles;
  wp.rbs = prm.rbs;
  wp.nclusters = (int)gridDim.x;
  wp.groups = prm.groups;
  wp.t_main = prm.t_main;
  wp.slots = prm.gp;
  wp.n_pad = prm.n_pad;
  wp.Ypart = prm.Ypart;
  wp.wpart = prm.wpart;
  constexpr bool kF32 = MCP_K1G_G2MAP && sizeof(VT) == 4;
  const int g2row = kF32 ? 2 * t : t;   // GEMM2 fragment row of k-step 0

  double wacc[NTW][2];
#pragma unroll
  for (int nt = 0; nt < NTW; ++nt) wacc[nt][0] = wacc[nt][1] = 0.0;
  bool first = true;
  // V streams through L2 (evict first); the CTA's Y partial should stay there (evict last)
  const uint64_t pol_v = MCP_K1G_HINTS ? l2_policy_evict_first() : 0;
  const uint64_t pol_y = MCP_K1G_HINTS ? l2_policy_evict_last() : 0;
  __shared__ uint32_t s_tmem;
  uint32_t tme = 0;   // this thread's TMEM base (lane in bits 31..16, column below)
  if constexpr (TM) {
    if (warp == 0) tmem_alloc<512>(smem_u32(&s_tmem));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    tme = s_tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(TCOLS * (warp >> 2));
  }

  // K1GT: chunks [0, CT) of the partial live in TMEM, the rest (RB = 64 at n = 1024: half of
  // it) in L2 -- half the L2 working set of K1G, which then stays resident
  const int CT = TM ? min(min(C, TCOLS / (4 * NTW)), MCP_K1GT_TMEM_CHUNKS) : 0;
  K1WTile ti;
  for (int64_t k = 0; k1w_tile_at(wp, blockIdx.x, k, ti); ++k) {
    const int64_t row0 = ti.tile * K1_TP;
    const double* __restrict__ Af = prm.Afrag + (size_t)ti.rb * C * 16 * NT * 32;
    double* __restrict__ Yp = prm.Ypart + ((size_t)ti.rb * prm.gp + ti.slot) * prm.n_pad * RB;

    // ---------------- GEMM1: Z[64 x RB] = V_tile[64 x n] * A[n x RB] ----------------
    double zacc[NTW][2];
#pragma unroll
    for (int nt = 0; nt < NTW; ++nt) zacc[nt][0] = zacc[nt][1] = 0.0;
    K1G_LOAD_V(sV0, V, prm.ldv, row0, 0);
    k1_load_a<NT, THREADS>(sA0, Af);
    cp_async_commit();
    for (int c = 0; c < C; ++c) {
      VT* sv = (c & 1) ? sV1 : sV0;
      double* sa = (c & 1) ? sA1 : sA0;
      if (c + 1 < C) {
        K1G_LOAD_V((c & 1) ? sV0 : sV1, V, prm.ldv, row0, c + 1);
        k1_load_a<NT, THREADS>((c & 1) ? sA0 : sA1, Af + (size_t)(c + 1) * 16 * NT * 32);
        cp_async_commit();
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      const VT* vrow = sv + (8 * wr + g) * K1_SV + t;
#pragma unroll
      for (int ks = 0; ks < 16; ++ks) {
        const double a = to_f64(vrow[4 * ks]);
#pragma unroll
        for (int nt = 0; nt < NTW; ++nt)
          dmma884(zacc[nt], a, sa[(ks * NT + nt0 + nt) * 32 + lane]);
      }
      __syncthreads();
    }

    // ---------------- epilogue: P = nu * z^(d-1), w += P * z ----------------
    {
      const int lr = 8 * wr + g;
      const double nul = prm.nu ? prm.nu[row0 + lr] : prm.nu_const;
#pragma unroll
      for (int nt = 0; nt < NTW; ++nt) {
        double pv[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const double z = zacc[nt][e];
          pv[e] = nul * rm_pow(z, dm1);
          wacc[nt][e] += pv[e] * z;
        }
        *reinterpret_cast<double2*>(&sP[lr * SP + 8 * (nt0 + nt) + 2 * t]) =
            make_double2(pv[0], pv[1]);
      }
    }
    __syncthreads();

    // ---------------- GEMM2, chunk by chunk, last to first ----------------
    // the previous tile's reduce-adds have completed before this tile's (fixed add order)
    if (kTmaRed && !first && lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
    for (int c = C - 1; c >= 0; --c) {
      const VT* sv = (c & 1) ? sV1 : sV0;
      if (c >= 1 && c - 1 <= C - 3) {
        K1G_LOAD_V(((c - 1) & 1) ? sV1 : sV0, V, prm.ldv, row0, c - 1);
        cp_async_commit();
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      double* yrow = Yp + (size_t)(c * K1_NK + 8 * wr + g) * RB + 8 * nt0 + 2 * t;
      double2 prev[NTW];
      uint32_t tprev[4 * NTW];
      const bool in_tm = c < CT;   // uniform across the CTA
      if constexpr (TM) {
        if (in_tm && !first) tmem_ld_nowait<4 * NTW>(tme + 4 * NTW * c, tprev);
      }
      if (!in_tm && !first && !kTmaRed) {
#pragma unroll
        for (int nt = 0; nt < NTW; ++nt)
          prev[nt] = MCP_K1G_HINTS
                         ? ld_l2_hint(reinterpret_cast<const double2*>(yrow + 8 * nt), pol_y)
                         : *reinterpret_cast<const double2*>(yrow + 8 * nt);
      }
      double acc[NTW][2];
#pragma unroll
      for (int nt = 0; nt < NTW; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
      const VT* vcol = sv + g2row * K1_SV + 8 * wr + g;
      const double* prow = sP + g2row * SP + 8 * nt0 + g;
#pragma unroll 4
      for (int ks = 0; ks < 16; ++ks) {
        const int kr = kF32 ? 8 * (ks >> 1) + (ks & 1) : 4 * ks;   // + g2row: this lane's row
        const double a = to_f64(vcol[kr * K1_SV]);
#pragma unroll
        for (int nt = 0; nt < NTW; ++nt) dmma884(acc[nt], a, prow[kr * SP + 8 * nt]);
      }
      if (TM && in_tm) {
        if (!first) tmem_ld_wait();
        uint32_t tout[4 * NTW];
#pragma unroll
        for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            double o = acc[nt][e];
            if (!first)
              o += __hiloint2double((int)tprev[4 * nt + 2 * e + 1], (int)tprev[4 * nt + 2 * e]);
            tout[4 * nt + 2 * e] = (uint32_t)__double2loint(o);
            tout[4 * nt + 2 * e + 1] = (uint32_t)__double2hiint(o);
          }
        tmem_st<4 * NTW>(tme + 4 * NTW * c, tout);
      } else if (kTmaRed && !first) {
        double* stg = sStg + (size_t)warp * 8 * RB;   // [8 rows][RB]
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
        __syncwarp();
#pragma unroll
        for (int nt = 0; nt < NTW; ++nt)
          *reinterpret_cast<double2*>(stg + g * RB + 8 * (nt0 + nt) + 2 * t) =
              make_double2(acc[nt][0], acc[nt][1]);
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
        if (lane == 0)
          k1g_bulk_reduce_add_2d(&tm_y, 0,
                                 (int)(((size_t)ti.rb * prm.gp + ti.slot) * prm.n_pad +
                                       c * K1_NK + 8 * wr),
                                 stg);
      } else {
#pragma unroll
        for (int nt = 0; nt < NTW; ++nt) {
          double2 o = make_double2(acc[nt][0], acc[nt][1]);
          if (!first) {
            o.x += prev[nt].x;
            o.y += prev[nt].y;
          }
          if (MCP_K1G_HINTS)
            st_l2_hint(reinterpret_cast<double2*>(yrow + 8 * nt), o, pol_y);
          else
            *reinterpret_cast<double2*>(yrow + 8 * nt) = o;
        }
      }
      __syncthreads();
    }
    if constexpr (TM) tmem_st_wait();   // this tile's partial is in TMEM before the next reads it
    // a segment's first plain stores are seen by the later reduce-adds (async proxy)
    if (kTmaRed && first) asm volatile("fence.proxy.async.global;\n" ::: "memory");
    first = false;

    if (ti.last_in_seg) {
      // ---------------- segment end: this slot's partials leave the CTA ----------------
      if constexpr (TM) {
        for (int c = 0; c < CT; ++c) {
          uint32_t tv[4 * NTW];
          tmem_ld_nowait<4 * NTW>(tme + 4 * NTW * c, tv);
          tmem_ld_wait();
          double* yrow = Yp + (size_t)(c * K1_NK + 8 * wr + g) * RB + 8 * nt0 + 2 * t;
#pragma unroll
          for (int nt = 0; nt < NTW; ++nt)
            *reinterpret_cast<double2*>(yrow + 8 * nt) =
                make_double2(__hiloint2double((int)tv[4 * nt + 1], (int)tv[4 * nt]),
                             __hiloint2double((int)tv[4 * nt + 3], (int)tv[4 * nt + 2]));
        }
      }
#pragma unroll
      for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          double v = wacc[nt][e];
          v += __shfl_xor_sync(0xffffffffu, v, 4);
          v += __shfl_xor_sync(0xffffffffu, v, 8);
          v += __shfl_xor_sync(0xffffffffu, v, 16);
          if (g == 0) sW[wr * RB + 8 * (nt0 + nt) + 2 * t + e] = v;
          wacc[nt][e] = 0.0;
        }
      __syncthreads();
      if (threadIdx.x < RB) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) s += sW[w * RB + threadIdx.x];   // row blocks in order
        prm.wpart[((size_t)ti.rb * prm.gp + ti.slot) * RB + threadIdx.x] = s;
      }
      __syncthreads();
      first = true;
    }
  }
  if (kTmaRed && lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
  // partial slots no CTA writes (blocks touched by fewer leftover CTAs) are zero
  k1w_zero_holes<THREADS, RB>(wp, blockIdx.x, 0, prm.n_pad, true);
  if constexpr (TM) {
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc<512>(s_tmem);
  }
}

}  // namespace mcp
