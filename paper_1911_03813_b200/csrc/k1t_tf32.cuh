// K1T (fast mode, mode = "tf32x3"): fused f+grad partial on the 5th-gen tensor cores.
//
// Same algebra as K1 (reference pkg/src/momentcp/implicit.py:94-107) on 128-observation tiles:
//   GEMM1  Z[128 x RB] = V_tile[128 x n] A[n x RB]          tcgen05.mma kind::tf32, D in TMEM
//   epi    P = nu * Z^(d-1)  (fp64 arithmetic, stored as TF32 hi/lo bricks in shared memory)
//   GEMM2  Y[n x RB] += V_tile^T P                           tcgen05.mma kind::tf32, D in TMEM
// Roofline note: both operands come from shared memory (SS mode) and TMEM capacity caps the
// column block at RB <= 64 (Y needs (n/128) x RB TMEM columns), so each 3xTF32 k-step re-reads
// A and B three times: ~136 KB of smem traffic per 32-wide k-step against 128 B/clk/SM.  The
// kernel is shared-memory-bandwidth bound well below the TF32 tensor peak; TMEM-sourced A
// operands (tcgen05.cp) and 2-CTA pairs are the next step.
// Every product is the 3xTF32 split  x*y ~= xh*yh + xh*yl + xl*yh  (xh = top 10 mantissa bits,
// xl = x - xh), so the result carries ~1e-7 relative error instead of TF32's 1e-3 (SURVEY.md
// Appendix B); Z and P never reach HBM.  Y accumulates in fp32 TMEM for K1T_FLUSH tiles and is
// then flushed into an fp64 per-CTA partial (fixed order, deterministic); w = a_j^T y_j is formed
// from the reduced Y in fp64 by the tail (implicit.py:139).
//
// Roles (one CTA per SM, 10 warps): warp 0 = TMA producer (one lane), warp 1 = MMA issuer (one
// lane; also owns TMEM alloc), warps 2..9 = split / epilogue / flush.  V is read twice per tile
// through two tensor maps over the same fp32 rows: pass 1 with SWIZZLE_128B (K-major operand of
// GEMM1), pass 2 with SWIZZLE_128B_ATOM_32B (the MN-major operand GEMM2 needs -- the only layout
// tcgen05 accepts for MN-major TF32).  Stage ring: full (TMA) -> split (hi/lo by CUDA cores) ->
// empty (MMA commit).
#pragma once

#include <cuda.h>

#include "k1s_fp64.cuh"  // mbarrier helpers
#include "mcp_common.cuh"
#include "umma.cuh"

namespace mcp {

constexpr int K1T_TP = 128;
constexpr int K1T_MATH_WARPS = 8;
constexpr int K1T_THREADS = (2 + K1T_MATH_WARPS) * 32;
constexpr int K1T_VBYTES = 16384;  // V region of one stage (128 rows x 32 or 4 x 32 rows x 32)
constexpr int K1T_FLUSH = 8;       // tiles accumulated in fp32 TMEM between fp64 flushes

struct K1TParams {
  int n, r, d;
  int nkb;            // GEMM1 k-blocks of 32 variables
  int mt2;            // GEMM2 m-tiles of 128 variables
  int RB;             // factor columns per CTA (16, 32 or 64)
  int rbs, gp;
  int r_pad;          // rows of the hi half of the prepared A^T (lo half starts there)
  int stages;
  int64_t num_tiles;  // p_pad / 128
  const double* nu;
  double nu_const;
  double* Ypart;      // [rbs][gp][mt2*128][RB] fp64
  int zcat = 0;       // K1T2: GEMM1 as V_hi x [A_hi ; A_lo] (N = 2 RB) + V_lo x A_hi: Z takes
                      // 2 RB TMEM columns per buffer and the epilogue adds its two halves
  int serial = 0;     // K1T2: GEMM2(u) right after GEMM1(u) (reuse distance one tile) instead of
                      // GEMM1(u + 1) first (epilogue hidden, reuse distance two tiles)
  int hint = 0;       // K1T2: L2 policy -- GEMM1's V reads evict_last, everything else evict_first
  int flush = 8;      // K1T2: tiles accumulated in fp32 TMEM between fp64 flushes
  int g2_3d = 0;      // K1T2: tm_v2 / tm_l2 are 3-D chunk maps (one TMA per 16 KB operand)
  int g2x2 = 0;       // K1T2: GEMM2 as V P_hi (2 products) with P_hi rounded to nearest; the
                      // dropped V_hi P_lo term is unbiased and <= 2^-12 of each product
  int drain_tma = 0;  // K1T2: transient m-tiles drain by bulk tensor reduce-add (TMA) from a
                      // 2 KB staging slot per epilogue warp instead of per-element REDs
  int tr_wide = 0;    // K1T2: the (single) transient m-tile is wide (2 RB columns = all of Z):
                      // c3 runs every GEMM2 m-tile as the N = 2 RB [P_hi | P_lo] product
  int mt_tr = 0;      // K1T2 (serial, zcat): the last mt_tr GEMM2 m-tiles accumulate in the Z
                      // columns (free once the epilogue has read Z), run first in GEMM2's order
                      // and drain into the fp64 partial every tile -- RB = 64 where the
                      // persistent Y would not fit TMEM (c5: 128 + 6 x 64 = 512 columns)
  int insplit = 0;    // K1T2: V_lo = V - tf32(V) formed in shared memory by 4 splitter warps
                      // from the one TMA'd fp32 stage (no V_lo copy in HBM, DRAM ~1x V)
  int wide = 0;       // K1T2: GEMM2 m-tiles [0, wide) run V_hi [P_hi | P_lo] as ONE N = 2 RB
                      // product into two TMEM halves (spare columns), the V_hi operand read once
};

__host__ __device__ constexpr size_t k1t_stage_bytes(int RB) { return 2 * K1T_VBYTES + 256 * RB; }
__host__ __device__ constexpr size_t k1t_smem_bytes(int RB, int stages, bool drain_tma = false) {
  return 1024 /*align slack*/ + stages * k1t_stage_bytes(RB) + 1024 * (size_t)RB /*P hi+lo*/ +
         1024 /*barriers*/ + (drain_tma ? 8 * 2048 : 0) /*K1T2 drain staging*/;
}

__global__ void __launch_bounds__(K1T_THREADS, 1)
    k1t_fg_tf32(const __grid_constant__ CUtensorMap tm_v1, const __grid_constant__ CUtensorMap tm_v2,
                const __grid_constant__ CUtensorMap tm_a, K1TParams prm) {
  extern __shared__ __align__(16) unsigned char smem_raw_t[];
  // 1 KB alignment by an offset on the shared array itself, so the compiler keeps the shared
  // address space (LDS/STS, not generic loads) for everything derived from `base`
  unsigned char* base = smem_raw_t + ((1024u - (smem_u32(smem_raw_t) & 1023u)) & 1023u);
  const int RB = prm.RB, NS = prm.stages;
  const size_t SB = k1t_stage_bytes(RB);
  unsigned char* sPh = base + NS * SB;                 // 4 bricks x RB rows x 128 B
  unsigned char* sPl = sPh + 512 * RB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sPl + 512 * RB);
  uint64_t* full = bars;
  uint64_t* empty = bars + NS;
  uint64_t* split = bars + 2 * NS;
  uint64_t* z_full = bars + 3 * NS;
  uint64_t* p_full = z_full + 1;
  uint64_t* p_empty = z_full + 2;
  uint64_t* y_full = z_full + 3;
  uint64_t* y_empty = z_full + 4;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(z_full + 5);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rb = blockIdx.x % prm.rbs;
  const int pg = blockIdx.x / prm.rbs;
  const int64_t my_tiles =
      pg < prm.num_tiles ? (prm.num_tiles - pg + prm.gp - 1) / prm.gp : 0;
  const int mt2 = prm.mt2, nkb = prm.nkb;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&split[s], K1T_MATH_WARPS);
    }
    mbar_init(z_full, 1);
    mbar_init(p_full, K1T_MATH_WARPS);
    mbar_init(p_empty, 1);
    mbar_init(y_full, 1);
    mbar_init(y_empty, K1T_MATH_WARPS);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) tmem_alloc<512>(smem_u32(tslot));
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_v1);
    tma_prefetch_desc(&tm_v2);
    tma_prefetch_desc(&tm_a);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t tz = tmem;            // Z: columns [0, RB)
  const uint32_t ty = tmem + RB;       // Y[mt]: columns RB * (1 + mt)

  if (warp == 0) {
    // =========================== TMA producer ===========================
    if (lane == 0) {
      int64_t q = 0;
      for (int64_t u = 0; u < my_tiles; ++u) {
        const int row0 = (int)((pg + u * prm.gp) * K1T_TP);
        for (int step = 0; step < nkb + 4 * mt2; ++step, ++q) {
          const int s = (int)(q % NS);
          if (q >= NS) mbar_wait(&empty[s], (uint32_t)((q / NS) - 1) & 1);
          unsigned char* st = base + s * SB;
          if (step < nkb) {
            mbar_arrive_expect_tx(&full[s], K1T_VBYTES + 256 * RB);
            tma_load_2d(st, &tm_v1, step * 32, row0, smem_u32(&full[s]));
            tma_load_2d(st + 2 * K1T_VBYTES, &tm_a, step * 32, rb * RB, smem_u32(&full[s]));
            tma_load_2d(st + 2 * K1T_VBYTES + 128 * RB, &tm_a, step * 32, prm.r_pad + rb * RB,
                        smem_u32(&full[s]));
          } else {
            const int mt = (step - nkb) >> 2, rc = (step - nkb) & 3;
            mbar_arrive_expect_tx(&full[s], K1T_VBYTES);
#pragma unroll
            for (int b = 0; b < 4; ++b)
              tma_load_2d(st + b * 4096, &tm_v2, mt * 128 + b * 32, row0 + rc * 32,
                          smem_u32(&full[s]));
          }
        }
      }
    }
  } else if (warp == 1) {
    // =========================== MMA issuer ===========================
    if (lane == 0) {
      const uint32_t id1 = umma_idesc_tf32(128, RB, false, false);
      const uint32_t id2 = umma_idesc_tf32(128, RB, true, false);
      int64_t q = 0;
      int flushes = 0;
      bool fresh = true, wait_y = false;
      for (int64_t u = 0; u < my_tiles; ++u) {
        // ---- GEMM1: Z = V A (3xTF32) ----
        for (int kb = 0; kb < nkb; ++kb, ++q) {
          const int s = (int)(q % NS);
          mbar_wait(&split[s], (uint32_t)(q / NS) & 1);
          tc_fence_after();
          unsigned char* st = base + s * SB;
          const uint32_t v_hi = smem_u32(st), v_lo = v_hi + K1T_VBYTES;
          const uint32_t a_hi = v_hi + 2 * K1T_VBYTES, a_lo = a_hi + 128 * RB;
#pragma unroll
          for (int pr = 0; pr < 3; ++pr) {
            const uint32_t av = pr == 2 ? v_lo : v_hi, bv = pr == 1 ? a_lo : a_hi;
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
              umma_tf32(tz, umma_desc_sw128(av + ks * 32, 16, 1024),
                        umma_desc_sw128(bv + ks * 32, 16, 1024), id1,
                        (kb | pr | ks) != 0 ? 1u : 0u);
          }
          umma_commit(smem_u32(&empty[s]));
        }
        umma_commit(smem_u32(z_full));
        // ---- GEMM2: Y += V^T P (3xTF32), P from the epilogue ----
        mbar_wait(p_full, (uint32_t)u & 1);
        if (wait_y) {
          mbar_wait(y_empty, (uint32_t)(flushes - 1) & 1);
          wait_y = false;
          fresh = true;
        }
        tc_fence_after();
        const uint32_t p_hi = smem_u32(sPh), p_lo = smem_u32(sPl);
        for (int step = 0; step < 4 * mt2; ++step, ++q) {
          const int mt = step >> 2, rc = step & 3;
          const int s = (int)(q % NS);
          mbar_wait(&split[s], (uint32_t)(q / NS) & 1);
          tc_fence_after();
          const uint32_t v_hi = smem_u32(base + s * SB), v_lo = v_hi + K1T_VBYTES;
#pragma unroll
          for (int pr = 0; pr < 3; ++pr) {
            const uint32_t av = pr == 2 ? v_lo : v_hi;
            const uint32_t bv = (pr == 1 ? p_lo : p_hi) + rc * 128 * RB;
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
              umma_tf32(ty + mt * RB, umma_desc_sw128_32b(av + ks * 1024, 4096, 512),
                        umma_desc_sw128(bv + ks * 32, 16, 1024), id2,
                        (fresh && rc == 0 && pr == 0 && ks == 0) ? 0u : 1u);
          }
          umma_commit(smem_u32(&empty[s]));
        }
        fresh = false;
        umma_commit(smem_u32(p_empty));
        if ((u % K1T_FLUSH) == K1T_FLUSH - 1 || u == my_tiles - 1) {
          umma_commit(smem_u32(y_full));
          ++flushes;
          wait_y = true;
        }
      }
    }
  } else {
    // =========================== split / epilogue / flush warps ===========================
    const int mw = warp - 2;                 // 0..7
    const int sp = warp & 3;                 // TMEM sub-partition this warp may access
    const int half = mw >> 2;                // column half for the epilogue / flush
    const int mtid = mw * 32 + lane;         // 0..255
    const int l = 32 * sp + lane;            // tile row (TMEM lane) this thread owns
    // columns per warp for the epilogue / flush: halves of RB, at least one 16-column load
    const int hc = RB >= 32 ? RB / 2 : 16;
    const bool col_active = half * hc < RB;
    const int dm1 = prm.d - 1;
    int64_t q = 0;
    int flushes = 0;
    double* Yp = prm.Ypart + ((size_t)rb * prm.gp + pg) * (size_t)mt2 * 128 * RB;

    auto split_stage = [&](int64_t qq) {
      const int s = (int)(qq % NS);
      mbar_wait(&full[s], (uint32_t)(qq / NS) & 1);
      float4* vh = reinterpret_cast<float4*>(base + s * SB);
      float4* vl = reinterpret_cast<float4*>(base + s * SB + K1T_VBYTES);
#pragma unroll
      for (int k = 0; k < K1T_VBYTES / 16 / 256; ++k) {
        const int e = mtid + 256 * k;
        float4 x = vh[e];
        float4 hi = make_float4(tf32_hi(x.x), tf32_hi(x.y), tf32_hi(x.z), tf32_hi(x.w));
        vl[e] = make_float4(x.x - hi.x, x.y - hi.y, x.z - hi.z, x.w - hi.w);
        vh[e] = hi;
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&split[s]);
    };

    for (int64_t u = 0; u < my_tiles; ++u) {
      const int64_t row0 = (pg + u * prm.gp) * K1T_TP;
      for (int kb = 0; kb < nkb; ++kb, ++q) split_stage(q);

      // ---- epilogue: P = nu z^(d-1) -> TF32 hi/lo bricks (K-major B operand of GEMM2) ----
      mbar_wait(z_full, (uint32_t)u & 1);
      if (u > 0) mbar_wait(p_empty, (uint32_t)(u - 1) & 1);
      tc_fence_after();
      {
        const double nul = prm.nu ? prm.nu[row0 + l] : prm.nu_const;
        const int brick = l >> 5, col = l & 31;
        for (int c0 = half * hc; col_active && c0 < (half + 1) * hc; c0 += 16) {
          float zv[16];
          tmem_ld16(tz + ((uint32_t)(32 * sp) << 16) + c0, zv);
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) {
            const double z = (double)zv[jj];
            const float pf = (float)(nul * rm_pow(z, dm1));
            const float ph = tf32_hi(pf);
            const uint32_t off = brick * 128 * RB + brick_off(c0 + jj, col);
            *reinterpret_cast<float*>(sPh + off) = ph;
            *reinterpret_cast<float*>(sPl + off) = pf - ph;
          }
        }
      }
      fence_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);

      for (int step = 0; step < 4 * mt2; ++step, ++q) split_stage(q);

      // ---- flush: fp32 TMEM Y -> fp64 per-CTA partial (fixed order) ----
      if ((u % K1T_FLUSH) == K1T_FLUSH - 1 || u == my_tiles - 1) {
        mbar_wait(y_full, (uint32_t)flushes & 1);
        tc_fence_after();
        for (int mt = 0; mt < mt2; ++mt) {
          double* yrow = Yp + ((size_t)mt * 128 + l) * RB;
          for (int c0 = half * hc; col_active && c0 < (half + 1) * hc; c0 += 16) {
            float yv[16];
            tmem_ld16(ty + mt * RB + ((uint32_t)(32 * sp) << 16) + c0, yv);
#pragma unroll
            for (int jj = 0; jj < 16; ++jj)
              yrow[c0 + jj] = (flushes == 0 ? 0.0 : yrow[c0 + jj]) + (double)yv[jj];
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(y_empty);
        ++flushes;
      }
    }
    // CTAs without tiles still own a (zero) partial
    if (my_tiles == 0)
      for (int mt = 0; mt < mt2; ++mt)
        for (int c = half * hc; col_active && c < (half + 1) * hc; ++c)
          Yp[((size_t)mt * 128 + l) * RB + c] = 0.0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

// Prepared factor operand for K1T: At[h][j][i] (h = 0 hi, 1 lo), fp32, zero padded to
// r_pad rows and kpad = nkb*32 columns; the TF32 split of the fp32 rounding of A (fp64).
// hi_full = 1 (K1T2 with the in-kernel split): the hi half holds the fp32 value itself -- the
// tensor core reads it as its TF32 truncation, and the splitter warps form lo from it in shared
// memory, so only the hi half is streamed.
__global__ void k_prep_at_tf32(const double* __restrict__ A, int n, int r, int r_pad, int kpad,
                               float* __restrict__ At, int hi_full = 0) {
  const int64_t total = (int64_t)r_pad * kpad;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int j = idx / kpad, i = idx % kpad;
    const float a = (i < n && j < r) ? (float)A[(int64_t)j * n + i] : 0.0f;
    const float hi = tf32_hi(a);
    At[idx] = hi_full ? a : hi;
    At[total + idx] = a - hi;
  }
}

// Fast mode: w_j = a_j^T y_j from the reduced Y (implicit.py:139), fp64.
__global__ void k_w_from_y(const double* __restrict__ A, int n, int r, double* __restrict__ Yw) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= r) return;
  double s = 0.0;
  for (int i = lane; i < n; i += 32) s += A[(int64_t)warp * n + i] * Yw[(int64_t)warp * n + i];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) Yw[(int64_t)n * r + warp] = s;
}

// fp64 -> fp32 observation copy (fast mode on float64 data)
__global__ void k_f64_to_f32(const double* __restrict__ src, float* __restrict__ dst, int64_t rows,
                             int64_t ld_src, int64_t ld_dst, int64_t cols) {
  const int64_t total = rows * ld_dst;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rr = idx / ld_dst, c = idx % ld_dst;
    dst[idx] = c < cols ? (float)src[rr * ld_src + c] : 0.0f;
  }
}

// ---------------------------------------------------------------------------------------------
// K1T2: the fast-mode kernel without the CUDA-core split on the critical path.  The low halves
// V_lo = V - tf32(V) are computed ONCE per observation set (k_split_lo, kept in HBM next to the
// fp32 rows: +1x V of memory, c5 65.5 -> 131 GB) and streamed by TMA like V itself; the tensor
// core truncates the fp32 rows to TF32 on read, so the resident fp32 V doubles as V_hi.
// Tile order (prm.serial, the default): GEMM1(u), epilogue(u), GEMM2(u) with one Z buffer, so
// GEMM2 re-reads the V / V_lo tile GEMM1 just streamed while it is still in L2 (L2 policies:
// GEMM1's reads evict_last, GEMM2's evict_first) -- DRAM sees V + V_lo once.  The look-ahead
// order (serial = 0: Z double-buffered, GEMM1(u + 1) before GEMM2(u)) hides the epilogue but
// holds two tiles per SM between the reads, more than L2, and measured slower once the epilogue
// was vectorised (~2k cycles per tile).  The fp32 Y drains into the fp64 partial every
// prm.flush tiles, under the next GEMM1.
// Roles: warp 0 TMA producer, warp 1 MMA issuer + TMEM owner, warps 2..9 epilogue / flush (two
// per TMEM sub-partition, each on half of the columns).  TMEM: Z (one or two buffers, 2 RB
// columns each with zcat), then Y[mt]: (zbufs * ZW / RB + n/128) RB <= 512 columns.
// bulk tensor reduce-add (TMA, performed at L2) of a shared-memory box into global memory
__device__ __forceinline__ void k1t_bulk_reduce_add_2d(const CUtensorMap* tm, int c0, int c1,
                                                       const void* src) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];\n"
      "cp.async.bulk.commit_group;\n" ::"l"(tm),
      "r"(c0), "r"(c1), "r"((uint32_t)__cvta_generic_to_shared(src))
      : "memory");
}
__device__ __forceinline__ void k1t_bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}
__device__ __forceinline__ void k1t_bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

constexpr int K1T2_EPI_WARPS = 8;
constexpr int K1T2_THREADS = (2 + K1T2_EPI_WARPS) * 32;
constexpr int K1T2_SPLIT_WARPS = 4;                                   // prm.insplit
constexpr int K1T2_THREADS_S = K1T2_THREADS + K1T2_SPLIT_WARPS * 32;
#ifndef MCP_K1T2_ASPLIT
#define MCP_K1T2_ASPLIT 0   // 1: the factor's lo rows formed in smem too (measured 5.21 vs 5.11 ms at c3: off)
#endif
#ifndef MCP_K1T2_DRAIN_TMA
#define MCP_K1T2_DRAIN_TMA 1   // transient drain by bulk tensor reduce-add (0: per-element REDs)
#endif
#ifndef MCP_K1T2_DRAIN_RMW
#define MCP_K1T2_DRAIN_RMW 0   // 1: transient drain as owner read-modify-write (c5: 188.6-190 ms
                               // vs 185.2-185.4 with RED atomics)
#endif
#ifndef MCP_K1T2_KO
#define MCP_K1T2_KO 0   // timing knockouts (see the producer), experiment builds only
#endif
#ifndef MCP_K1T2_PROF
#define MCP_K1T2_PROF 0   // diagnostics only: CTA 0 prints per-role wait / busy cycles
#endif
#if MCP_K1T2_PROF
#define K1T2_T0() const long long _t0 = clock64()
#define K1T2_ACC(v) v += clock64() - _t0
#else
#define K1T2_T0()
#define K1T2_ACC(v)
#endif

// TR: the kernel handles transient m-tiles (prm.mt_tr > 0); the TR = false instance compiles that
// logic away (the single MMA-issuing thread's per-step work measured 4% at c3 otherwise)
template <bool TR>
__global__ void __launch_bounds__(K1T2_THREADS_S, 1)
    k1t2_fg_tf32(const __grid_constant__ CUtensorMap tm_v1, const __grid_constant__ CUtensorMap tm_v2,
                 const __grid_constant__ CUtensorMap tm_l1, const __grid_constant__ CUtensorMap tm_l2,
                 const __grid_constant__ CUtensorMap tm_a,
                 const __grid_constant__ CUtensorMap tm_y, K1TParams prm) {
  extern __shared__ __align__(16) unsigned char smem_raw_t2[];
  unsigned char* base = smem_raw_t2 + ((1024u - (smem_u32(smem_raw_t2) & 1023u)) & 1023u);
  const int RB = prm.RB, NS = prm.stages;
  const size_t SB = k1t_stage_bytes(RB);
  // P bricks: brick b (32 tile rows) holds RB rows of P_hi then RB rows of P_lo, so one K-major
  // descriptor with N = 2 RB covers [P_hi | P_lo]
  unsigned char* sP2 = base + NS * SB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP2 + 1024 * RB);
  uint64_t* full = bars;
  uint64_t* empty = bars + NS;
  uint64_t* z_full = bars + 2 * NS;     // [2]
  uint64_t* p_full = z_full + 2;
  uint64_t* p_empty = z_full + 3;
  uint64_t* y_full = z_full + 4;
  uint64_t* y_empty = z_full + 5;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(z_full + 6);
  uint64_t* split = z_full + 8;         // [NS], prm.insplit: V_lo of the stage is formed
  uint64_t* yt_full = z_full + 16;      // prm.mt_tr: this tile's transient m-tiles are complete
  uint64_t* yt_empty = z_full + 17;     //            ... and read out of TMEM
  // prm.drain_tma: one 2 KB staging slot (32 rows x 8 doubles) per epilogue warp
  double* drain_stage = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(bars) + 1024);
  // the MMA consumes a stage once its data is complete: TMA bytes (full) or, with the in-kernel
  // split, the splitter warps' V_lo as well (split)
  uint64_t* ready = prm.insplit ? split : full;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rb = blockIdx.x % prm.rbs;
  const int pg = blockIdx.x / prm.rbs;
  const int64_t my_tiles =
      pg < prm.num_tiles ? (prm.num_tiles - pg + prm.gp - 1) / prm.gp : 0;
  const int mt2 = prm.mt2, nkb = prm.nkb;
  const int mtr = TR ? prm.mt_tr : 0, mt_p = mt2 - mtr;   // transient / persistent m-tiles
  // GEMM2 m-tile of step group i: the transient m-tiles [mt_p, mt2) first
  auto g2_mt = [&](int i) -> int { return i < mtr ? mt_p + i : i - mtr; };
  auto flush_after = [&](int64_t v) {   // tile v ends a group of prm.flush tiles (or the last)
    return (v % prm.flush) == prm.flush - 1 || v == my_tiles - 1;
  };
  // Z buffer of tile u: alternating under look-ahead; serial order needs only one (TMEM freed)
  auto zbuf = [&](int64_t u) -> int { return prm.serial ? 0 : (int)(u & 1); };

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&split[s], K1T2_SPLIT_WARPS);
    }
    mbar_init(&z_full[0], 1);
    mbar_init(&z_full[1], 1);
    mbar_init(p_full, K1T2_EPI_WARPS);
    mbar_init(p_empty, 1);
    mbar_init(y_full, 1);
    mbar_init(y_empty, K1T2_EPI_WARPS);
    mbar_init(yt_full, 1);
    mbar_init(yt_empty, K1T2_EPI_WARPS);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) tmem_alloc<512>(smem_u32(tslot));
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_v1);
    tma_prefetch_desc(&tm_v2);
    tma_prefetch_desc(&tm_l1);
    tma_prefetch_desc(&tm_l2);
    tma_prefetch_desc(&tm_a);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const int ZW = prm.zcat ? 2 * RB : RB;          // TMEM columns of one Z buffer
  // Z[b] at b ZW; Y[mt] after the Z buffers (two under look-ahead, one in serial order); a wide
  // m-tile has two RB-column halves (V_hi P_hi + V_lo P_hi, V_hi P_lo)
  const uint32_t ty = tmem + (prm.serial ? 1 : 2) * ZW;
  auto ycol = [&](int mt) -> uint32_t {
    return (uint32_t)(mt < prm.wide ? 2 * RB * mt : 2 * RB * prm.wide + RB * (mt - prm.wide));
  };
  // accumulator of GEMM2 m-tile mt: persistent Y after the Z buffer, transient in Z's columns
  auto ydst = [&](int mt) -> uint32_t {
    return mt >= mt_p ? tmem + (uint32_t)(RB * (mt - mt_p)) : ty + ycol(mt);
  };
  // m-tiles with the N = 2 RB product: the first prm.wide persistent ones, a wide transient one
  auto is_wide = [&](int mt) -> bool { return mt < prm.wide || (TR && mt >= mt_p && prm.tr_wide); };

  if (warp == 0) {
    // =========================== TMA producer (same order as the MMA issuer) ===========================
    if (lane == 0) {
      int64_t q = 0;
      auto stage = [&](int64_t qq) -> unsigned char* {
        const int s = (int)(qq % NS);
        if (qq >= NS) mbar_wait(&empty[s], (uint32_t)((qq / NS) - 1) & 1);
        return base + s * SB;
      };
      uint64_t pol_keep = 0, pol_drop = 0;
      if (prm.hint) {
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol_keep));
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol_drop));
      }
      auto load = [&](void* dst, const CUtensorMap* tm, int c0, int c1, uint64_t* fb, uint64_t pol) {
        if (prm.hint)
          tma_load_2d_hint(dst, tm, c0, c1, smem_u32(fb), pol);
        else
          tma_load_2d(dst, tm, c0, c1, smem_u32(fb));
      };
      auto load3 = [&](void* dst, const CUtensorMap* tm, int row, int chunk, uint64_t* fb,
                       uint64_t pol) {
        if (prm.hint)
          tma_load_3d_hint(dst, tm, 0, row, chunk, smem_u32(fb), pol);
        else
          tma_load_3d(dst, tm, 0, row, chunk, smem_u32(fb));
      };
      auto g1 = [&](int64_t u) {
        const int row0 = (int)((pg + u * prm.gp) * K1T_TP);
        for (int kb = 0; kb < nkb; ++kb, ++q) {
          unsigned char* st = stage(q);
          uint64_t* fb = &full[q % NS];
          // MCP_K1T2_KO (timing knockouts, wrong results, experiment builds only): bit 0 = no
          // V_lo loads, bit 1 = factor loaded for the first tile only, bit 2 = no GEMM2 loads
          const bool ko_lo = (MCP_K1T2_KO & 1) || prm.insplit;
          const bool ko_a = (MCP_K1T2_KO & 2) && q >= NS;
          const bool a_lo =   // else formed in smem by the splitter warps
              !ko_a && !(prm.insplit && prm.serial && MCP_K1T2_ASPLIT);
          mbar_arrive_expect_tx(fb, (ko_lo ? 1 : 2) * K1T_VBYTES +
                                        (ko_a ? 0 : a_lo ? 256 * RB : 128 * RB));
          load(st, &tm_v1, kb * 32, row0, fb, pol_keep);
          if (!ko_lo) load(st + K1T_VBYTES, &tm_l1, kb * 32, row0, fb, pol_keep);
          if (!ko_a) tma_load_2d(st + 2 * K1T_VBYTES, &tm_a, kb * 32, rb * RB, smem_u32(fb));
          if (a_lo)
            tma_load_2d(st + 2 * K1T_VBYTES + 128 * RB, &tm_a, kb * 32, prm.r_pad + rb * RB,
                        smem_u32(fb));
        }
      };
      auto g2 = [&](int64_t v) {
        const int row0 = (int)((pg + v * prm.gp) * K1T_TP);
        for (int step = 0; step < 4 * mt2; ++step, ++q) {
          const int mt = g2_mt(step >> 2), rc = step & 3;
          unsigned char* st = stage(q);
          uint64_t* fb = &full[q % NS];
          if (MCP_K1T2_KO & 4) {
            mbar_arrive(fb);
            continue;
          }
          const bool no_lo = (MCP_K1T2_KO & 1) || prm.insplit;
          mbar_arrive_expect_tx(fb, (no_lo ? 1 : 2) * K1T_VBYTES);
          if (no_lo) {
            if (prm.g2_3d) {
              load3(st, &tm_v2, row0 + rc * 32, mt * 4, fb, pol_drop);
            } else {
#pragma unroll
              for (int b = 0; b < 4; ++b)
                load(st + b * 4096, &tm_v2, mt * 128 + b * 32, row0 + rc * 32, fb, pol_drop);
            }
            continue;
          }
          if (prm.g2_3d) {
            load3(st, &tm_v2, row0 + rc * 32, mt * 4, fb, pol_drop);
            load3(st + K1T_VBYTES, &tm_l2, row0 + rc * 32, mt * 4, fb, pol_drop);
          } else {
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              load(st + b * 4096, &tm_v2, mt * 128 + b * 32, row0 + rc * 32, fb, pol_drop);
              load(st + K1T_VBYTES + b * 4096, &tm_l2, mt * 128 + b * 32, row0 + rc * 32, fb,
                     pol_drop);
            }
          }
        }
      };
      if (prm.serial) {
        for (int64_t u = 0; u < my_tiles; ++u) {
          g1(u);
          g2(u);
        }
      } else {
        for (int64_t u = 0; u <= my_tiles; ++u) {
          if (u < my_tiles) g1(u);
          if (u >= 1) g2(u - 1);
        }
      }
    }
  } else if (warp == 1) {
    // =========================== MMA issuer ===========================
    if (lane == 0) {
      const uint32_t id1 = umma_idesc_tf32(128, RB, false, false);
      const uint32_t id1c = umma_idesc_tf32(128, 2 * RB, false, false);
      const uint32_t id2 = umma_idesc_tf32(128, RB, true, false);
      const uint32_t id2w = umma_idesc_tf32(128, 2 * RB, true, false);
      int64_t q = 0;
      int flushes = 0;
      bool fresh = true, wait_y = false;
      long long w_full1 = 0, w_full2 = 0, w_p = 0, w_y = 0;
      const long long t_begin = clock64();
      auto g1 = [&](int64_t u) {
          // ---- GEMM1(u): Z[zb] = V A (3xTF32) ----
          const uint32_t tz = tmem + (uint32_t)(zbuf(u) * ZW);
          // Z's columns held tile u - 1's transient m-tiles: wait until they are read out
          if (mtr && u >= 1) mbar_wait(yt_empty, (uint32_t)(u - 1) & 1);
          for (int kb = 0; kb < nkb; ++kb, ++q) {
            const int s = (int)(q % NS);
            {
              K1T2_T0();
              mbar_wait(&ready[s], (uint32_t)(q / NS) & 1);
              K1T2_ACC(w_full1);
            }
            tc_fence_after();
            // descriptors are affine in the smem address: +16 B adds 1 to the start field, so
            // the 12 instructions of a stage reuse 4 base descriptors (cheap single-lane issue)
            const uint32_t v_hi = smem_u32(base + s * SB);
            const uint64_t dvh = umma_desc_sw128(v_hi, 16, 1024);
            const uint64_t dvl = dvh + (K1T_VBYTES >> 4);
            const uint64_t dah = dvh + ((2 * K1T_VBYTES) >> 4);
            const uint64_t dal = dah + ((128 * RB) >> 4);
            if (prm.zcat) {
              // A_hi and A_lo rows are adjacent in the stage: one N = 2 RB product gives
              // [V_hi A_hi | V_hi A_lo]; V_lo A_hi accumulates into the second half
#pragma unroll
              for (int ks = 0; ks < 4; ++ks)
                umma_tf32(tz, dvh + 2 * ks, dah + 2 * ks, id1c, (kb | ks) != 0 ? 1u : 0u);
#pragma unroll
              for (int ks = 0; ks < 4; ++ks)
                if (!(MCP_K1T2_KO & 8)) umma_tf32(tz + RB, dvl + 2 * ks, dah + 2 * ks, id1, 1u);
            } else {
#pragma unroll
              for (int pr = 0; pr < 3; ++pr) {
                const uint64_t av = pr == 2 ? dvl : dvh, bv = pr == 1 ? dal : dah;
#pragma unroll
                for (int ks = 0; ks < 4; ++ks)
                  umma_tf32(tz, av + 2 * ks, bv + 2 * ks, id1, (kb | pr | ks) != 0 ? 1u : 0u);
              }
            }
            umma_commit(smem_u32(&empty[s]));
          }
          umma_commit(smem_u32(&z_full[zbuf(u)]));
      };
      auto g2 = [&](int64_t v) {
          // ---- GEMM2(v): Y += V^T P (3xTF32) ----
          {
            K1T2_T0();
            mbar_wait(p_full, (uint32_t)v & 1);
            K1T2_ACC(w_p);
          }
          if (wait_y) {
            K1T2_T0();
            mbar_wait(y_empty, (uint32_t)(flushes - 1) & 1);
            K1T2_ACC(w_y);
            wait_y = false;
            fresh = true;
          }
          tc_fence_after();
          const uint64_t dph = umma_desc_sw128(smem_u32(sP2), 16, 1024);
          const uint64_t dpl = dph + ((128 * RB) >> 4);
          for (int step = 0; step < 4 * mt2; ++step, ++q) {
            const int mt = g2_mt(step >> 2), rc = step & 3;
            const bool fr = mt >= mt_p || fresh;   // transient m-tiles start fresh every tile
            const int s = (int)(q % NS);
            {
              K1T2_T0();
              mbar_wait(&ready[s], (uint32_t)(q / NS) & 1);
              K1T2_ACC(w_full2);
            }
            tc_fence_after();
            const uint64_t dvh = umma_desc_sw128_32b(smem_u32(base + s * SB), 4096, 512);
            const uint64_t dvl = dvh + (K1T_VBYTES >> 4);
            const uint64_t boff = (uint64_t)((rc * 256 * RB) >> 4);
            if (is_wide(mt)) {
              // [V_hi P_hi | V_hi P_lo] in one N = 2 RB product, then V_lo P_hi into the first half
#pragma unroll
              for (int ks = 0; ks < 4; ++ks)
                umma_tf32(ydst(mt), dvh + 64 * ks, dph + boff + 2 * ks, id2w,
                          (fr && rc == 0 && ks == 0) ? 0u : 1u);
#pragma unroll
              for (int ks = 0; ks < 4; ++ks)
                if (!(MCP_K1T2_KO & 8))
                  umma_tf32(ydst(mt), dvl + 64 * ks, dph + boff + 2 * ks, id2, 1u);
            } else {
#pragma unroll
              for (int pr = 0; pr < 3; ++pr) {
                if (pr == 1 && prm.g2x2) continue;
                if (pr == 2 && (MCP_K1T2_KO & 8)) continue;
                const uint64_t av = pr == 2 ? dvl : dvh;
                const uint64_t bv = (pr == 1 ? dpl : dph) + boff;
#pragma unroll
                for (int ks = 0; ks < 4; ++ks)
                  umma_tf32(ydst(mt), av + 64 * ks, bv + 2 * ks, id2,
                            (fr && rc == 0 && pr == 0 && ks == 0) ? 0u : 1u);
              }
            }
            umma_commit(smem_u32(&empty[s]));
            if (mtr && step == 4 * mtr - 1) umma_commit(smem_u32(yt_full));
          }
          fresh = false;
          umma_commit(smem_u32(p_empty));
          if (flush_after(v)) {
            umma_commit(smem_u32(y_full));
            ++flushes;
            wait_y = true;
          }
      };
      long long t_g1 = 0, t_g2 = 0;
      if (prm.serial) {
        for (int64_t u = 0; u < my_tiles; ++u) {
#if MCP_K1T2_PROF
          const long long a0 = clock64();
          g1(u);
          const long long a1 = clock64();
          g2(u);
          t_g1 += a1 - a0;
          t_g2 += clock64() - a1;
#else
          g1(u);
          g2(u);
#endif
        }
      } else {
        for (int64_t u = 0; u <= my_tiles; ++u) {
          if (u < my_tiles) g1(u);
          if (u >= 1) g2(u - 1);
        }
      }
#if MCP_K1T2_PROF
      if (blockIdx.x == 0) printf("K1T2 MMA phases: g1 %lld g2 %lld\n", t_g1, t_g2);
#else
      (void)t_g1;
      (void)t_g2;
#endif
#if MCP_K1T2_PROF
      if (blockIdx.x == 0)
        printf("K1T2 MMA: total %lld  wait full(G1) %lld  full(G2) %lld  p_full %lld  y_empty %lld  tiles %lld\n",
               clock64() - t_begin, w_full1, w_full2, w_p, w_y, (long long)my_tiles);
#endif
      (void)t_begin;
    }
  } else if (warp >= 2 + K1T2_EPI_WARPS) {
    // =========================== splitter warps (prm.insplit) ===========================
    // every stage in ring order (the same sequence for either tile order): V_lo = V - tf32(V)
    // elementwise into the stage's V_lo half -- the same swizzled position, since both halves
    // are 1 KB-aligned copies of one layout -- then release the stage to the MMA issuer
    const int st_id = (warp - 2 - K1T2_EPI_WARPS) * 32 + lane;   // 0..127
    const int64_t total = my_tiles * (int64_t)(nkb + 4 * mt2);
    const int per_tile = nkb + 4 * mt2;
    int s = 0, in_tile = 0;
    uint32_t ph = 0;
    for (int64_t q = 0; q < total; ++q) {
      mbar_wait(&full[s], ph);
      // GEMM1 stages (the first nkb of a tile in the serial order): the factor block's lo rows
      // from its fp32 rows (MCP_K1T2_ASPLIT), same swizzle position RB rows further on
      if (MCP_K1T2_ASPLIT && prm.serial && in_tile < nkb) {
        const float4* ah = reinterpret_cast<const float4*>(base + s * SB + 2 * K1T_VBYTES);
        float4* al = reinterpret_cast<float4*>(base + s * SB + 2 * K1T_VBYTES + 128 * RB);
        for (int e = st_id; e < 8 * RB; e += 128) {
          const float4 x = ah[e];
          al[e] = make_float4(x.x - tf32_hi(x.x), x.y - tf32_hi(x.y), x.z - tf32_hi(x.z),
                              x.w - tf32_hi(x.w));
        }
      }
      if (++in_tile == per_tile) in_tile = 0;
      const float4* vh = reinterpret_cast<const float4*>(base + s * SB);
      float4* vl = reinterpret_cast<float4*>(base + s * SB + K1T_VBYTES);
      float4 x[K1T_VBYTES / 16 / 128];
#pragma unroll
      for (int k = 0; k < K1T_VBYTES / 16 / 128; ++k) x[k] = vh[st_id + 128 * k];
#pragma unroll
      for (int k = 0; k < K1T_VBYTES / 16 / 128; ++k)
        vl[st_id + 128 * k] = make_float4(x[k].x - tf32_hi(x[k].x), x[k].y - tf32_hi(x[k].y),
                                          x[k].z - tf32_hi(x[k].z), x[k].w - tf32_hi(x[k].w));
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&split[s]);
      if (++s == NS) {
        s = 0;
        ph ^= 1u;
      }
    }
  } else {
    // =========================== epilogue / flush warps ===========================
    const int ew = warp - 2;                 // 0..7
    const int sp = warp & 3;                 // TMEM sub-partition this warp may access
    const int half = ew >> 2;
    const int l = 32 * sp + lane;            // tile row (TMEM lane) this thread owns
    const int hc = ((RB / 2 + 15) / 16) * 16;  // columns per warp, whole 16-column loads
    const bool col_active = half * hc < RB;
    const int c_end = min(RB, (half + 1) * hc);
    const int dm1 = prm.d - 1;
    int flushes = 0;
    double* Yp = prm.Ypart + ((size_t)rb * prm.gp + pg) * (size_t)mt2 * 128 * RB;
    long long e_wz = 0, e_wp = 0, e_epi = 0, e_fl = 0;
    // 16 columns of this warp's 32 rows of m-tile mt (wide: halves summed first, fp64) added into
    // the fp64 partial by two bulk tensor reduce-adds (TMA, at L2) through the warp's 2 KB
    // staging slot; the caller's previous reduce-adds to these rows have completed (fixed order)
    auto stage_reduce = [&](const float (&tv)[16], const float (&t2)[16], bool wide, int mt,
                            int c0) {
      double* stg = drain_stage + (size_t)ew * 256;   // [32 rows][8]
      const int grow = (int)((((size_t)rb * prm.gp + pg) * mt2 + mt) * 128 + 32 * sp);
#pragma unroll
      for (int k8 = 0; k8 < 2; ++k8) {
        if (lane == 0) k1t_bulk_wait_read();   // the slot's previous reduce has read it
        __syncwarp();
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int a = 8 * k8 + 2 * jj;
          const double v0 = wide ? (double)tv[a] + (double)t2[a] : (double)tv[a];
          const double v1 = wide ? (double)tv[a + 1] + (double)t2[a + 1] : (double)tv[a + 1];
          reinterpret_cast<double2*>(stg + 8 * lane)[jj] = make_double2(v0, v1);
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) k1t_bulk_reduce_add_2d(&tm_y, c0 + 8 * k8, grow, stg);
      }
    };
    auto flush = [&]() {
      K1T2_T0();
      mbar_wait(y_full, (uint32_t)flushes & 1);
      tc_fence_after();
      if (prm.drain_tma && flushes > 0 && lane == 0) k1t_bulk_wait_all();
      for (int mt = 0; mt < mt_p; ++mt) {   // persistent m-tiles (transient ones drain per tile)
        double* yrow = Yp + ((size_t)mt * 128 + l) * RB;
        for (int c0 = half * hc; col_active && c0 < c_end; c0 += 16) {
          float yv[16], y2[16];
          tmem_ld16(ty + ycol(mt) + ((uint32_t)(32 * sp) << 16) + c0, yv);
          const bool wide = mt < prm.wide;
          if (wide) tmem_ld16(ty + ycol(mt) + RB + ((uint32_t)(32 * sp) << 16) + c0, y2);
          if (prm.drain_tma && flushes > 0) {
            stage_reduce(yv, y2, wide, mt, c0);
            continue;
          }
          // each partial element has exactly one owner thread and flushes are in program order,
          // so fire-and-forget reductions (RED, no load latency) keep the sum order fixed
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) {
            const double yd = wide ? (double)yv[jj] + (double)y2[jj] : (double)yv[jj];
            if (flushes == 0)
              yrow[c0 + jj] = yd;
            else
              atomicAdd(yrow + c0 + jj, yd);
          }
        }
      }
      // the first flush's plain stores are seen by the later reduce-adds (async proxy)
      if (prm.drain_tma && flushes == 0) asm volatile("fence.proxy.async.global;\n" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(y_empty);
      ++flushes;
      K1T2_ACC(e_fl);
    };
    for (int64_t u = 0; u < my_tiles; ++u) {
      const int64_t row0 = (pg + u * prm.gp) * K1T_TP;
      // serial order: the group ending at tile u - 1 drains while GEMM1(u) runs
      if (prm.serial && u >= 1 && flush_after(u - 1)) flush();
      {
        K1T2_T0();
        if (prm.serial)
          mbar_wait(&z_full[0], (uint32_t)u & 1);
        else
          mbar_wait(&z_full[u & 1], (uint32_t)(u >> 1) & 1);
        K1T2_ACC(e_wz);
      }
      if (u > 0) {
        K1T2_T0();
        mbar_wait(p_empty, (uint32_t)(u - 1) & 1);   // GEMM2(u - 1) has consumed P
        K1T2_ACC(e_wp);
      }
      tc_fence_after();
      {
        K1T2_T0();
        const uint32_t tz = tmem + (uint32_t)(zbuf(u) * ZW);
        const double nul = prm.nu ? prm.nu[row0 + l] : prm.nu_const;
        const int brick = l >> 5, col = l & 31;
        for (int c0 = half * hc; col_active && c0 < c_end; c0 += 16) {
          float zv[16];
          tmem_ld16(tz + ((uint32_t)(32 * sp) << 16) + c0, zv);
          if (prm.zcat) {
            float z2[16];
            tmem_ld16(tz + RB + ((uint32_t)(32 * sp) << 16) + c0, z2);
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) zv[jj] += z2[jj];
          }
          // powers for all 16 columns at once (one warp-uniform switch on d - 1, independent
          // chains), same left-to-right products as rm_pow (implicit.py:82-91)
          double zd[16], pw[16];
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) zd[jj] = (double)zv[jj];
          rm_pow_vec<16>(zd, pw, dm1);
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) {
            const float pf = (float)(nul * pw[jj]);
            const float ph = prm.g2x2 ? tf32_rna(pf) : tf32_hi(pf);
            const uint32_t off = brick * 256 * RB + brick_off(c0 + jj, col);
            *reinterpret_cast<float*>(sP2 + off) = ph;
            *reinterpret_cast<float*>(sP2 + off + 128 * RB) = pf - ph;
          }
        }
        K1T2_ACC(e_epi);
      }
      fence_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
      if (mtr) {
        // this tile's transient m-tiles (GEMM2 runs them first): 16 columns at a time out of
        // TMEM into the fp64 partial (one owner per element, in order; fire-and-forget REDs
        // keep the registers low -- 4 warps per sub-partition cap them at 128), then Z's
        // columns go back to GEMM1(u + 1).  The drain costs ~13% at c5 (a no-drain timing
        // knockout: 160.6 vs 185.2 ms); reading every value out of TMEM before the release
        // (188.2 ms, spills) and owner read-modify-writes instead of REDs (188.6 ms) lost.
        mbar_wait(yt_full, (uint32_t)u & 1);
        tc_fence_after();
        // the previous tile's reduce-adds to these rows have completed (fixed add order)
        if (TR && prm.drain_tma && u != 0 && lane == 0) k1t_bulk_wait_all();
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c0 = half * hc + 16 * h;
            if (i < mtr && col_active && c0 < c_end) {
              float tv[16];
              tmem_ld16(tmem + (uint32_t)(RB * i) + ((uint32_t)(32 * sp) << 16) + c0, tv);
              if (MCP_K1T2_KO & 16) continue;   // knockout: no drain (timing only)
              if (TR && prm.drain_tma && u != 0) {
                float t2[16];
                if (prm.tr_wide)
                  tmem_ld16(tmem + (uint32_t)RB + ((uint32_t)(32 * sp) << 16) + c0, t2);
                stage_reduce(tv, t2, prm.tr_wide != 0, mt_p + i, c0);
                continue;
              }
              if (prm.tr_wide) {   // the wide m-tile's second half (V_hi P_lo)
                float t2[16];
                tmem_ld16(tmem + (uint32_t)RB + ((uint32_t)(32 * sp) << 16) + c0, t2);
                double* yrow = Yp + ((size_t)(mt_p + i) * 128 + l) * RB;
#pragma unroll
                for (int jj = 0; jj < 16; ++jj) {
                  const double yd = (double)tv[jj] + (double)t2[jj];
                  if (u == 0)
                    yrow[c0 + jj] = yd;
                  else
                    atomicAdd(yrow + c0 + jj, yd);
                }
                continue;
              }
              double* yrow = Yp + ((size_t)(mt_p + i) * 128 + l) * RB;
              if (MCP_K1T2_DRAIN_RMW && u != 0) {
                // owner-thread read-modify-write: 8 x 16-byte loads in flight, then the stores
                double2* y2p = reinterpret_cast<double2*>(yrow + c0);
                double2 cur[8];
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) cur[jj] = y2p[jj];
#pragma unroll
                for (int jj = 0; jj < 8; ++jj)
                  y2p[jj] = make_double2(cur[jj].x + (double)tv[2 * jj],
                                         cur[jj].y + (double)tv[2 * jj + 1]);
              } else {
#pragma unroll
                for (int jj = 0; jj < 16; ++jj) {
                  if (u == 0)
                    yrow[c0 + jj] = (double)tv[jj];
                  else
                    atomicAdd(yrow + c0 + jj, (double)tv[jj]);   // fire-and-forget RED
                }
              }
            }
          }
        // tile 0's plain stores are seen by the later reduce-adds (async proxy)
        if (TR && prm.drain_tma && u == 0) asm volatile("fence.proxy.async.global;\n" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(yt_empty);
      }
      if (!prm.serial && u >= 1 && flush_after(u - 1)) flush();   // committed after GEMM2(u - 1)
    }
    if (my_tiles > 0) flush();                      // the group ending at the last tile
#if MCP_K1T2_PROF
    if (blockIdx.x == 0 && threadIdx.x == 64)
      printf("K1T2 EPI: wait z %lld  wait p_empty %lld  epilogue %lld  flush %lld\n", e_wz, e_wp,
             e_epi, e_fl);
#endif
    if (my_tiles == 0)
      for (int mt = 0; mt < mt2; ++mt)
        for (int c = half * hc; col_active && c < c_end; ++c)
          Yp[((size_t)mt * 128 + l) * RB + c] = 0.0;
    if (TR && prm.drain_tma && lane == 0) k1t_bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

// V_lo = V - tf32(V) for the fast mode, once per observation set (padding stays zero)
__global__ void k_split_lo(const float* __restrict__ v, float* __restrict__ lo, int64_t total) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float x = v[i];
    lo[i] = x - tf32_hi(x);
  }
}

}  // namespace mcp
