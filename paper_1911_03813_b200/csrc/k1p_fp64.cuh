// K1P (FP64 mode, n <= 128): self-fed warp pairs -- the successor of K1S for the HBM-bound
// small-n configs (BASELINE c1, c2).  Same arithmetic and fixed reduction order as K1/K1S
// (reference pkg/src/momentcp/implicit.py:94-107 + w of :124-140).
//
// K1S couples all warp pairs of a CTA through one producer-fed ring: the producer refills a
// stage only when every pair that shares it is done, so the whole CTA runs at the pace of its
// slowest pair -- and with 14 math warps on 4 SM sub-partitions (4,4,3,3) the pairs on the
// 4-warp sub-partitions ARE slower, leaving the others' FP64 pipes idle.  K1P removes the
// coupling and the producer warp:
//   * 6 pairs = 12 math warps, exactly 3 per sub-partition (balanced FP64 pipes, and 168
//     registers per thread instead of 128);
//   * every pair owns a private ring of SP slab stages (16 rows each) and its own full
//     mbarriers; lane 0 of the pair's first warp issues the pair's 1-D TMA bulk copies itself,
//     refilling the stage freed by the previous slab right after the pair's per-slab barrier;
//   * a pair's slab list is static (slab k of the CTA goes to pair k mod 6), so partial sums,
//     and hence results, are bitwise reproducible.
// Per slab and pair: warp h runs GEMM1 (DMMA.8x8x4, factor columns 8*NTM, DFMA for TAIL
// columns) on rows 8h..8h+7 with software-pipelined operand loads, the epilogue
// P = nu z^(d-1), w += P z, one 64-thread named barrier, then GEMM2 Y += V_slab^T P over its
// half of the n m-tiles.  Y partials stay in registers for the whole kernel.
#pragma once

#include "k1s_fp64.cuh"
#include "mcp_common.cuh"

namespace mcp {

constexpr int K1P_PAIRS = 6;
constexpr int K1P_THREADS = 2 * K1P_PAIRS * 32;   // 384: 3 warps per sub-partition
constexpr int K1P_MAXREG = 168;                    // 16384 / (3 * 32), rounded down to 8

// doubles of P staging, reused as the fused-tail scratch before the first epilogue
__host__ __device__ constexpr size_t k1p_pstage_elems(int cw) {
  return (size_t)K1P_PAIRS * 2 * K1S_SR * k1s_pp(cw);
}

// fixed smem bytes besides the rings (factor fragments, tail factor, P staging)
__host__ __device__ inline size_t k1p_fixed_bytes(int kh, int ntm, int cw) {
  return (size_t)kh * ntm * 32 * 8 + (size_t)kh * 16 * 8 +
         (size_t)K1P_PAIRS * 2 * K1S_SR * k1s_pp(cw) * 8;
}

template <int NTM, int TAIL, int MTH, int KH>
__global__ void __maxnreg__(K1P_MAXREG) k1p_fg_pairs(K1SParams prm) {
  constexpr int CW = 8 * NTM + TAIL;
  constexpr int PP = k1s_pp(CW);
  constexpr int TL = TAIL > 0 ? TAIL : 1;
  constexpr int NP = K1P_PAIRS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int64_t ldv = prm.ldv;
  const int SP = prm.stages;                               // stages per pair
  const size_t slab_elems = (size_t)K1S_SR * ldv;
  double* ring = reinterpret_cast<double*>(smem_raw);      // [NP][SP][SR*ldv]
  double* sAf = ring + (size_t)NP * SP * slab_elems;       // [KH][NTM][32]
  double* sAt = sAf + (size_t)KH * NTM * 32;               // [KH*4 rows][4]
  double* sP = sAt + KH * 16;                              // [NP][2][SR][PP]
  uint64_t* full = reinterpret_cast<uint64_t*>(sP + NP * 2 * K1S_SR * PP);   // [NP][SP]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int rb = blockIdx.x % prm.rbs;
  const int pg = blockIdx.x / prm.rbs;
  const int col0 = rb * CW;

  for (int idx = threadIdx.x; idx < KH * NTM * 32; idx += blockDim.x) {
    const int ln = idx & 31, nt = (idx >> 5) % NTM, ks = (idx >> 5) / NTM;
    const int i = 4 * ks + (ln & 3), j = col0 + 8 * nt + (ln >> 2);
    sAf[idx] = (i < prm.n && j < prm.r) ? prm.A[(int64_t)j * prm.n + i] : 0.0;
  }
  for (int idx = threadIdx.x; idx < KH * 16; idx += blockDim.x) {
    const int i = idx >> 2, c = idx & 3, j = col0 + 8 * NTM + c;
    sAt[idx] = (c < TAIL && i < prm.n && j < prm.r) ? prm.A[(int64_t)j * prm.n + i] : 0.0;
  }
  // zeroed ring: GEMM1's padding k-steps read past a row's n values (the next row, or zeros)
  // and multiply them by exact zeros
  // GEMM1's padding k-steps (4 KH > ldv) read past a row's end -- into the next row or, for a
  // stage's last row, the next stage -- and multiply by exact zeros, so never-loaded stages
  // must not hold NaN/Inf bit patterns: zero the ring only when such reads exist.
  if (4 * KH > ldv)
    for (size_t idx = threadIdx.x; idx < (size_t)NP * SP * slab_elems; idx += blockDim.x)
      ring[idx] = 0.0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NP * SP; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // the zero fill above is generic-proxy; the bulk copies below are async-proxy writes
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");

  const int q = warp >> 1, h = warp & 1;
  // CTA pg owns slabs pg, pg + gp, ...; its k-th slab goes to pair k mod NP
  const int64_t my_slabs =
      pg < prm.num_slabs ? (prm.num_slabs - pg + prm.gp - 1) / prm.gp : 0;
  const int64_t n_mine = my_slabs > q ? (my_slabs - q + NP - 1) / NP : 0;  // this pair's slabs
  const uint32_t slab_bytes = (uint32_t)(slab_elems * sizeof(double));
  double* my_ring = ring + (size_t)q * SP * slab_elems;
  uint64_t* my_full = full + q * SP;
  const bool issuer = h == 0 && lane == 0;
  // global row offset of this pair's i-th slab: (pg + (q + i NP) gp) * SR
  const int64_t slab_stride = (int64_t)NP * prm.gp * K1S_SR * ldv;
  const double* src0 = prm.V + ((int64_t)pg + (int64_t)q * prm.gp) * K1S_SR * ldv;
  if (issuer) {
    for (int s = 0; s < SP && s < n_mine; ++s) {
      mbar_arrive_expect_tx(&my_full[s], slab_bytes);
      tma_bulk_g2s(my_ring + (size_t)s * slab_elems, src0 + s * slab_stride, slab_bytes,
                   &my_full[s]);
    }
  }
  const int mbase = h * MTH;
  const int mcnt = h == 0 ? min(MTH, prm.MT) : max(0, prm.MT - MTH);
  double yacc[MTH][NTM][2];
  double ytl[MTH][TL];
  double wacc[NTM][2];
  double wtl = 0.0;
#pragma unroll
  for (int m = 0; m < MTH; ++m) {
#pragma unroll
    for (int nt = 0; nt < NTM; ++nt) yacc[m][nt][0] = yacc[m][nt][1] = 0.0;
#pragma unroll
    for (int c = 0; c < TL; ++c) ytl[m][c] = 0.0;
  }
#pragma unroll
  for (int nt = 0; nt < NTM; ++nt) wacc[nt][0] = wacc[nt][1] = 0.0;
  const int dm1 = prm.d - 1;

  int s = 0;
  uint32_t ph = 0;
  int buf = 0;
  for (int64_t i = 0; i < n_mine; ++i) {
    mbar_wait(&my_full[s], ph);
    const double* sv = my_ring + (size_t)s * slab_elems;
    const int64_t row0 = ((int64_t)pg + (q + i * NP) * (int64_t)prm.gp) * K1S_SR;
    const int s_prev = s == 0 ? SP - 1 : s - 1;
    if (++s == SP) {
      s = 0;
      ph ^= 1;
    }
    double* Pb = sP + ((size_t)q * 2 + buf) * K1S_SR * PP;
    buf ^= 1;

    // ---- GEMM1 on rows 8h..8h+7 (two DMMA chains, operands of step kk+1 loaded first) ----
    double z[2][NTM][2], zt[2][TL];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
      for (int nt = 0; nt < NTM; ++nt) z[mt][nt][0] = z[mt][nt][1] = 0.0;
#pragma unroll
      for (int c = 0; c < TL; ++c) zt[mt][c] = 0.0;
    }
    const double* v0 = sv + (8 * h + g) * ldv + t;
    const double* bp = sAf + lane;
    const double* at = sAt + t * 4;
    double a_c = v0[0], b_c[NTM];
    double2 t_c = make_double2(0.0, 0.0);
#pragma unroll
    for (int nt = 0; nt < NTM; ++nt) b_c[nt] = bp[nt * 32];
    if constexpr (TAIL > 0) t_c = *reinterpret_cast<const double2*>(at);
#pragma unroll
    for (int kk = 0; kk < KH; ++kk) {
      const int e2 = kk & 1;
      double a_n = 0.0, b_n[NTM];
      double2 t_n = make_double2(0.0, 0.0);
      if (kk + 1 < KH) {
        a_n = v0[4 * (kk + 1)];
#pragma unroll
        for (int nt = 0; nt < NTM; ++nt) b_n[nt] = bp[((kk + 1) * NTM + nt) * 32];
        if constexpr (TAIL > 0) t_n = *reinterpret_cast<const double2*>(at + 16 * (kk + 1));
      }
#pragma unroll
      for (int nt = 0; nt < NTM; ++nt) dmma884(z[e2][nt], a_c, b_c[nt]);
      if constexpr (TAIL > 0) {
        zt[e2][0] = fma(a_c, t_c.x, zt[e2][0]);
        if constexpr (TAIL > 1) zt[e2][TL - 1] = fma(a_c, t_c.y, zt[e2][TL - 1]);
      }
      if (kk + 1 < KH) {
        a_c = a_n;
#pragma unroll
        for (int nt = 0; nt < NTM; ++nt) b_c[nt] = b_n[nt];
        t_c = t_n;
      }
    }
#pragma unroll
    for (int nt = 0; nt < NTM; ++nt) {
      z[0][nt][0] += z[1][nt][0];
      z[0][nt][1] += z[1][nt][1];
    }
#pragma unroll
    for (int c = 0; c < TL; ++c) zt[0][c] += zt[1][c];
    static_assert(TAIL <= 2, "tail columns are loaded as one double2");

    // ---- epilogue on row 8h + g: P = nu z^(d-1), w += P z ----
    {
      const int lr = 8 * h + g;
      const double nul = prm.nu ? prm.nu[row0 + lr] : prm.nu_const;
      constexpr int NV = 2 * NTM + 1;
      double zv[NV], pw[NV];
#pragma unroll
      for (int nt = 0; nt < NTM; ++nt) {
        zv[2 * nt] = z[0][nt][0];
        zv[2 * nt + 1] = z[0][nt][1];
      }
      zv[2 * NTM] = 0.0;
      if constexpr (TAIL > 0) {
#pragma unroll
        for (int c = 0; c < TAIL; ++c) {
          double zz = zt[0][c];
          zz += __shfl_xor_sync(0xffffffffu, zz, 1);
          zz += __shfl_xor_sync(0xffffffffu, zz, 2);
          if (t == c) zv[2 * NTM] = zz;
        }
      }
      rm_pow_vec<NV>(zv, pw, dm1);
#pragma unroll
      for (int nt = 0; nt < NTM; ++nt) {
        double pv[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          pv[e] = nul * pw[2 * nt + e];
          wacc[nt][e] = fma(pv[e], zv[2 * nt + e], wacc[nt][e]);
        }
        *reinterpret_cast<double2*>(&Pb[lr * PP + 8 * nt + 2 * t]) = make_double2(pv[0], pv[1]);
      }
      if constexpr (TAIL > 0) {
        if (t < TAIL) {
          const double pv = nul * pw[2 * NTM];
          wtl = fma(pv, zv[2 * NTM], wtl);
          Pb[lr * PP + 8 * NTM + t] = pv;
        }
      }
    }
    asm volatile("bar.sync %0, 64;\n" ::"r"(1 + q) : "memory");
    // both warps of the pair are past GEMM2 of the previous slab: refill its stage
    if (issuer && i >= 1 && i - 1 + SP < n_mine) {
      mbar_arrive_expect_tx(&my_full[s_prev], slab_bytes);
      tma_bulk_g2s(my_ring + (size_t)s_prev * slab_elems, src0 + (i - 1 + SP) * slab_stride,
                   slab_bytes, &my_full[s_prev]);
    }

    // ---- GEMM2: Y[m-tiles of this half] += V_slab^T P over the slab's 16 rows ----
#pragma unroll
    for (int k2 = 0; k2 < K1S_SR / 4; ++k2) {
      const double* prow = Pb + (4 * k2 + t) * PP;
      double b[NTM], bt[TL];
#pragma unroll
      for (int nt = 0; nt < NTM; ++nt) b[nt] = prow[8 * nt + g];
#pragma unroll
      for (int c = 0; c < TAIL; ++c) bt[c] = prow[8 * NTM + c];
      const double* vr = sv + (4 * k2 + t) * ldv + 8 * mbase + g;
#pragma unroll
      for (int m = 0; m < MTH; ++m) {
        double a = vr[8 * m];
        if (m >= MTH - 2) a = (8 * (mbase + m) + g < prm.n) ? a : 0.0;
#pragma unroll
        for (int nt = 0; nt < NTM; ++nt) dmma884(yacc[m][nt], a, b[nt]);
#pragma unroll
        for (int c = 0; c < TAIL; ++c) ytl[m][c] = fma(a, bt[c], ytl[m][c]);
      }
    }
  }
  // ---------------- fixed-order combine of the math warps' partials ----------------
#pragma unroll
  for (int m = 0; m < MTH; ++m)
#pragma unroll
    for (int c = 0; c < TAIL; ++c) {
      ytl[m][c] += __shfl_xor_sync(0xffffffffu, ytl[m][c], 1);
      ytl[m][c] += __shfl_xor_sync(0xffffffffu, ytl[m][c], 2);
    }
#pragma unroll
  for (int nt = 0; nt < NTM; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      double v = wacc[nt][e];
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      wacc[nt][e] = v;
    }
  wtl += __shfl_xor_sync(0xffffffffu, wtl, 4);
  wtl += __shfl_xor_sync(0xffffffffu, wtl, 8);
  wtl += __shfl_xor_sync(0xffffffffu, wtl, 16);
  const int MT = prm.MT;
  __syncthreads();   // every warp has consumed all of its slabs -> the rings are free
  double* stage = ring + (size_t)q * MT * 8 * CW;
#pragma unroll
  for (int m = 0; m < MTH; ++m) {
    if (m < mcnt) {
      const int row = 8 * (mbase + m) + g;
#pragma unroll
      for (int nt = 0; nt < NTM; ++nt) {
        stage[row * CW + 8 * nt + 2 * t] = yacc[m][nt][0];
        stage[row * CW + 8 * nt + 2 * t + 1] = yacc[m][nt][1];
      }
#pragma unroll
      for (int c = 0; c < TAIL; ++c)
        if (t == c) stage[row * CW + 8 * NTM + c] = ytl[m][c];
    }
  }
  double* wst = ring + (size_t)NP * MT * 8 * CW + warp * CW;
  if (g == 0) {
#pragma unroll
    for (int nt = 0; nt < NTM; ++nt) {
      wst[8 * nt + 2 * t] = wacc[nt][0];
      wst[8 * nt + 2 * t + 1] = wacc[nt][1];
    }
    if (t < TAIL) wst[8 * NTM + t] = wtl;
  }
  __syncthreads();
  const int per_cta = MT * 8 * CW;
  double* Yp = prm.Ypart + ((size_t)rb * prm.gp + pg) * per_cta;
  for (int e = threadIdx.x; e < per_cta; e += blockDim.x) {
    double acc = 0.0;
#pragma unroll
    for (int w = 0; w < NP; ++w) acc += ring[(size_t)w * per_cta + e];
    Yp[e] = acc;
  }
  if (threadIdx.x < CW) {
    double acc = 0.0;
#pragma unroll
    for (int w = 0; w < 2 * NP; ++w) acc += ring[(size_t)NP * per_cta + w * CW + threadIdx.x];
    prm.wpart[((size_t)rb * prm.gp + pg) * CW + threadIdx.x] = acc;
  }
}

}  // namespace mcp
