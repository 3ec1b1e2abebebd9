// K1S (FP64 mode, n <= 128): warp-specialised streaming f+grad partial over 16-row slabs.
//
// Same arithmetic as K1 (reference pkg/src/momentcp/implicit.py:94-107 + w of :124-140):
//   Z = V_slab A  ->  P = nu * Z^(d-1), w += P*Z  ->  Y += V_slab^T P
// organised for the HBM-bound small-n configs (BASELINE c1, c2):
//   * one producer warp streams contiguous 16-row slabs HBM -> SMEM with 1-D TMA bulk copies
//     (cp.async.bulk + mbarrier complete_tx) into an S-stage ring, V read from HBM exactly once;
//   * 7 pairs of math warps; slab k of the CTA goes to pair k mod 7.  In a pair, warp h runs
//     GEMM1 over its half of the k-steps for all 16 slab rows (fixed KH steps, zero padded),
//     the two K-halves are added through a small exchange
//     buffer, warp h runs the epilogue for rows 8h..8h+7 and GEMM2 for its half of the n
//     m-tiles.  Synchronisation is two 64-thread named barriers per slab -- no CTA-wide
//     barrier in the main loop;
//   * the factor block is 8*NTM DMMA columns plus TAIL (0..3) DFMA columns, so r = 10 (c2) runs
//     as 8 DMMA + 2 DFMA columns with no padded FP64 work (DMMA and DFMA share the FP64 pipe).
// The smem row pitch equals the global pitch ldv (== 4 mod 16 doubles, chosen at upload) so both
// GEMMs' 8-byte fragment loads are bank-conflict free.  Per-warp Y partials stay in registers for
// the whole kernel; warps and CTAs are combined in a fixed order (bitwise reproducible).
#pragma once

#include "mcp_common.cuh"

namespace mcp {

constexpr int K1S_SR = 16;   // observations per slab (one pair, 8 rows per warp in GEMM1)
constexpr int K1S_MT1 = K1S_SR / 16;  // GEMM1 m-tiles per warp

struct K1SParams {
  const double* V;       // p_pad x ldv observation-major, fp64
  int64_t ldv;           // row pitch (elements), == 4 mod 16
  int64_t num_slabs;     // p_pad / K1S_SR (a multiple of spc)
  int spc;               // slabs per TMA copy unit (one bulk copy fills spc slabs)
  int n;
  int MT;                // ceil(n / 8) m-tiles of GEMM2
  const double* nu;      // nullptr -> nu_const
  double nu_const;
  const double* A;       // n x r column-major (packed x + r)
  int r;
  int d;
  int rbs;               // column blocks of width 8*NTM + TAIL
  int gp;                // CTAs per column block
  int stages;            // ring depth in copy units
  double* Ypart;         // [rbs][gp][MT*8][CW]
  double* wpart;         // [rbs][gp][CW]
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Bounded wait: a pipeline bug traps (loud kernel error) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  if (mbar_try_wait(bar, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try_wait(bar, parity)) {
    if (clock64() - t0 > (1ll << 35)) __trap();
  }
}
// 1-D TMA: global -> shared bulk copy completing on an mbarrier (bytes % 16 == 0).
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                             uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// P staging pitch (doubles) for a CW-column block: == 12 or 20 (mod 32 words: 24t / 8t), which
// makes the GEMM2 B-fragment loads P[4ks + t][8nt + g] bank-conflict free.
__host__ __device__ constexpr int k1s_pp(int cw) { return cw <= 12 ? 12 : 20; }

// Dynamic smem layout, in order:
//   ring: stages * SR * ldv doubles | Afrag: (ldv/4) * NTM * 32 doubles | Atail: ldv * 4 doubles
//   P staging: pairs * 2 * SR * PP doubles (double buffered) | barriers
__host__ __device__ inline size_t k1s_fixed_bytes(int kh, int ntm, int cw, int pairs) {
  return (size_t)kh * ntm * 32 * 8 + (size_t)kh * 16 * 8 +
         (size_t)pairs * 2 * K1S_SR * k1s_pp(cw) * 8;
}


#ifndef MCP_K1S_PAIRS
#define MCP_K1S_PAIRS 7
#endif
constexpr int K1S_PAIRS = MCP_K1S_PAIRS;  // math warp pairs per CTA (6: 13 warps -> 152 regs)
constexpr int K1S_THREADS = (2 * K1S_PAIRS + 1) * 32;  // + 1 producer warp
// registers per thread: each of the 4 SM sub-partitions has its own 16K-register file and
// receives ceil(warps / 4) of the CTA's warps
constexpr int K1S_MAXREG =
    (16384 / (32 * ((K1S_THREADS / 32 + 3) / 4))) / 8 * 8 > 255
        ? 255
        : (16384 / (32 * ((K1S_THREADS / 32 + 3) / 4))) / 8 * 8;

// NTM: 8-column DMMA tiles, TAIL: DFMA columns, MTH: GEMM2 m-tiles per warp (warp 0 of a pair
// takes [0, MTH), warp 1 [MTH, MT)), KH: GEMM1 k-steps (>= ldv / 4, zero-padded factor).
template <int NTM, int TAIL, int MTH, int KH>
__global__ void __maxnreg__(K1S_MAXREG) k1s_fg_stream(K1SParams prm) {
  constexpr int CW = 8 * NTM + TAIL;
  constexpr int PP = k1s_pp(CW);
  constexpr int TL = TAIL > 0 ? TAIL : 1;
  constexpr int NP = K1S_PAIRS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int64_t ldv = prm.ldv;
  const int S = prm.stages;
  const int kst = (int)(ldv / 4);
  const int spc = prm.spc;
  double* ring = reinterpret_cast<double*>(smem_raw);
  double* sAf = ring + (size_t)S * spc * K1S_SR * ldv;  // [KH][NTM][32]
  double* sAt = sAf + (size_t)KH * NTM * 32;             // [KH*4 rows][4]
  double* sP = sAt + KH * 16;                            // [NP][2][SR][PP]
  uint64_t* full = reinterpret_cast<uint64_t*>(sP + NP * 2 * K1S_SR * PP);
  uint64_t* empty = full + S;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int rb = blockIdx.x % prm.rbs;
  const int pg = blockIdx.x / prm.rbs;
  const int col0 = rb * CW;

  // factor block (zero beyond n / r and for the padding k-steps) and a zeroed ring: the
  // padding k-steps multiply finite data (the next row, or zeros) by exact zeros
  for (int idx = threadIdx.x; idx < KH * NTM * 32; idx += blockDim.x) {
    const int ln = idx & 31, nt = (idx >> 5) % NTM, ks = (idx >> 5) / NTM;
    const int i = 4 * ks + (ln & 3), j = col0 + 8 * nt + (ln >> 2);
    sAf[idx] = (i < prm.n && j < prm.r) ? prm.A[(int64_t)j * prm.n + i] : 0.0;
  }
  for (int idx = threadIdx.x; idx < KH * 16; idx += blockDim.x) {
    const int i = idx >> 2, c = idx & 3, j = col0 + 8 * NTM + c;
    sAt[idx] = (c < TAIL && i < prm.n && j < prm.r) ? prm.A[(int64_t)j * prm.n + i] : 0.0;
  }
  for (size_t idx = threadIdx.x; idx < (size_t)S * spc * K1S_SR * ldv; idx += blockDim.x)
    ring[idx] = 0.0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 2 * spc);   // both warps of each slab's pair release
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // CTA pg owns copy units pg, pg + gp, ... (a unit = spc consecutive slabs, one bulk copy);
  // its k-th slab is slab (k mod spc) of its (k / spc)-th unit.
  const int64_t num_units = prm.num_slabs / spc;
  const int64_t my_units = pg < num_units ? (num_units - pg + prm.gp - 1) / prm.gp : 0;
  const int64_t my_slabs = my_units * spc;
  const uint32_t unit_bytes = (uint32_t)(spc * K1S_SR * ldv * sizeof(double));

  if (warp == 2 * NP) {
    // ---------------- producer: one lane streams copy units into the ring ----------------
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      const double* src = prm.V + (int64_t)pg * spc * K1S_SR * ldv;
      const int64_t step = (int64_t)prm.gp * spc * K1S_SR * ldv;
      for (int64_t j = 0; j < my_units; ++j) {
        if (j >= S) mbar_wait(&empty[s], ph);
        mbar_arrive_expect_tx(&full[s], unit_bytes);
        tma_bulk_g2s(ring + (size_t)s * spc * K1S_SR * ldv, src, unit_bytes, &full[s]);
        src += step;
        if (++s == S) {
          s = 0;
          if (j >= S) ph ^= 1;
          else ph = 0;
        }
      }
    }
    return;
  }

  // ---------------- math warps ----------------
  const int q = warp >> 1, h = warp & 1;
  const int mbase = h * MTH;
  // m-tiles this warp owns (warp 0: [0, MTH), warp 1: [MTH, MT)); 0 <= mcnt <= MTH.  It bounds
  // the final staging writes, which must never spill into the next pair's region.
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
  (void)kst;

  // Slab walk without divisions: k advances by NP, so the unit index advances by
  // (sub + NP) / spc and sub becomes (sub + NP) % spc -- both functions of sub < spc <= 14 only.
  int64_t j = q / spc;
  int sub = q % spc;
  int s = (int)(j % S);
  uint32_t ph = (uint32_t)((j / S) & 1);
  const int dj_lo = NP / spc, sub_step = NP % spc;
  int buf = 0;
  for (int64_t k = q; k < my_slabs; k += NP) {
    mbar_wait(&full[s], ph);
    const double* sv = ring + ((size_t)s * spc + sub) * K1S_SR * ldv;
    const int64_t row0 = ((pg + j * prm.gp) * spc + sub) * K1S_SR;
    const int s_cur = s;
    {
      int nsub = sub + sub_step, dj = dj_lo;
      if (nsub >= spc) {
        nsub -= spc;
        ++dj;
      }
      sub = nsub;
      j += dj;
      s += dj;
      if (s >= S) {
        s -= S;
        ph ^= 1;
      }
    }
    double* Pb = sP + ((size_t)q * 2 + buf) * K1S_SR * PP;
    buf ^= 1;

    // ---- GEMM1 on rows 8h..8h+7, all k-steps ----
    constexpr int M1 = K1S_MT1 > 0 ? K1S_MT1 : 1;
    double z[2][NTM][2], zt[2][TL];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
      for (int nt = 0; nt < NTM; ++nt) z[mt][nt][0] = z[mt][nt][1] = 0.0;
#pragma unroll
      for (int c = 0; c < TL; ++c) zt[mt][c] = 0.0;
    }
    // even / odd k-steps accumulate separately (2 independent DMMA chains), added below.
    // Operands of step kk + 1 are loaded before step kk's math (explicit software pipeline:
    // with the register cap ptxas otherwise reuses one register set and serialises every step
    // on its shared-memory load).
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
#pragma unroll
    for (int mt = 0; mt < M1; ++mt) {
      const int lr = 8 * h + g;
      const double nul = prm.nu ? prm.nu[row0 + lr] : prm.nu_const;
      constexpr int NV = 2 * NTM + 1;   // this lane's z values: DMMA columns, then a tail column
      double zv[NV], pw[NV];
#pragma unroll
      for (int nt = 0; nt < NTM; ++nt) {
        zv[2 * nt] = z[mt][nt][0];
        zv[2 * nt + 1] = z[mt][nt][1];
      }
      zv[2 * NTM] = 0.0;
      if constexpr (TAIL > 0) {
#pragma unroll
        for (int c = 0; c < TAIL; ++c) {
          double zz = zt[mt][c];
          zz += __shfl_xor_sync(0xffffffffu, zz, 1);   // lane t summed i == t (mod 4)
          zz += __shfl_xor_sync(0xffffffffu, zz, 2);
          if (t == c) zv[2 * NTM] = zz;                // lane t == c owns tail column c
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
        // every warp runs MTH m-tiles; rows past n (incl. warp 1's spare tile) read as zero
        double a = vr[8 * m];
        if (m >= MTH - 2) a = (8 * (mbase + m) + g < prm.n) ? a : 0.0;
#pragma unroll
        for (int nt = 0; nt < NTM; ++nt) dmma884(yacc[m][nt], a, b[nt]);
#pragma unroll
        for (int c = 0; c < TAIL; ++c) ytl[m][c] = fma(a, bt[c], ytl[m][c]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s_cur]);
  }
  // ---------------- fixed-order combine of the math warps' partials ----------------
#pragma unroll
  for (int m = 0; m < MTH; ++m)
#pragma unroll
    for (int c = 0; c < TAIL; ++c) {
      ytl[m][c] += __shfl_xor_sync(0xffffffffu, ytl[m][c], 1);   // lane t summed l == t (mod 4)
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
  // every math warp has consumed all of its slabs -> the ring is free for staging
  asm volatile("bar.sync 15, %0;\n" ::"n"(2 * NP * 32) : "memory");
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
  asm volatile("bar.sync 15, %0;\n" ::"n"(2 * NP * 32) : "memory");
  const int per_cta = MT * 8 * CW;
  double* Yp = prm.Ypart + ((size_t)rb * prm.gp + pg) * per_cta;
  for (int e = threadIdx.x; e < per_cta; e += 2 * NP * 32) {
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
