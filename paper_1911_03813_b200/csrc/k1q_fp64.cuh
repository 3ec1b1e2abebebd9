// K1Q (FP64 mode, n <= 128): warp-specialised self-fed pairs.  Same arithmetic as K1/K1S/K1P
// (reference pkg/src/momentcp/implicit.py:94-107 + w of :124-140), different division of labour
// inside a pair:
//   * warp 0 of the pair ("GEMM1 warp") computes Z = V_slab A for ALL 16 rows of a slab (two
//     m-tiles share every factor fragment it loads -- half the factor traffic of K1P), runs the
//     epilogue P = nu z^(d-1), w += P z, and hands P over through a double-buffered smem slot;
//   * warp 1 ("GEMM2 warp") accumulates Y += V_slab^T P over ALL n m-tiles (13 independent DMMA
//     accumulators at n = 100 -- plenty of FP64 ILP), then releases the P slot and refills the
//     slab's ring stage with the pair's next-but-SP slab (1-D TMA bulk copy, lane 0).
// The two warps run one slab apart (P double buffered), synchronised only by mbarriers -- no
// lockstep named barrier.  6 pairs = 12 warps, 3 per sub-partition, 168 registers.
// Static slab -> pair assignment and fixed combine order keep results bitwise reproducible.
#pragma once

#include "k1p_fp64.cuh"
#include "k1s_fp64.cuh"
#include "mcp_common.cuh"

namespace mcp {

#ifndef MCP_K1Q_PAIRS
#define MCP_K1Q_PAIRS 6        // warp pairs per CTA (6: 3 warps per sub-partition, ring of 2)
#endif
constexpr int K1Q_PAIRS = MCP_K1Q_PAIRS;
constexpr int K1Q_THREADS = 2 * K1Q_PAIRS * 32;
constexpr int K1Q_MAXREG = (65536 / K1Q_THREADS) > 255 ? 255 : ((65536 / K1Q_THREADS) & ~7);
#ifndef MCP_K1Q_ODD_CHAINS
#define MCP_K1Q_ODD_CHAINS 0   // 1: GEMM1 with separate even / odd k-step chains (no gain)
#endif
#ifndef MCP_K1Q_PROF
#define MCP_K1Q_PROF 0         // diagnostics only: CTAs 0 and gridDim-1 print phase clocks
#endif
#ifndef MCP_K1Q_L2_AHEAD
#define MCP_K1Q_L2_AHEAD 1     // slabs beyond the ring prefetched into L2 (0: off)
#endif

// L2 prefetch of a global range (bulk, no smem destination)
__device__ __forceinline__ void l2_prefetch_bulk(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}

__host__ __device__ inline size_t k1q_fixed_bytes(int kh, int ntm, int cw) {
  return (size_t)kh * ntm * 32 * 8 + (size_t)kh * 16 * 8 +
         (size_t)K1Q_PAIRS * 2 * K1S_SR * k1s_pp(cw) * 8;
}

// NTM: 8-column DMMA tiles, TAIL: DFMA columns, MT2: GEMM2 m-tiles held by the GEMM2 warp
// (>= ceil(n / 8)), KH: GEMM1 k-steps (>= ldv / 4).
template <int NTM, int TAIL, int MT2, int KH>
__global__ void __maxnreg__(K1Q_MAXREG) k1q_fg_pairs(K1SParams prm) {
  constexpr int CW = 8 * NTM + TAIL;
  constexpr int PP = k1s_pp(CW);
  constexpr int TL = TAIL > 0 ? TAIL : 1;
  constexpr int NP = K1Q_PAIRS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int64_t ldv = prm.ldv;
  const int SP = prm.stages;
  const size_t slab_elems = (size_t)K1S_SR * ldv;
  double* ring = reinterpret_cast<double*>(smem_raw);      // [NP][SP][SR*ldv]
  double* sAf = ring + (size_t)NP * SP * slab_elems;       // [KH][NTM][32]
  double* sAt = sAf + (size_t)KH * NTM * 32;               // [KH*4 rows][4]
  double* sP = sAt + KH * 16;                              // [NP][2][SR][PP]
  uint64_t* full = reinterpret_cast<uint64_t*>(sP + NP * 2 * K1S_SR * PP);  // [NP][SP]
  uint64_t* pfull = full + NP * SP;                                          // [NP][2]
  uint64_t* pempty = pfull + NP * 2;                                         // [NP][2]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int rb = blockIdx.x % prm.rbs;
  const int pg = blockIdx.x / prm.rbs;
  const int col0 = rb * CW;
#if MCP_K1Q_PROF
  const long long pt0 = clock64();
  long long pt_wait = 0, pt_pro = 0, pt_first = 0, pt_loop = 0, pt_sync = 0, w_full = 0, w_p = 0;
  const bool prof = (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1) && lane == 0 &&
                    (warp == 0 || warp == 1);
#endif

  // GEMM1's padding k-steps (4 KH > ldv) read past a row's end -- into the next row or, for a
  // stage's last row, the next stage -- and multiply by exact zeros, so never-loaded stages
  // must not hold NaN/Inf bit patterns: zero the ring only when such reads exist.
  if (4 * KH > ldv)
    for (size_t idx = threadIdx.x; idx < (size_t)NP * SP * slab_elems; idx += blockDim.x)
      ring[idx] = 0.0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NP * SP; ++s) mbar_init(&full[s], 1);
    for (int s = 0; s < NP * 2; ++s) {
      mbar_init(&pfull[s], 32);
      mbar_init(&pempty[s], 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");

  // roles: warp w sits on sub-partition w % 4; alternate the roles along each sub-partition so
  // every FP64 pipe serves a mix of the (heavier) GEMM1 warps and the GEMM2 warps:
  // GEMM1 warps {0, 2, 5, 7, 8, 10}, GEMM2 warps {1, 3, 4, 6, 9, 11}; pair q = q-th of each.
  const int h = ((warp & 3) + (warp >> 2)) & 1;
  const int q = ((warp >> 2) * 4 + (warp & 3)) >> 1;   // rank of w within its role list
  const int64_t my_slabs =
      pg < prm.num_slabs ? (prm.num_slabs - pg + prm.gp - 1) / prm.gp : 0;
  const int64_t n_mine = my_slabs > q ? (my_slabs - q + NP - 1) / NP : 0;
  const uint32_t slab_bytes = (uint32_t)(slab_elems * sizeof(double));
  double* my_ring = ring + (size_t)q * SP * slab_elems;
  uint64_t* my_full = full + q * SP;
  uint64_t* my_pfull = pfull + q * 2;
  uint64_t* my_pempty = pempty + q * 2;
  double* my_P = sP + (size_t)q * 2 * K1S_SR * PP;
  const int64_t slab_stride = (int64_t)NP * prm.gp * K1S_SR * ldv;
  const double* src0 = prm.V + ((int64_t)pg + (int64_t)q * prm.gp) * K1S_SR * ldv;
  if (h == 1 && lane == 0) {
    for (int s = 0; s < SP && s < n_mine; ++s) {
      mbar_arrive_expect_tx(&my_full[s], slab_bytes);
      tma_bulk_g2s(my_ring + (size_t)s * slab_elems, src0 + s * slab_stride, slab_bytes,
                   &my_full[s]);
    }
    for (int a = 0; a < MCP_K1Q_L2_AHEAD; ++a)
      if (SP + a < n_mine) l2_prefetch_bulk(src0 + (SP + a) * slab_stride, slab_bytes);
  }
  // Programmatic dependent launch: everything above depends only on V, so under PDL it overlaps
  // the previous kernel's tail; x (A, lam) may be produced by that kernel and our partials / M /
  // u are read by it -- wait for its completion here (a no-op without PDL).
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
#if MCP_K1Q_PROF
  pt_wait = clock64() - pt0;
#endif
  {
    // factor fragments: every global load of the thread is issued before the first store (one
    // L2 round trip on the critical path instead of one per loop trip)
    constexpr int NAF = KH * NTM * 32, NAT = KH * 16;
    constexpr int PER = (NAF + NAT + K1Q_THREADS - 1) / K1Q_THREADS;
    double av[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int idx = threadIdx.x + u * K1Q_THREADS;
      int i = 0, j = prm.r;
      if (idx < NAF) {
        const int ln = idx & 31, nt = (idx >> 5) % NTM, ks = (idx >> 5) / NTM;
        i = 4 * ks + (ln & 3);
        j = col0 + 8 * nt + (ln >> 2);
      } else if (idx < NAF + NAT) {
        const int it = idx - NAF, c = it & 3;
        i = it >> 2;
        j = c < TAIL ? col0 + 8 * NTM + c : prm.r;
      }
      av[u] = (i < prm.n && j < prm.r) ? prm.A[(int64_t)j * prm.n + i] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int idx = threadIdx.x + u * K1Q_THREADS;
      if (idx < NAF)
        sAf[idx] = av[u];
      else if (idx < NAF + NAT)
        sAt[idx - NAF] = av[u];
    }
  }
  __syncthreads();
  const int dm1 = prm.d - 1;
  const int MT = prm.MT;
#if MCP_K1Q_PROF
  pt_pro = clock64() - pt0;
#endif

  if (h == 0) {
    // ================= GEMM1 warp: Z for 16 rows, epilogue, P hand-off =================
    double wacc[NTM][2];
    double wtl = 0.0;
#pragma unroll
    for (int nt = 0; nt < NTM; ++nt) wacc[nt][0] = wacc[nt][1] = 0.0;
    int s = 0;
    uint32_t ph = 0;
    for (int64_t i = 0; i < n_mine; ++i) {
#if MCP_K1Q_PROF
      const long long tw = clock64();
#endif
      mbar_wait(&my_full[s], ph);
#if MCP_K1Q_PROF
      w_full += clock64() - tw;
      if (i == 0) pt_first = clock64() - pt0;
#endif
      const double* sv = my_ring + (size_t)s * slab_elems;
      if (++s == SP) {
        s = 0;
        ph ^= 1;
      }
      const int64_t row0 = ((int64_t)pg + (q + i * NP) * (int64_t)prm.gp) * K1S_SR;
      // two m-tiles x (even, odd k-steps) = 4 independent DMMA chains per column tile
      double z[2][NTM][2], zo[2][NTM][2], zt[2][TL];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
        for (int nt = 0; nt < NTM; ++nt)
          z[mt][nt][0] = z[mt][nt][1] = zo[mt][nt][0] = zo[mt][nt][1] = 0.0;
#pragma unroll
        for (int c = 0; c < TL; ++c) zt[mt][c] = 0.0;
      }
      const double* v0 = sv + g * ldv + t;         // rows g and 8 + g
      const double* v1 = v0 + 8 * ldv;
      const double* bp = sAf + lane;
      const double* at = sAt + t * 4;
      double a0c = v0[0], a1c = v1[0], b_c[NTM];
      double2 t_c = make_double2(0.0, 0.0);
#pragma unroll
      for (int nt = 0; nt < NTM; ++nt) b_c[nt] = bp[nt * 32];
      if constexpr (TAIL > 0) t_c = *reinterpret_cast<const double2*>(at);
#pragma unroll
      for (int kk = 0; kk < KH; ++kk) {
        double a0n = 0.0, a1n = 0.0, b_n[NTM];
        double2 t_n = make_double2(0.0, 0.0);
        if (kk + 1 < KH) {
          a0n = v0[4 * (kk + 1)];
          a1n = v1[4 * (kk + 1)];
#pragma unroll
          for (int nt = 0; nt < NTM; ++nt) b_n[nt] = bp[((kk + 1) * NTM + nt) * 32];
          if constexpr (TAIL > 0) t_n = *reinterpret_cast<const double2*>(at + 16 * (kk + 1));
        }
#pragma unroll
        for (int nt = 0; nt < NTM; ++nt) {
          if (MCP_K1Q_ODD_CHAINS && (kk & 1)) {
            dmma884(zo[0][nt], a0c, b_c[nt]);
            dmma884(zo[1][nt], a1c, b_c[nt]);
          } else {
            dmma884(z[0][nt], a0c, b_c[nt]);
            dmma884(z[1][nt], a1c, b_c[nt]);
          }
        }
        if constexpr (TAIL > 0) {
          zt[0][0] = fma(a0c, t_c.x, zt[0][0]);
          zt[1][0] = fma(a1c, t_c.x, zt[1][0]);
          if constexpr (TAIL > 1) {
            zt[0][TL - 1] = fma(a0c, t_c.y, zt[0][TL - 1]);
            zt[1][TL - 1] = fma(a1c, t_c.y, zt[1][TL - 1]);
          }
        }
        if (kk + 1 < KH) {
          a0c = a0n;
          a1c = a1n;
#pragma unroll
          for (int nt = 0; nt < NTM; ++nt) b_c[nt] = b_n[nt];
          t_c = t_n;
        }
      }
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < NTM; ++nt) {
          z[mt][nt][0] += zo[mt][nt][0];
          z[mt][nt][1] += zo[mt][nt][1];
        }
      // the P slot of slab i was last read by GEMM2 of slab i - 2
      const int b = (int)(i & 1);
      if (i >= 2) mbar_wait(&my_pempty[b], (uint32_t)(((i - 2) >> 1) & 1));
      double* Pb = my_P + (size_t)b * K1S_SR * PP;
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const int lr = 8 * mt + g;
        const double nul = prm.nu ? prm.nu[row0 + lr] : prm.nu_const;
        constexpr int NV = 2 * NTM + 1;
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
          *reinterpret_cast<double2*>(&Pb[lr * PP + 8 * nt + 2 * t]) =
              make_double2(pv[0], pv[1]);
        }
        if constexpr (TAIL > 0) {
          if (t < TAIL) {
            const double pv = nul * pw[2 * NTM];
            wtl = fma(pv, zv[2 * NTM], wtl);
            Pb[lr * PP + 8 * NTM + t] = pv;
          }
        }
      }
      mbar_arrive(&my_pfull[b]);
    }
    // w partial of the pair (this warp saw every row of the pair's slabs)
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
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
#if MCP_K1Q_PROF
    pt_loop = clock64() - pt0;
#endif
    __syncthreads();   // (A) all slabs consumed by both warps of every pair
#if MCP_K1Q_PROF
    pt_sync = clock64() - pt0;
#endif
    double* wst = ring + (size_t)NP * MT * 8 * CW + q * CW;
    if (g == 0) {
#pragma unroll
      for (int nt = 0; nt < NTM; ++nt) {
        wst[8 * nt + 2 * t] = wacc[nt][0];
        wst[8 * nt + 2 * t + 1] = wacc[nt][1];
      }
      if (t < TAIL) wst[8 * NTM + t] = wtl;
    }
  } else {
    // ================= GEMM2 warp: Y over all m-tiles, ring refills =================
    double yacc[MT2][NTM][2];
    double ytl[MT2][TL];
#pragma unroll
    for (int m = 0; m < MT2; ++m) {
#pragma unroll
      for (int nt = 0; nt < NTM; ++nt) yacc[m][nt][0] = yacc[m][nt][1] = 0.0;
#pragma unroll
      for (int c = 0; c < TL; ++c) ytl[m][c] = 0.0;
    }
    int s = 0;
    uint32_t ph = 0;
    for (int64_t i = 0; i < n_mine; ++i) {
      const int b = (int)(i & 1);
      mbar_wait(&my_full[s], ph);     // (already complete: the GEMM1 warp waited on it)
#if MCP_K1Q_PROF
      const long long tw = clock64();
#endif
      mbar_wait(&my_pfull[b], (uint32_t)((i >> 1) & 1));
#if MCP_K1Q_PROF
      w_p += clock64() - tw;
      if (i == 0) pt_first = clock64() - pt0;
#endif
      const double* sv = my_ring + (size_t)s * slab_elems;
      const double* Pb = my_P + (size_t)b * K1S_SR * PP;
#pragma unroll
      for (int k2 = 0; k2 < K1S_SR / 4; ++k2) {
        const double* prow = Pb + (4 * k2 + t) * PP;
        double bb[NTM], bt[TL];
#pragma unroll
        for (int nt = 0; nt < NTM; ++nt) bb[nt] = prow[8 * nt + g];
#pragma unroll
        for (int c = 0; c < TAIL; ++c) bt[c] = prow[8 * NTM + c];
        const double* vr = sv + (4 * k2 + t) * ldv + g;
#pragma unroll
        for (int m = 0; m < MT2; ++m) {
          double a = vr[8 * m];
          if (m >= MT2 - 2) a = (8 * m + g < prm.n) ? a : 0.0;
#pragma unroll
          for (int nt = 0; nt < NTM; ++nt) dmma884(yacc[m][nt], a, bb[nt]);
#pragma unroll
          for (int c = 0; c < TAIL; ++c) ytl[m][c] = fma(a, bt[c], ytl[m][c]);
        }
      }
      mbar_arrive(&my_pempty[b]);
      __syncwarp();
      if (lane == 0 && i + SP < n_mine) {
        mbar_arrive_expect_tx(&my_full[s], slab_bytes);
        tma_bulk_g2s(my_ring + (size_t)s * slab_elems, src0 + (i + SP) * slab_stride, slab_bytes,
                     &my_full[s]);
        if (MCP_K1Q_L2_AHEAD > 0 && i + SP + MCP_K1Q_L2_AHEAD < n_mine)
          l2_prefetch_bulk(src0 + (i + SP + MCP_K1Q_L2_AHEAD) * slab_stride, slab_bytes);
      }
      if (++s == SP) {
        s = 0;
        ph ^= 1;
      }
    }
#pragma unroll
    for (int m = 0; m < MT2; ++m)
#pragma unroll
      for (int c = 0; c < TAIL; ++c) {
        ytl[m][c] += __shfl_xor_sync(0xffffffffu, ytl[m][c], 1);
        ytl[m][c] += __shfl_xor_sync(0xffffffffu, ytl[m][c], 2);
      }
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
#if MCP_K1Q_PROF
    pt_loop = clock64() - pt0;
#endif
    __syncthreads();   // (A)
#if MCP_K1Q_PROF
    pt_sync = clock64() - pt0;
#endif
    double* stage = ring + (size_t)q * MT * 8 * CW;
#pragma unroll
    for (int m = 0; m < MT2; ++m) {
      if (m < MT) {
        const int row = 8 * m + g;
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
  }
  __syncthreads();
#if MCP_K1Q_PROF
  const long long pt_staged = clock64() - pt0;
#endif
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
    for (int w = 0; w < NP; ++w) acc += ring[(size_t)NP * per_cta + w * CW + threadIdx.x];
    prm.wpart[((size_t)rb * prm.gp + pg) * CW + threadIdx.x] = acc;
  }
#if MCP_K1Q_PROF
  if (prof)
    printf("K1Q cta %d warp %d slabs %lld: wait %lld prologue %lld first %lld loop_end %lld "
           "after_sync %lld staged %lld end %lld | w_full %lld w_pfull %lld\n", blockIdx.x, warp,
           (long long)n_mine, pt_wait, pt_pro, pt_first, pt_loop, pt_sync, pt_staged, clock64() - pt0,
           w_full, w_p);
#endif
}

}  // namespace mcp
