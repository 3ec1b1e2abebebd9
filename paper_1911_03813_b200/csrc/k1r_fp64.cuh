// K1R (FP64 mode, n <= 128, r mod 8 != 0): warp TRIADS.  Same arithmetic as K1Q (reference
// pkg/src/momentcp/implicit.py:94-107 + w of :124-140); the GEMM1 role of a K1Q pair is split
// by columns between two warps, because at c2 the GEMM1 warp is the critical role of K1Q
// (skipping only its DFMA tail columns saves 9%):
//   * warp G1a: Z for the 8 NTM DMMA columns of a 16-row slab (two m-tiles share each factor
//     fragment), their epilogue P = nu z^(d-1), w += P z, P hand-off;
//   * warp G1b: the r mod 8 tail columns on DFMA (lane-strided over k, butterfly over the 4
//     k-lanes), their epilogue and P hand-off;
//   * warp G2: Y += V_slab^T P over all n m-tiles (as K1Q's GEMM2 warp), then the ring refill.
// 4 triads = 12 warps, one triad per SM sub-partition.  With 4 slab streams instead of 6 the
// same shared memory holds a 3-slab ring per triad (GEMM1 on slab i, GEMM2 on slab i - 1, slab
// i + 1 in flight).  Static slab -> triad assignment and fixed combine order keep the results
// bitwise reproducible.
#pragma once

#include "k1q_fp64.cuh"
#include "k1s_fp64.cuh"
#include "mcp_common.cuh"

namespace mcp {

constexpr int K1R_TRIADS = 4;
constexpr int K1R_THREADS = 3 * K1R_TRIADS * 32;
constexpr int K1R_MAXREG = 168;

__host__ __device__ inline size_t k1r_fixed_bytes(int kh, int ntm, int cw) {
  return (size_t)kh * ntm * 32 * 8 + (size_t)kh * 16 * 8 +
         (size_t)K1R_TRIADS * 2 * K1S_SR * k1s_pp(cw) * 8;
}

template <int NTM, int TAIL, int MT2, int KH>
__global__ void __maxnreg__(K1R_MAXREG) k1r_fg_triads(K1SParams prm) {
  static_assert(TAIL > 0, "K1R needs DFMA tail columns (else K1Q)");
  constexpr int CW = 8 * NTM + TAIL;
  constexpr int PP = k1s_pp(CW);
  constexpr int NT = K1R_TRIADS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int64_t ldv = prm.ldv;
  const int SP = prm.stages;
  const size_t slab_elems = (size_t)K1S_SR * ldv;
  double* ring = reinterpret_cast<double*>(smem_raw);      // [NT][SP][SR*ldv]
  double* sAf = ring + (size_t)NT * SP * slab_elems;       // [KH][NTM][32]
  double* sAt = sAf + (size_t)KH * NTM * 32;               // [KH*4 rows][4]
  double* sP = sAt + KH * 16;                              // [NT][2][SR][PP]
  uint64_t* full = reinterpret_cast<uint64_t*>(sP + NT * 2 * K1S_SR * PP);  // [NT][SP]
  uint64_t* pfull = full + NT * SP;                                          // [NT][2]
  uint64_t* pempty = pfull + NT * 2;                                         // [NT][2]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int rb = blockIdx.x % prm.rbs;
  const int pg = blockIdx.x / prm.rbs;
  const int col0 = rb * CW;

  if (4 * KH > ldv)
    for (size_t idx = threadIdx.x; idx < (size_t)NT * SP * slab_elems; idx += blockDim.x)
      ring[idx] = 0.0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NT * SP; ++s) mbar_init(&full[s], 1);
    for (int s = 0; s < NT * 2; ++s) {
      mbar_init(&pfull[s], 64);    // G1a and G1b
      mbar_init(&pempty[s], 32);   // G2
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");

  // warp w sits on sub-partition w % 4: triad q = w % 4 lives on sub-partition q, role = w / 4
  const int role = warp >> 2;   // 0: G1a (DMMA columns), 1: G1b (DFMA tail), 2: G2
  const int q = warp & 3;
  const int64_t my_slabs =
      pg < prm.num_slabs ? (prm.num_slabs - pg + prm.gp - 1) / prm.gp : 0;
  const int64_t n_mine = my_slabs > q ? (my_slabs - q + NT - 1) / NT : 0;
  const uint32_t slab_bytes = (uint32_t)(slab_elems * sizeof(double));
  double* my_ring = ring + (size_t)q * SP * slab_elems;
  uint64_t* my_full = full + q * SP;
  uint64_t* my_pfull = pfull + q * 2;
  uint64_t* my_pempty = pempty + q * 2;
  double* my_P = sP + (size_t)q * 2 * K1S_SR * PP;
  const int64_t slab_stride = (int64_t)NT * prm.gp * K1S_SR * ldv;
  const double* src0 = prm.V + ((int64_t)pg + (int64_t)q * prm.gp) * K1S_SR * ldv;
  if (role == 2 && lane == 0) {
    for (int s = 0; s < SP && s < n_mine; ++s) {
      mbar_arrive_expect_tx(&my_full[s], slab_bytes);
      tma_bulk_g2s(my_ring + (size_t)s * slab_elems, src0 + s * slab_stride, slab_bytes,
                   &my_full[s]);
    }
    for (int a = 0; a < MCP_K1Q_L2_AHEAD; ++a)
      if (SP + a < n_mine) l2_prefetch_bulk(src0 + (SP + a) * slab_stride, slab_bytes);
  }
  // PDL: the prologue above depends only on V; x may come from the previous kernel
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  {
    constexpr int NAF = KH * NTM * 32, NAT = KH * 16;
    constexpr int PER = (NAF + NAT + K1R_THREADS - 1) / K1R_THREADS;
    double av[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int idx = threadIdx.x + u * K1R_THREADS;
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
      const int idx = threadIdx.x + u * K1R_THREADS;
      if (idx < NAF)
        sAf[idx] = av[u];
      else if (idx < NAF + NAT)
        sAt[idx - NAF] = av[u];
    }
  }
  __syncthreads();
  const int dm1 = prm.d - 1;
  const int MT = prm.MT;
  double* wst = ring + (size_t)NT * MT * 8 * CW + q * CW;   // final staging (after the loop)

  if (role == 0) {
    // ================= G1a: DMMA columns of Z, their epilogue =================
    double wacc[NTM][2];
#pragma unroll
    for (int nt = 0; nt < NTM; ++nt) wacc[nt][0] = wacc[nt][1] = 0.0;
    int s = 0;
    uint32_t ph = 0;
    for (int64_t i = 0; i < n_mine; ++i) {
      mbar_wait(&my_full[s], ph);
      const double* sv = my_ring + (size_t)s * slab_elems;
      if (++s == SP) {
        s = 0;
        ph ^= 1;
      }
      const int64_t row0 = ((int64_t)pg + (q + i * NT) * (int64_t)prm.gp) * K1S_SR;
      double z[2][NTM][2];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < NTM; ++nt) z[mt][nt][0] = z[mt][nt][1] = 0.0;
      const double* v0 = sv + g * ldv + t;
      const double* v1 = v0 + 8 * ldv;
      const double* bp = sAf + lane;
#pragma unroll
      for (int kk = 0; kk < KH; ++kk) {
        const double a0 = v0[4 * kk], a1 = v1[4 * kk];
#pragma unroll
        for (int nt = 0; nt < NTM; ++nt) {
          const double b = bp[(kk * NTM + nt) * 32];
          dmma884(z[0][nt], a0, b);
          dmma884(z[1][nt], a1, b);
        }
      }
      const int b = (int)(i & 1);
      if (i >= 2) mbar_wait(&my_pempty[b], (uint32_t)(((i - 2) >> 1) & 1));
      double* Pb = my_P + (size_t)b * K1S_SR * PP;
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const int lr = 8 * mt + g;
        const double nul = prm.nu ? prm.nu[row0 + lr] : prm.nu_const;
        constexpr int NV = 2 * NTM;
        double zv[NV], pw[NV];
#pragma unroll
        for (int nt = 0; nt < NTM; ++nt) {
          zv[2 * nt] = z[mt][nt][0];
          zv[2 * nt + 1] = z[mt][nt][1];
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
      }
      mbar_arrive(&my_pfull[b]);
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
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    __syncthreads();   // (A) all slabs consumed
    if (g == 0) {
#pragma unroll
      for (int nt = 0; nt < NTM; ++nt) {
        wst[8 * nt + 2 * t] = wacc[nt][0];
        wst[8 * nt + 2 * t + 1] = wacc[nt][1];
      }
    }
  } else if (role == 1) {
    // ================= G1b: DFMA tail columns of Z, their epilogue =================
    double wtl = 0.0;
    int s = 0;
    uint32_t ph = 0;
    for (int64_t i = 0; i < n_mine; ++i) {
      mbar_wait(&my_full[s], ph);
      const double* sv = my_ring + (size_t)s * slab_elems;
      if (++s == SP) {
        s = 0;
        ph ^= 1;
      }
      const int64_t row0 = ((int64_t)pg + (q + i * NT) * (int64_t)prm.gp) * K1S_SR;
      double zt[2][TAIL];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int c = 0; c < TAIL; ++c) zt[mt][c] = 0.0;
      const double* v0 = sv + g * ldv + t;
      const double* v1 = v0 + 8 * ldv;
      const double* at = sAt + t * 4;
#pragma unroll
      for (int kk = 0; kk < KH; ++kk) {
        const double a0 = v0[4 * kk], a1 = v1[4 * kk];
        const double2 tc = *reinterpret_cast<const double2*>(at + 16 * kk);
        zt[0][0] = fma(a0, tc.x, zt[0][0]);
        zt[1][0] = fma(a1, tc.x, zt[1][0]);
        if constexpr (TAIL > 1) {
          zt[0][TAIL - 1] = fma(a0, tc.y, zt[0][TAIL - 1]);
          zt[1][TAIL - 1] = fma(a1, tc.y, zt[1][TAIL - 1]);
        }
      }
      const int b = (int)(i & 1);
      if (i >= 2) mbar_wait(&my_pempty[b], (uint32_t)(((i - 2) >> 1) & 1));
      double* Pb = my_P + (size_t)b * K1S_SR * PP;
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const int lr = 8 * mt + g;
        const double nul = prm.nu ? prm.nu[row0 + lr] : prm.nu_const;
        double zmine = 0.0;
#pragma unroll
        for (int c = 0; c < TAIL; ++c) {
          double zz = zt[mt][c];
          zz += __shfl_xor_sync(0xffffffffu, zz, 1);
          zz += __shfl_xor_sync(0xffffffffu, zz, 2);
          if (t == c) zmine = zz;
        }
        if (t < TAIL) {
          const double pv = nul * rm_pow(zmine, dm1);
          wtl = fma(pv, zmine, wtl);
          Pb[lr * PP + 8 * NTM + t] = pv;
        }
      }
      mbar_arrive(&my_pfull[b]);
    }
    wtl += __shfl_xor_sync(0xffffffffu, wtl, 4);
    wtl += __shfl_xor_sync(0xffffffffu, wtl, 8);
    wtl += __shfl_xor_sync(0xffffffffu, wtl, 16);
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    __syncthreads();   // (A)
    if (g == 0 && t < TAIL) wst[8 * NTM + t] = wtl;
  } else {
    // ================= G2: Y over all m-tiles, ring refills =================
    double yacc[MT2][NTM][2];
    double ytl[MT2][TAIL];
#pragma unroll
    for (int m = 0; m < MT2; ++m) {
#pragma unroll
      for (int nt = 0; nt < NTM; ++nt) yacc[m][nt][0] = yacc[m][nt][1] = 0.0;
#pragma unroll
      for (int c = 0; c < TAIL; ++c) ytl[m][c] = 0.0;
    }
    int s = 0;
    uint32_t ph = 0;
    for (int64_t i = 0; i < n_mine; ++i) {
      const int b = (int)(i & 1);
      mbar_wait(&my_full[s], ph);
      mbar_wait(&my_pfull[b], (uint32_t)((i >> 1) & 1));
      const double* sv = my_ring + (size_t)s * slab_elems;
      const double* Pb = my_P + (size_t)b * K1S_SR * PP;
#pragma unroll
      for (int k2 = 0; k2 < K1S_SR / 4; ++k2) {
        const double* prow = Pb + (4 * k2 + t) * PP;
        double bb[NTM], bt[TAIL];
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
    __syncthreads();   // (A)
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
  const int per_cta = MT * 8 * CW;
  double* Yp = prm.Ypart + ((size_t)rb * prm.gp + pg) * per_cta;
  for (int e = threadIdx.x; e < per_cta; e += blockDim.x) {
    double acc = 0.0;
#pragma unroll
    for (int w = 0; w < NT; ++w) acc += ring[(size_t)w * per_cta + e];
    Yp[e] = acc;
  }
  if (threadIdx.x < CW) {
    double acc = 0.0;
#pragma unroll
    for (int w = 0; w < NT; ++w) acc += ring[(size_t)NT * per_cta + w * CW + threadIdx.x];
    prm.wpart[((size_t)rb * prm.gp + pg) * CW + threadIdx.x] = acc;
  }
}

}  // namespace mcp
