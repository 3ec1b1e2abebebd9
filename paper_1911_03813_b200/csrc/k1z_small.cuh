// K1Z: the whole f+grad evaluation of a SMALL problem in ONE launch (config 1, the mini-batches
// and estimate subsets of the stochastic path).
//
// Reference path: ttsv_batch (pkg/src/momentcp/implicit.py:94-107), model_data_inner
// (implicit.py:124-140), build_gram_cache (implicit.py:143-151), _finish (objective.py:51-56),
// and -- with an index list -- sample_observations' row gather (objective.py:97-113).
//
// These evaluations are launch / latency bound (a few MFLOP): the K1Q -> K3F chain spends its
// time in launches, mbarrier and tensor-map set-up and the hand-over between kernels.  K1Z is a
// cooperative grid of up to one CTA per SM:
//   1. CTA b takes a contiguous range of rows and starts their cp.async copies into shared
//      memory (rows read straight from the resident set through an optional index list: no
//      gathered copy).  While they fly it stages A and lam, forms G = A^T A, C = G^(d-1), the
//      M = (A o lam) C entries of the outputs it will finish and (last CTA) u -- everything that
//      depends on x alone;
//   2. Z = V A by DMMA.8x8x4 in passes of 8 / 16 / 32 rows, k split over the 8 warps and the
//      partial Z summed in warp order through shared memory (plain DFMA loops measured bound by
//      shared-memory wavefronts: 13 FMA per wavefront against 64 for DMMA fragments);
//      P = nu Z^(d-1) and its share of w; then Y_b = V^T P by DMMA, warp w owning the 8-variable
//      tiles w, w + 8, ... with Y_b in registers across passes and slabs;
//   3. writes [Y_b ; w_b] to its partial slot and arrives on a grid barrier (bounded spin);
//   4. after the barrier the outputs are split over the CTAs: each output sums its G partials
//      in a fixed (slot-strided, then sequential) order and is finished in place --
//      g_A = -2d (Y - M) o lam, and on the last CTA g_lam = -2 (w - u), f = alpha + lam.u - 2 w.lam.
// The split and every summation order depend on (p, n, r, SM count) only, so evaluations are
// bitwise reproducible and independent of how the rows got there (uploaded set, gathered view or
// index list).
#pragma once

#include "mcp_common.cuh"
#include "tail_pieces.cuh"
#include "tuning.h"
#include "pdl.h"
#if MCP_K1Z_PROF
#include <cstdio>
#endif

namespace mcp {

constexpr int K1Z_T = 256;
constexpr int K1Z_MAXR = 32;
constexpr int K1Z_MAXN = 512;

// Optional Adam update fused into the finish (stochastic path, optimize.py:425-430): after the
// grid barrier nobody reads x from global memory any more (every CTA staged it before arriving),
// so the thread that finishes gradient entry k also updates m1[k], m2[k] and x[k] in place, in
// the reference's operation order with explicit round-to-nearest operations.
struct K1ZAdam {
  double* x = nullptr;            // the packed variables (same buffer K1ZParams::x reads)
  double* m1 = nullptr;
  double* m2 = nullptr;
  const double* bc = nullptr;     // bc[2 it], bc[2 it + 1] = 1 - b1^t, 1 - b2^t
  const double* lr = nullptr;
  int* it = nullptr;              // iteration cursor, advanced by the last CTA
  double b1 = 0, omb1 = 0, b2 = 0, omb2 = 0, eps = 0;
};

struct K1ZParams {
  const void* V = nullptr;        // observation-major rows, pitch ldv elements
  int64_t ldv = 0;
  const int64_t* idx = nullptr;   // optional: row l of the problem is row idx[base + l] of V
  const int* it_dev = nullptr;    // optional: base = *it_dev * p (the stochastic path's cursor)
  const double* nu = nullptr;     // weights by row of V, or nu_const for every row
  double nu_const = 0.0;
  const double* x = nullptr;      // [lam ; vec_F(A)]
  const double* alpha_dev = nullptr;
  double alpha_host = 0.0;
  double* part = nullptr;         // [G][PS] partial slots
  unsigned* bar = nullptr;        // [0] arrivals, [1] generation, [2] error flag
  double* out = nullptr;          // [f ; g_lam ; vec_F(g_A)]
  int64_t p = 0;
  int n = 0, r = 0, d = 0;
  int rows_per_cta = 0;           // contiguous rows per CTA (multiple of the pass height)
  int R = 0;                      // slab rows staged at once (multiple of the pass height)
  int ns = 0;                     // shared-memory row pitch of a staged row (elements)
  int np = 0;                     // shared-memory pitch of a factor column (doubles, odd)
  int PS = 0;                     // partial slot pitch (doubles)
  K1ZAdam adam;                   // adam.x == nullptr: no fused update
  int Gp = 0;                     // CTAs that own rows (partial slots); CTAs Gp .. gridDim - 1 only
                                  // take a share of the finish (tiny batches: few row CTAs)
};

__device__ __forceinline__ unsigned long long k1z_now_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;\n" : "=l"(t));
  return t;
}

// Fixed-order sum over the G partial slots of outputs e0 .. e0 + cnt - 1, handed to fin(e, sum)
// by one thread per output.  GP lanes per output stride the slots (g = q, q + GP, ...: loads of
// sixteen slots in flight), then the GP lane sums are added sequentially.
template <class F>
__device__ __forceinline__ void k1z_reduce(const double* part, int PS, int G, int e0, int cnt,
                                           double* sR, F&& fin) {
  int GP = 1;
  while (GP < 32 && GP * 2 * cnt <= K1Z_T && GP * 2 <= G) GP *= 2;
  const int EC = K1Z_T / GP;
  const int el = threadIdx.x % EC, q = threadIdx.x / EC;
  for (int base = 0; base < cnt; base += EC) {
    const bool valid = base + el < cnt;
    const int e = e0 + base + el;
    double s = 0.0;
    if (valid) {
      for (int g0 = q; g0 < G; g0 += 16 * GP) {
        double t[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int g = g0 + u * GP;
          t[u] = g < G ? __ldcg(part + (int64_t)g * PS + e) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) s += t[u];
      }
    }
    sR[q * EC + el] = s;
    __syncthreads();
    if (q == 0 && valid) {
      double tot = sR[el];
      for (int qq = 1; qq < GP; ++qq) tot += sR[qq * EC + el];
      fin(e, tot);
    }
    __syncthreads();
  }
}

// TV: element type of V.  RP: padded factor columns (8, 16 or 32).  MT1: 8-row DMMA tiles per
// GEMM1 pass (a pass covers 8 MT1 rows).
#if MCP_K1Z_PROF
#define K1Z_STAMP(k) do { if (threadIdx.x == 0) stamps[k] = clock64(); } while (0)
#else
#define K1Z_STAMP(k) do { } while (0)
#endif

constexpr int K1Z_NW = K1Z_T / 32;
// doubles of the partial-sum area: NW GEMM1 pass partials or NW / 2 slots of the factor Gram
__host__ __device__ constexpr int k1z_sz_elems(int RP, int MT1) {
  return (K1Z_NW * 8 * MT1 * RP) > (K1Z_NW / 2 * RP * RP) ? (K1Z_NW * 8 * MT1 * RP)
                                                          : (K1Z_NW / 2 * RP * RP);
}
constexpr int K1Z_MAXMT = K1Z_MAXN / 8 / K1Z_NW;   // GEMM2 m-tiles per warp

template <typename TV, int RP, int MT1>
__global__ void __launch_bounds__(K1Z_T) k1z_fg_small(const K1ZParams a) {
  constexpr int NT = RP / 8;      // 8-column DMMA tiles
  constexpr int RS = 8 * MT1;     // rows per GEMM1 pass
  constexpr int NW = K1Z_NW;
#if MCP_K1Z_PROF
  long long stamps[12];
  K1Z_STAMP(0);
#endif
  extern __shared__ __align__(16) unsigned char k1z_smem[];
  const int tid = threadIdx.x, G = gridDim.x, b = blockIdx.x;
  const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int n = a.n, r = a.r, d = a.d, ns = a.ns, np = a.np, R = a.R;
  const int n4 = (n + 3) & ~3;
#if MCP_K1Z_KO & 2
  if (a.n > 0) return;
#endif
  // the factor, column-major with an odd pitch (zero padded to np rows and RP columns):
  // conflict-free across variables (the fill, M) and across the 8 x 4 DMMA fragment lanes
  double* sAT = reinterpret_cast<double*>(k1z_smem);         // [RP][np]
  double* sP = sAT + (size_t)RP * np;                         // [R][RP]
  double* sZ = sP + (size_t)R * RP;                           // partials: [NW][RS][RP] of a GEMM1
                                                              // pass, [NW / 2][RP][RP] of G
  double* sW = sZ + k1z_sz_elems(RP, MT1);                    // [256]
  double* sG = sW + K1Z_T;                                    // [r][r]
  double* sC = sG + RP * RP;                                  // [r][r]
  double* sR = sC + RP * RP;                                  // [256] reduce lanes
  double* sM = sR + K1Z_T;                                    // [256] M entries of my outputs
  double* sL = sM + K1Z_T;                                    // [RP] lam, zero padded
  double* sS = sL + RP;                                       // [2 RP] w, u of the finish
  TV* sV = reinterpret_cast<TV*>(sS + 2 * RP);                // [R][ns] (+ 8 elements of slack)
  const double* __restrict__ A = a.x + r;

  // under programmatic dependent launch the grid may be resident before its predecessor (the
  // previous iteration's update kernel) has finished: nothing of x, the cursor or the index
  // list is read before this wait (a no-op for a plain launch)
  pdl_wait();
  const int64_t base = (a.idx && a.it_dev) ? (int64_t)(*a.it_dev) * a.p : 0;
  const int it0 = a.adam.x ? *a.adam.it : 0;
  const int64_t row_lo = (int64_t)b * a.rows_per_cta;
  const int64_t row_hi = min(a.p, row_lo + a.rows_per_cta);
  constexpr int EPC = 16 / (int)sizeof(TV);          // elements per 16-byte chunk
  const int CH = n4 / EPC;                            // the source rows are zero padded past n
  auto issue_slab = [&](int64_t row0, int rows) {
    for (int c = tid; c < rows * CH; c += K1Z_T) {
      const int l = c / CH, k = c % CH;
      const int64_t grow = a.idx ? a.idx[base + row0 + l] : row0 + l;
      cp_async16(sV + (size_t)l * ns + k * EPC,
                 reinterpret_cast<const TV*>(a.V) + grow * a.ldv + k * EPC, 16);
    }
    cp_async_commit();
    // rows of the last pass beyond the range: zeros (their P is zero; 0 x stale could be NaN)
    const int pad_to = min(R, (rows + RS - 1) / RS * RS);
    for (int c = rows * ns + tid; c < pad_to * ns; c += K1Z_T) sV[c] = TV(0);
  };
  // ---- the first slab's rows in flight; everything that depends on x alone meanwhile ----
  if (row_lo < row_hi) issue_slab(row_lo, (int)min((int64_t)R, row_hi - row_lo));
  // coalesced column reads: the loads of all r columns of two variables in flight before the
  // stores (every CTA reads the same lines of L2 at once: ~2.3k cycles per round trip)
  for (int i0 = tid; i0 < np; i0 += 2 * K1Z_T) {
    double v[2][RP];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int j = 0; j < RP; ++j) {
        const int i = i0 + h * K1Z_T;
        v[h][j] = (j < r && i < n) ? A[(int64_t)j * n + i] : 0.0;
      }
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int j = 0; j < RP; ++j) {
        const int i = i0 + h * K1Z_T;
        if (j < r && i < np) sAT[(size_t)j * np + i] = v[h][j];
      }
  }
  for (int e = r * np + tid; e < RP * np; e += K1Z_T) sAT[e] = 0.0;   // padded columns
  if (tid < RP) sL[tid] = tid < r ? a.x[tid] : 0.0;
  __syncthreads();
  K1Z_STAMP(9);
  {
    // G = A^T A by DMMA: the fragment A^T[j0 + g][4 ks + t] is both the row operand of tile row
    // j0 and the column operand of tile column j0; k-steps strided over the warps, partial
    // tiles summed in warp order; upper tiles only, mirrored.  C = G^(d-1) by repeated
    // multiplication (implicit.py:82-91, 147-148).
    double cg[NT][NT][2];
#pragma unroll
    for (int jt = 0; jt < NT; ++jt)
#pragma unroll
      for (int kt = 0; kt < NT; ++kt) cg[jt][kt][0] = cg[jt][kt][1] = 0.0;
    for (int ks = warp; ks < n4 / 4; ks += NW) {
      double f[NT];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) f[nt] = sAT[(size_t)(nt * 8 + g) * np + 4 * ks + t];
#pragma unroll
      for (int jt = 0; jt < NT; ++jt)
#pragma unroll
        for (int kt = jt; kt < NT; ++kt) dmma884(cg[jt][kt], f[jt], f[kt]);
    }
    // partial tiles of warps 0..3 stored, those of warps 4..7 added onto them (slot w - 4 is
    // touched by one warp per round), then the four slots summed in order
    {
      double* slot = sZ + (size_t)(warp & (NW / 2 - 1)) * RP * RP;
      if (warp < NW / 2) {
#pragma unroll
        for (int jt = 0; jt < NT; ++jt)
#pragma unroll
          for (int kt = jt; kt < NT; ++kt)
            *reinterpret_cast<double2*>(slot + (size_t)(jt * 8 + g) * RP + kt * 8 + 2 * t) =
                make_double2(cg[jt][kt][0], cg[jt][kt][1]);
      }
      __syncthreads();
      if (warp >= NW / 2) {
#pragma unroll
        for (int jt = 0; jt < NT; ++jt)
#pragma unroll
          for (int kt = jt; kt < NT; ++kt) {
            double2* q = reinterpret_cast<double2*>(slot + (size_t)(jt * 8 + g) * RP + kt * 8 + 2 * t);
            const double2 o = *q;
            *q = make_double2(o.x + cg[jt][kt][0], o.y + cg[jt][kt][1]);
          }
      }
    }
    __syncthreads();
    for (int e = tid; e < r * r; e += K1Z_T) {
      const int j = e / r, k = e % r;
      if (j > k) continue;
      double s = sZ[(size_t)j * RP + k];
      for (int w = 1; w < NW / 2; ++w) s += sZ[((size_t)w * RP + j) * RP + k];
      const double c = rm_pow(s, d - 1);
      sG[j * r + k] = s;
      sG[k * r + j] = s;
      sC[j * r + k] = c;
      sC[k * r + j] = c;
    }
  }
  __syncthreads();
  K1Z_STAMP(10);
  // my outputs of the finish: entries e0 .. e1 - 1 of vec_F(g_A); the last CTA also takes w
  const int n_out = n * r;
  const int chunk = (n_out + G - 1) / G;
  const int e0 = min(n_out, b * chunk), e1 = min(n_out, e0 + chunk);
  auto m_entry = [&](int e) {   // M_ij = sum_k (A_ik lam_k) C_kj (objective.py:55)
    const int j = e / n, i = e % n;
    double m = 0.0;
    for (int k = 0; k < r; ++k) m += (sAT[(size_t)k * np + i] * sL[k]) * sC[k * r + j];
    return m;
  };
  if (tid < e1 - e0) sM[tid] = m_entry(e0 + tid);
  double* s_w = sS;
  double* s_u = sS + RP;
  if (b == G - 1 && tid < r) s_u[tid] = tail_u_entry(sG, sC, sL, r, tid);

  double wacc = 0.0;              // this thread's share of w_(tid % RP)
  double acc[K1Z_MAXMT][NT][2];   // Y_b tiles (8 warp + m) of this warp
#pragma unroll
  for (int m = 0; m < K1Z_MAXMT; ++m)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[m][nt][0] = acc[m][nt][1] = 0.0;
  const int n_mt = (n + 7) / 8;
  K1Z_STAMP(1);

  for (int64_t row0 = row_lo; row0 < row_hi; row0 += R) {
    const int rows = (int)min((int64_t)R, row_hi - row0);
    if (row0 != row_lo) {
      __syncthreads();   // the previous slab's GEMM2 is done with sV / sP
      issue_slab(row0, rows);
    }
    cp_async_wait<0>();
    __syncthreads();
    K1Z_STAMP(2);
    // ---- GEMM1 + epilogue per pass: z = v_l . a_j, P = nu z^(d-1), w += P z ----
    for (int sub0 = 0; sub0 < rows; sub0 += RS) {
      double cz[2][MT1][NT][2];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int mt = 0; mt < MT1; ++mt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) cz[h][mt][nt][0] = cz[h][mt][nt][1] = 0.0;
      const TV* vrow = sV + (size_t)(sub0 + g) * ns + t;
      const double* acol = sAT + (size_t)g * np + t;
      auto kstep = [&](int ks, int h) {
        double fb[NT], fa[MT1];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) fb[nt] = acol[(size_t)nt * 8 * np + 4 * ks];
#pragma unroll
        for (int mt = 0; mt < MT1; ++mt) fa[mt] = to_f64(vrow[(size_t)mt * 8 * ns + 4 * ks]);
#pragma unroll
        for (int mt = 0; mt < MT1; ++mt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) dmma884(cz[h][mt][nt], fa[mt], fb[nt]);
      };
      int ks = warp;
      for (; ks + NW < n4 / 4; ks += 2 * NW) {   // two accumulator sets: two chains per tile
        kstep(ks, 0);
        kstep(ks + NW, 1);
      }
      if (ks < n4 / 4) kstep(ks, 0);
#pragma unroll
      for (int mt = 0; mt < MT1; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
          *reinterpret_cast<double2*>(sZ + ((size_t)warp * RS + mt * 8 + g) * RP + nt * 8 + 2 * t) =
              make_double2(cz[0][mt][nt][0] + cz[1][mt][nt][0], cz[0][mt][nt][1] + cz[1][mt][nt][1]);
      __syncthreads();
      for (int e = tid; e < RS * RP; e += K1Z_T) {   // column e % RP == tid % RP on every trip
        const int row = e / RP, col = e % RP;
        double z = sZ[(size_t)row * RP + col];
        for (int w = 1; w < NW; ++w) z += sZ[((size_t)w * RS + row) * RP + col];
        const int l = sub0 + row;
        double pv = 0.0;
        if (l < rows) {
          double nul = a.nu_const;
          if (a.nu) nul = a.nu[a.idx ? a.idx[base + row0 + l] : row0 + l];
          pv = nul * rm_pow(z, d - 1);
          wacc += pv * z;
        }
        if (l < R) sP[(size_t)l * RP + col] = pv;
      }
      __syncthreads();   // P of this pass written; sZ free for the next pass
    }
    K1Z_STAMP(3);
    // ---- GEMM2: Y[8 m + g][:] += sum_l v_l[8 m + g] P[l][:], k-steps of 4 rows in order ----
    const int ksteps2 = (rows + 3) / 4;
    for (int ks = 0; ks < ksteps2; ++ks) {
      double fb[NT];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) fb[nt] = sP[(size_t)(4 * ks + t) * RP + nt * 8 + g];
      const TV* vk = sV + (size_t)(4 * ks + t) * ns + g;
#pragma unroll
      for (int m = 0; m < K1Z_MAXMT; ++m) {
        const int mt = warp + m * NW;
        if (mt < n_mt) {
          const double fa = to_f64(vk[mt * 8]);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) dmma884(acc[m][nt], fa, fb[nt]);
        }
      }
    }
  }
  __syncthreads();
  K1Z_STAMP(4);

  // ---- this CTA's partial [vec_F(Y_b) ; w_b] (row-owning CTAs only) ----
  const bool owner = b < a.Gp;
  double* mine = a.part + (int64_t)b * a.PS;
  sW[tid] = wacc;
#pragma unroll
  for (int m = 0; m < K1Z_MAXMT; ++m) {
    const int i = (warp + m * NW) * 8 + g;
    if (owner && i < n) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int j = nt * 8 + 2 * t + e;
          if (j < r) __stcg(mine + (int64_t)j * n + i, acc[m][nt][e]);
        }
    }
  }
  __syncthreads();
  if (owner && tid < r) {
    double s = sW[tid];
    for (int k = 1; k < K1Z_T / RP; ++k) s += sW[k * RP + tid];
    __stcg(mine + (int64_t)n * r + tid, s);
  }
#if MCP_K1Z_KO & 1
  if (a.n > 0) return;
#endif

  // ---- grid barrier ----
  K1Z_STAMP(5);
  bool failed = false;
  if (G > 1) {
    __threadfence();
    __syncthreads();
    K1Z_STAMP(6);
    if (tid == 0) {
      volatile unsigned* vgen = a.bar + 1;
      const unsigned gen = *vgen;
      __threadfence();
      if (atomicAdd(a.bar, 1u) == (unsigned)G - 1) {
        a.bar[0] = 0u;
        __threadfence();
        atomicAdd(a.bar + 1, 1u);
      } else {
        const unsigned long long t0 = k1z_now_ns();
        unsigned spins = 0;
        while (*vgen == gen) {
          if ((++spins & 1023u) == 0 && k1z_now_ns() - t0 > 4000000000ull) {
            atomicExch(a.bar + 2, 1u);   // 4 s: never under a cooperative launch
            break;
          }
        }
      }
      __threadfence();
    }
    __syncthreads();
    failed = *reinterpret_cast<volatile unsigned*>(a.bar + 2) != 0u;
  } else {
    __syncthreads();
    K1Z_STAMP(6);
  }
  K1Z_STAMP(7);
  // a dependent launched with the programmatic attribute (the Adam update) may become resident
  // now; it waits for this grid's completion before reading the gradient
  pdl_trigger();

  // ---- reduce + finish, outputs split over the CTAs ----
  const double s2d = -2.0 * d;
  const double bad = failed ? __longlong_as_double(0x7ff8000000000000ll) : 0.0;
  const int cnt = e1 - e0 + (b == G - 1 ? r : 0);   // the last CTA's entries end at n_out: w follows
  double bc1 = 1.0, bc2 = 1.0, lr = 0.0;
  if (a.adam.x) {
    bc1 = a.adam.bc[2 * it0];
    bc2 = a.adam.bc[2 * it0 + 1];
    lr = *a.adam.lr;
  }
  auto adam_update = [&](int k, double gk) {   // k_adam_step's arithmetic (csrc/adam.cu)
    const K1ZAdam& ad = a.adam;
    const double u = __dadd_rn(__dmul_rn(ad.b1, ad.m1[k]), __dmul_rn(ad.omb1, gk));
    const double v = __dadd_rn(__dmul_rn(ad.b2, ad.m2[k]), __dmul_rn(__dmul_rn(ad.omb2, gk), gk));
    ad.m1[k] = u;
    ad.m2[k] = v;
    const double mh = __ddiv_rn(u, bc1);
    const double vh = __ddiv_rn(v, bc2);
    ad.x[k] = __dsub_rn(ad.x[k], __ddiv_rn(__dmul_rn(lr, mh), __dadd_rn(__dsqrt_rn(vh), ad.eps)));
  };
  k1z_reduce(a.part, a.PS, a.Gp, e0, cnt, sR, [&](int e, double y) {
    if (e < n_out) {
      const double m = e - e0 < K1Z_T ? sM[e - e0] : m_entry(e);
      const double gk = (s2d * (y - m)) * sL[e / n] + bad;
      a.out[1 + r + e] = gk;
      if (a.adam.x) adam_update(r + e, gk);
    } else {
      const int j = e - n_out;
      s_w[j] = y;
      const double gk = -2.0 * (y - s_u[j]) + bad;
      a.out[1 + j] = gk;
      if (a.adam.x) adam_update(j, gk);
    }
  });
  if (b == G - 1 && tid == 0) {
    double lu = 0.0, wl = 0.0;
    for (int j = 0; j < r; ++j) lu += sL[j] * s_u[j];
    for (int j = 0; j < r; ++j) wl += s_w[j] * sL[j];
    const double alpha = a.alpha_dev ? *a.alpha_dev : a.alpha_host;
    a.out[0] = alpha + lu - 2.0 * wl + bad;
    if (a.adam.x) *a.adam.it = it0 + 1;
  }
#if MCP_K1Z_PROF
  K1Z_STAMP(8);
  if (tid == 0 && (b == 0 || b == G - 1 || b == G / 2))
    printf("k1z cta %d: fill %lld gc %lld m %lld | pre %lld load %lld g1 %lld g2 %lld comb %lld fence %lld bar %lld red %lld total %lld\n",
           b, stamps[9] - stamps[0], stamps[10] - stamps[9], stamps[1] - stamps[10],
           stamps[1] - stamps[0], stamps[2] - stamps[1], stamps[3] - stamps[2],
           stamps[4] - stamps[3], stamps[5] - stamps[4], stamps[6] - stamps[5],
           stamps[7] - stamps[6], stamps[8] - stamps[7], stamps[8] - stamps[0]);
#endif
}

}  // namespace mcp
