// K1X (FP64 mode, float32 observations, large n): 16 warps, double-buffered tiles, resident
// factor block.
//
// Same arithmetic as the other K1 kernels (reference pkg/src/momentcp/implicit.py:94-107 and the
// w of :124-140): per tile of T observations and an RB-column factor block
//   Z = V_tile A  (GEMM1, DMMA.8x8x4)  ->  P = nu Z^(d-1), w += P Z  ->  Y += V_tile^T P (GEMM2).
// Two shapes, both with a 64 KB tile and a 64 KB factor block:
//   NL = 512,  T = 32, RB = 16   (c3: n = 512, r = 64)
//   NL = 1024, T = 16, RB = 8    (c5: n = 1024, r = 256)
//
// Why this shape (tools/probe_dmma_lds.cu, the K1W ncu source profiles): the
// DMMA inner loops themselves run at 93-98% of the FP64 pipe with operands from shared memory,
// but with 2 warps per SM sub-partition every cross-warp dependency (factor ring, P, chunk
// refills) leaves one warp issuing alone while its partner waits, and a lone warp cannot keep
// the pipe full.  K1X therefore runs 4 warps per sub-partition (16 warps; Y is NL / 16 x RB per
// warp, 32 doubles) and removes the waits that are not data dependencies:
//
//  * the factor block (NL x RB, fragment order) is loaded ONCE per column block with one bulk copy
//    and stays resident -- no factor ring;
//  * V is double-buffered: one 3-D TMA per tile lands its NL / 32 chunks (T rows x 32 floats,
//    128-byte swizzle) of tile u + 2 while tile u + 1 is computed; the last warp to finish
//    tile u's GEMM2 issues it (counter, nobody waits);
//  * GEMM1 is split over KS = 16 / (T / 8) K-slices (warp = row block x slice, 1 x NT DMMA tiles,
//    the KS warps of a row block spread over the sub-partitions); the partial Z are merged
//    through shared memory in slice order (one named barrier per row block) and the row block's
//    warps form P element by element, publishing it on the row block's mbarrier;
//  * GEMM2: warp w owns variables w NL/16 .. (w+1) NL/16 - 1 (NL/128 x NT DMMA tiles, Y in
//    registers), starts with its own row block and waits only for row blocks it has not seen.
// Fixed-order merges and per-element ownership keep results deterministic and exactly linear
// in nu.  A 2-CTA cluster form (each CTA half of n, half-Z exchanged through distributed shared
// memory per tile) measured 69% at c5 (the pair waits for its slower SM every tile) and was
// dropped for the NL = 1024 shape (git history).
#pragma once

#include <cuda.h>

#include "k1_dispatch.h"
#include "k1s_fp64.cuh"    // mbarrier helpers
#include "k1x_common.cuh"  // work split, proxy fence, ordered shared loads
#include "mcp_common.cuh"
#include "pdl.h"
#include "umma.cuh"        // TMA helpers

namespace mcp {

constexpr int K1X_THREADS = 512;      // 16 warps
constexpr int K1X_TILE_BYTES = 65536; // V tile (T x NL floats)
constexpr int K1X_A_BYTES = 65536;    // factor fragments (NL x RB doubles)

template <int NL, int T, int RB>
struct K1XShape {
  static_assert(T * NL * 4 == K1X_TILE_BYTES && NL * RB * 8 == K1X_A_BYTES, "64 KB tiles");
  static constexpr int C = NL / 32;        // 32-variable chunks per tile
  static constexpr int RBK = T / 8;        // GEMM1 row blocks
  static constexpr int KS = 16 / RBK;      // GEMM1 K-slices (warps per row block)
  static constexpr int CPS = C / KS;       // chunks per K-slice
  static constexpr int NT = RB / 8;        // column tiles
  static constexpr int MTW = NL / 128;     // GEMM2 m-tiles per warp (NL / 16 variables)
  static constexpr int SP = RB + 2;        // P row pitch (doubles), == 2 mod 16
  static constexpr int EL = 8 * RB;        // epilogue elements per row block
  static constexpr uint32_t CHUNK_BYTES = T * 128;   // one 32-float chunk of the tile
  static constexpr int ZM = RBK * KS * 8 * RB;       // Z merge slots (doubles)
};

template <int NL, int T, int RB>
__host__ __device__ constexpr size_t k1x_smem_bytes() {
  using S = K1XShape<NL, T, RB>;
  // (the w flush scratch aliases the Z merge slots)
  return 1024 /*alignment*/ + 2 * (size_t)K1X_TILE_BYTES + K1X_A_BYTES +
         2 * (size_t)T * S::SP * 8 /*P*/ +
         (size_t)(S::ZM > K1X_THREADS ? S::ZM : K1X_THREADS) * 8 /*Z merge / w flush*/ +
         512 /*barriers*/;
}

__device__ __forceinline__ void k1x_bar_rowblock(int rbk, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(1 + rbk), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void k1x_bar_all() {
  asm volatile("bar.sync 15, %0;\n" ::"n"(K1X_THREADS) : "memory");
}

// tmV: 3-D map over the fp32 observations viewed as (32 floats, rows, ldv / 32 chunks), box
// (32, T, NL / 32), 128-byte swizzle.  K1WParams: n_pad = NL.
template <int NL, int T, int RB>
__global__ void __launch_bounds__(K1X_THREADS, 1)
    k1x_fg_dmma(const __grid_constant__ CUtensorMap tmV, K1WParams prm) {
  using S = K1XShape<NL, T, RB>;
  constexpr int NT = S::NT, SP = S::SP, MTW = S::MTW;
  extern __shared__ __align__(16) unsigned char k1x_smem_raw[];
  unsigned char* base =
      k1x_smem_raw + ((1024u - (smem_u32(k1x_smem_raw) & 1023u)) & 1023u);
  float* sV = reinterpret_cast<float*>(base);                                   // [2][C][T][32]
  double* sA = reinterpret_cast<double*>(base + 2 * (size_t)K1X_TILE_BYTES);    // [NL/4 ks][NT][32]
  double* sP = sA + K1X_A_BYTES / 8;                                            // [2][T][SP]
  double* sZm = sP + 2 * T * SP;                                                // [RBK][KS][8][RB]
  double* sW = sZm;                                                             // [512] flush
  uint64_t* fullV =
      reinterpret_cast<uint64_t*>(sZm + (S::ZM > K1X_THREADS ? S::ZM : K1X_THREADS));  // [2]
  uint64_t* fullA = fullV + 2;                                                  // [1]
  uint64_t* fullP = fullA + 1;                                                  // [2][RBK]
  unsigned* cntV = reinterpret_cast<unsigned*>(fullP + 2 * S::RBK);             // [2]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int rbk = warp / S::KS;    // GEMM1 row block (tile rows 8 rbk .. +7)
  const int kq = warp % S::KS;     // GEMM1 K-slice (chunks CPS kq .. CPS kq + CPS - 1)
  const int cid = blockIdx.x;
  const int dm1 = prm.d - 1;

  if (threadIdx.x == 0) {
    mbar_init(&fullV[0], 1);
    mbar_init(&fullV[1], 1);
    mbar_init(fullA, 1);
    for (int i = 0; i < 2 * S::RBK; ++i) mbar_init(&fullP[i], S::KS);   // the row block's warps
    cntV[0] = cntV[1] = 0;
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    tma_prefetch_desc(&tmV);
  }
  __syncthreads();

  K1WTile cur;
  const bool any = k1w_tile_at(prm, cid, 0, cur);
  if (any && threadIdx.x == 0) {
    // V never changes: the first two tiles load before the factor prep kernel is waited for
    for (int b = 0; b < 2; ++b) {
      K1WTile tb;
      if (!k1w_tile_at(prm, cid, b, tb)) break;
      mbar_arrive_expect_tx(&fullV[b], K1X_TILE_BYTES);
      tma_load_3d(sV + (size_t)b * (K1X_TILE_BYTES / 4), &tmV, 0, (int)(tb.tile * T), 0,
                  smem_u32(&fullV[b]));
    }
  }
  pdl_enter();   // Afrag comes from the preceding prep kernel
  auto load_a = [&](int rb) {
    mbar_arrive_expect_tx(fullA, K1X_A_BYTES);
    tma_bulk_g2s(sA, prm.Afrag + (size_t)rb * (K1X_A_BYTES / 8), K1X_A_BYTES, fullA);
  };
  if (any && threadIdx.x == 0) load_a(cur.rb);
  uint32_t aphase = 0;
  int a_rb = any ? cur.rb : -1;

  // per-lane shared-memory offsets (bytes)
  // GEMM1: row 8 rbk + g of a chunk, k = 4 ks + t -> 16-byte unit ks ^ g
  uint32_t v1off[8];
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) v1off[ks] = 4u * ((8 * rbk + g) * 32 + ((ks ^ g) << 2) + t);
  // GEMM2: column 8 mt + g of a chunk at row 2t + p (+ 8 blk)
  uint32_t v2off[2][4];
#pragma unroll
  for (int p = 0; p < 2; ++p)
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
      v2off[p][mt] = 4u * ((2 * t + p) * 32 + (((2 * mt + (g >> 2)) ^ (2 * t + p)) << 2) + (g & 3));
  const uint32_t sV_u = smem_u32(sV), sA_u = smem_u32(sA) + 8u * lane;

  double y[MTW][NT][2];
#pragma unroll
  for (int mt = 0; mt < MTW; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) y[mt][nt][0] = y[mt][nt][1] = 0.0;
  double wacc = 0.0;   // this lane's epilogue element column (if it owns an element)
  const int e_idx = kq * 32 + lane;                 // element of its row block
  const bool e_own = e_idx < S::EL;
  const int e_row = e_idx / RB, e_col = e_idx % RB;

  int64_t it = 0;
  while (any) {
    const int buf = (int)(it & 1);
    const uint32_t vpar = (uint32_t)((it >> 1) & 1);
    const int64_t row0 = cur.tile * T;
    K1WTile nxt;
    const bool has_next = k1w_tile_at(prm, cid, it + 1, nxt);
    if (cur.rb != a_rb) {
      // a new column block (block-major ranges only): every warp is past its GEMM1 of the
      // previous tile, so the resident factor block can be replaced
      k1x_bar_all();
      if (threadIdx.x == 0) {
        k1w_fence_proxy_async();
        load_a(cur.rb);
      }
      aphase ^= 1u;
      a_rb = cur.rb;
    }
    mbar_wait(fullA, aphase);
    mbar_wait(&fullV[buf], vpar);
    const uint32_t vt = sV_u + (uint32_t)buf * K1X_TILE_BYTES;

    // ---------------- GEMM1: partial Z[8 rows x RB] over this warp's K-slice ----------------
    double z[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) z[nt][0] = z[nt][1] = 0.0;
    {
      float fa_n;
      double b_n[NT];
      auto load = [&](int cc, int ks) {   // cc: chunk within the K-slice
        const int c = S::CPS * kq + cc;
        fa_n = k1w_lds_f32(vt + (uint32_t)c * S::CHUNK_BYTES + v1off[ks]);
        const uint32_t ab = sA_u + 8u * (uint32_t)(((c * 8 + ks) * NT) * 32);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) b_n[nt] = k1w_lds_f64(ab + 256u * nt);
      };
      load(0, 0);
#pragma unroll
      for (int cc = 0; cc < S::CPS; ++cc)
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          const double a = (double)fa_n;
          double b[NT];
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) b[nt] = b_n[nt];
          if (ks < 7) load(cc, ks + 1);
          else if (cc < S::CPS - 1) load(cc + 1, 0);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) dmma884(z[nt], a, b[nt]);
        }
    }

    // ---------------- merge the K-slices, epilogue one element per lane ----------------
    {
      double* zm = sZm + (size_t)(rbk * S::KS + kq) * 8 * RB;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
        *reinterpret_cast<double2*>(&zm[g * RB + 8 * nt + 2 * t]) = make_double2(z[nt][0], z[nt][1]);
      k1x_bar_rowblock(rbk, 32 * S::KS);
      if (e_own) {
        const double* zr = sZm + (size_t)rbk * S::KS * 8 * RB + e_row * RB + e_col;
        double zz = zr[0];
#pragma unroll
        for (int q = 1; q < S::KS; ++q) zz += zr[q * 8 * RB];
        const int lr = 8 * rbk + e_row;
        const double nul = prm.nu ? prm.nu[row0 + lr] : prm.nu_const;
        const double pv = nul * rm_pow(zz, dm1);
        wacc += pv * zz;
        sP[(size_t)buf * T * SP + lr * SP + e_col] = pv;
      }
      // (the merge slots are rewritten next tile only after GEMM2, which waits for this row
      // block's P barrier -- i.e. for all of its warps to have read their partials)
      __syncwarp();
      if (lane == 0) mbar_arrive(&fullP[buf * S::RBK + rbk]);
    }

    // ---------------- GEMM2: Y[NL/16 variables x RB] += V^T P over the T tile rows ----------------
    {
      const uint32_t pbase = smem_u32(sP + (size_t)buf * T * SP + 2 * t * SP + g);
      float fa_n[MTW];
      double b_n[NT];
      auto load = [&](int blk, int p) {
        const uint32_t pk = pbase + 8u * (uint32_t)(blk * 8 * SP + p * SP);
#pragma unroll
        for (int mt = 0; mt < MTW; ++mt) {
          const uint32_t vc = vt + (uint32_t)(warp * (MTW / 4) + mt / 4) * S::CHUNK_BYTES;
          fa_n[mt] = k1w_lds_f32(vc + 1024u * (uint32_t)blk + v2off[p][mt % 4]);
        }
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) b_n[nt] = k1w_lds_f64(pk + 64u * nt);
      };
      mbar_wait(&fullP[buf * S::RBK + rbk], vpar);
      load(rbk, 0);
#pragma unroll
      for (int i = 0; i < S::RBK; ++i) {
        const int blk = (rbk + i) % S::RBK;
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          double a[MTW], b[NT];
#pragma unroll
          for (int mt = 0; mt < MTW; ++mt) a[mt] = (double)fa_n[mt];
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) b[nt] = b_n[nt];
          if (p == 0) load(blk, 1);
#pragma unroll
          for (int mt = 0; mt < MTW; ++mt)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) dmma884(y[mt][nt], a[mt], b[nt]);
          if (p == 1 && i < S::RBK - 1) {
            const int nb = (rbk + i + 1) % S::RBK;
            mbar_wait(&fullP[buf * S::RBK + nb], vpar);
            load(nb, 0);
          }
        }
      }
    }
    // the tile's V buffer is free once all 16 warps are past GEMM2: the last one refills it
    // with tile u + 2 (GEMM1 reads of it ended before each warp's P was published)
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      if (atomicAdd(&cntV[buf], 1u) == K1X_THREADS / 32 - 1) {
        cntV[buf] = 0;
        __threadfence_block();
        K1WTile t2;
        if (k1w_tile_at(prm, cid, it + 2, t2)) {
          k1w_fence_proxy_async();
          mbar_arrive_expect_tx(&fullV[buf], K1X_TILE_BYTES);
          tma_load_3d(sV + (size_t)buf * (K1X_TILE_BYTES / 4), &tmV, 0, (int)(t2.tile * T), 0,
                      smem_u32(&fullV[buf]));
        }
      }
    }

    // ---------------- end of a segment: flush this CTA's partial ----------------
    if (cur.last_in_seg || !has_next) {
      double* Yp = prm.Ypart + ((size_t)cur.rb * prm.slots + cur.slot) * prm.n_pad * RB;
#pragma unroll
      for (int mt = 0; mt < MTW; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          *reinterpret_cast<double2*>(
              &Yp[(size_t)(warp * (NL / 16) + 8 * mt + g) * RB + 8 * nt + 2 * t]) =
              make_double2(y[mt][nt][0], y[mt][nt][1]);
          y[mt][nt][0] = y[mt][nt][1] = 0.0;
        }
      // (sW aliases the Z merge slots: every warp is past this tile's merge reads)
      k1x_bar_all();
      sW[threadIdx.x] = e_own ? wacc : 0.0;
      wacc = 0.0;
      k1x_bar_all();
      if (threadIdx.x < RB) {
        // column j's partial sums sit at every thread whose element column is j, i.e. every
        // RB-th thread (element e = kq 32 + lane of each row block): added in thread order
        double s = 0.0;
        for (int q = 0; q < K1X_THREADS / RB; ++q) s += sW[q * RB + threadIdx.x];
        prm.wpart[((size_t)cur.rb * prm.slots + cur.slot) * RB + threadIdx.x] = s;
      }
      k1x_bar_all();
    }
    if (!has_next) break;
    cur = nxt;
    ++it;
  }
  k1w_zero_holes<K1X_THREADS, RB>(prm, cid, 0, NL, true);
}

}  // namespace mcp
