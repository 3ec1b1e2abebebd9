// K1X (FP64 mode, float32 observations, n <= 512 per CTA): 16 warps, double-buffered tiles,
// resident factor block.
//
// Same arithmetic as the other K1 kernels (reference pkg/src/momentcp/implicit.py:94-107 and the
// w of :124-140): per tile of 32 observations and a 16-column factor block
//   Z = V_tile A  (GEMM1, DMMA.8x8x4)  ->  P = nu Z^(d-1), w += P Z  ->  Y += V_tile^T P (GEMM2).
//
// Why this shape (tools/probe_dmma_lds.cu, K1W ncu source profiles): the
// DMMA inner loops themselves run at 93-98% of the FP64 pipe with operands from shared memory,
// but with 2 warps per SM sub-partition every cross-warp dependency (factor ring, P, chunk
// refills) leaves one warp issuing alone while its partner waits, and a lone warp cannot keep
// the pipe full.  K1X therefore runs 4 warps per sub-partition (16 warps, registers are no
// longer the limit: Y is 32 x 16 per warp) and removes the waits that are not data
// dependencies:
//
//  * the factor block (n x 16, fragment order, 64 KB) is loaded ONCE per column block with one
//    bulk copy and stays resident -- no factor ring;
//  * V is double-buffered: one 3-D TMA per 64 KB tile lands the 16 chunks (32 rows x 32 floats,
//    128-byte swizzle) of tile u + 2 while tile u + 1 is computed; the last warp to finish
//    tile u's GEMM2 issues it (counter, nobody waits);
//  * GEMM1 is split over 4 K-quarters (warp = row block x quarter, 1 x 2 DMMA tiles, the 4
//    warps of a row block on 4 different sub-partitions); the partial Z are merged through
//    shared memory in quarter order (one 128-thread named barrier per row block) and each of
//    the 4 warps forms P for a quarter of the row block's elements, published on the row
//    block's mbarrier;
//  * GEMM2: warp w owns variables 32w .. 32w+31 (4 x 2 DMMA tiles, Y in registers), starts with
//    its own row block and waits only for row blocks it has not seen;
//  * CL = 2 (n <= 1024, c5): a cluster of two CTAs splits the variables in halves; after the
//    K-quarter merge each lane stores its element's half-Z into the PEER's shared memory
//    (st.shared::cluster) and arrives on the peer's row-block mbarrier (release.cluster); both
//    CTAs add the halves in cluster-rank order (bitwise the same Z and P on both) and run GEMM2
//    on their own half of the tile.  No cluster-wide barrier per tile.
// Fixed-order merges and per-element ownership keep results deterministic and exactly linear
// in nu.
#pragma once

#include <cuda.h>

#include "k1s_fp64.cuh"   // mbarrier helpers
#include "k1x_common.cuh" // work split, cluster/proxy helpers, ordered shared loads
#include "mcp_common.cuh"
#include "pdl.h"
#include "umma.cuh"       // TMA helpers

namespace mcp {

#include "k1_dispatch.h"

constexpr int K1X_T = K1X_BOX_ROWS;   // observations per tile
constexpr int K1X_RB = 16;            // factor columns per block
constexpr int K1X_C = K1X_BOX_CHUNKS; // 32-variable chunks per tile (n <= 512)
constexpr int K1X_THREADS = 512;      // 16 warps
constexpr int K1X_SP = 18;            // P row pitch (doubles), == 2 mod 16
constexpr int K1X_TILE_BYTES = K1X_T * 32 * 4 * K1X_C;          // 64 KB of V
constexpr int K1X_A_BYTES = K1X_C * 8 * (K1X_RB / 8) * 32 * 8;  // 64 KB of factor fragments

template <int CL>
__host__ __device__ constexpr size_t k1x_smem_bytes() {
  // (the w flush scratch aliases the Z merge slots; CL = 2 adds the peer's half-Z slots)
  return 1024 /*alignment*/ + 2 * (size_t)K1X_TILE_BYTES + K1X_A_BYTES +
         2 * (size_t)K1X_T * K1X_SP * 8 /*P*/ + (size_t)4 * 4 * 8 * K1X_RB * 8 /*Z merge*/ +
         (CL > 1 ? (size_t)2 * 4 * 128 * 8 : 0) /*peer half-Z*/ + 512 /*barriers*/;
}

__device__ __forceinline__ uint32_t k1x_peer_addr(const void* local, uint32_t peer) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n"
               : "=r"(remote)
               : "r"(smem_u32(local)), "r"(peer));
  return remote;
}
__device__ __forceinline__ void k1x_st_peer(uint32_t remote, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;\n" ::"r"(remote), "d"(v) : "memory");
}
__device__ __forceinline__ void k1x_arrive_peer(uint32_t remote_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(remote_bar)
               : "memory");
}
// parity wait with cluster-scope acquire (the arrivals come from the peer CTA)
__device__ __forceinline__ void k1x_wait_cluster(uint64_t* bar, uint32_t parity) {
  auto try_once = [&]() {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
  };
  if (try_once()) return;
  const long long t0 = clock64();
  while (!try_once()) {
    if (clock64() - t0 > (1ll << 35)) __trap();
  }
}

__device__ __forceinline__ void k1x_bar_rowblock(int rbk) {
  asm volatile("bar.sync %0, 128;\n" ::"r"(1 + rbk) : "memory");
}
__device__ __forceinline__ void k1x_bar_all() {
  asm volatile("bar.sync 5, %0;\n" ::"n"(K1X_THREADS) : "memory");
}

// tmV: 3-D map over the fp32 observations viewed as (32 floats, rows, ldv / 32 chunks), box
// (32, 32, 16), 128-byte swizzle.  Uses K1WParams (n_pad = 512 CL, RB = 16).
template <int CL>
__global__ void __launch_bounds__(K1X_THREADS, 1)
    k1x_fg_dmma(const __grid_constant__ CUtensorMap tmV, K1WParams prm) {
  constexpr int NT = K1X_RB / 8;   // 2 column tiles
  constexpr int SP = K1X_SP;
  extern __shared__ __align__(16) unsigned char k1x_smem_raw[];
  unsigned char* base =
      k1x_smem_raw + ((1024u - (smem_u32(k1x_smem_raw) & 1023u)) & 1023u);
  float* sV = reinterpret_cast<float*>(base);                                   // [2][16][32][32]
  double* sA = reinterpret_cast<double*>(base + 2 * (size_t)K1X_TILE_BYTES);    // [128 ks][NT][32]
  double* sP = sA + K1X_A_BYTES / 8;                                            // [2][32][SP]
  double* sZm = sP + 2 * K1X_T * SP;                                            // [4][4][8][16]
  double* sW = sZm;                                                             // [512] flush
  double* sXz = sZm + 4 * 4 * 8 * K1X_RB;                                       // [2][4][128]
  uint64_t* fullV = reinterpret_cast<uint64_t*>(sXz + (CL > 1 ? 2 * 4 * 128 : 0));  // [2]
  uint64_t* fullA = fullV + 2;                                                  // [1]
  uint64_t* fullP = fullA + 1;                                                  // [2][4]
  uint64_t* fullX = fullP + 8;                                                  // [2][4] peer half-Z
  unsigned* cntV = reinterpret_cast<unsigned*>(fullX + 8);                      // [2]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int rbk = warp >> 2;       // GEMM1 row block (tile rows 8 rbk .. +7)
  const int kq = warp & 3;         // GEMM1 K-quarter (chunks 4 kq .. 4 kq + 3)
  const uint32_t crank = CL > 1 ? k1w_cluster_rank() : 0;
  const int cid = blockIdx.x / CL;   // cluster index (the unit of the work split)
  const int c0 = (int)crank * K1X_C; // this CTA's first 32-variable chunk
  const int dm1 = prm.d - 1;

  if (threadIdx.x == 0) {
    mbar_init(&fullV[0], 1);
    mbar_init(&fullV[1], 1);
    mbar_init(fullA, 1);
    for (int i = 0; i < 8; ++i) mbar_init(&fullP[i], 4);   // the row block's 4 warps
    for (int i = 0; i < 8; ++i) mbar_init(&fullX[i], 4);   // the peer row block's 4 warps
    cntV[0] = cntV[1] = 0;
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    tma_prefetch_desc(&tmV);
  }
  __syncthreads();
  if constexpr (CL > 1) k1w_cluster_sync();   // both CTAs' barriers exist before any remote arrive

  K1WTile cur;
  const bool any = k1w_tile_at(prm, cid, 0, cur);
  if (any && threadIdx.x == 0) {
    // V never changes: the first two tiles load before the factor prep kernel is waited for
    for (int b = 0; b < 2; ++b) {
      K1WTile tb;
      if (!k1w_tile_at(prm, cid, b, tb)) break;
      mbar_arrive_expect_tx(&fullV[b], K1X_TILE_BYTES);
      tma_load_3d(sV + (size_t)b * (K1X_TILE_BYTES / 4), &tmV, 0, (int)(tb.tile * K1X_T), c0,
                  smem_u32(&fullV[b]));
    }
  }
  pdl_enter();   // Afrag comes from the preceding prep kernel
  auto load_a = [&](int rb) {
    mbar_arrive_expect_tx(fullA, K1X_A_BYTES);
    tma_bulk_g2s(sA, prm.Afrag + (size_t)rb * CL * (K1X_A_BYTES / 8) + (size_t)crank * (K1X_A_BYTES / 8),
                 K1X_A_BYTES, fullA);
  };
  if (any && threadIdx.x == 0) load_a(cur.rb);
  uint32_t aphase = 0;
  int a_rb = any ? cur.rb : -1;

  // per-lane shared-memory offsets (bytes)
  // GEMM1: row 8 rbk + g of a chunk, k = 4 ks + t -> 16-byte unit ks ^ g
  uint32_t v1off[8];
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) v1off[ks] = 4u * ((8 * rbk + g) * 32 + ((ks ^ g) << 2) + t);
  // GEMM2: column 8 mt + g at row 2t + p (+ 8 blk) of the warp's own chunk
  uint32_t v2off[2][4];
#pragma unroll
  for (int p = 0; p < 2; ++p)
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
      v2off[p][mt] = 4u * ((2 * t + p) * 32 + (((2 * mt + (g >> 2)) ^ (2 * t + p)) << 2) + (g & 3));
  const uint32_t sV_u = smem_u32(sV), sA_u = smem_u32(sA) + 8u * lane;

  double y[4][NT][2];
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) y[mt][nt][0] = y[mt][nt][1] = 0.0;
  double wacc = 0.0;   // this lane's epilogue element column: (kq * 32 + lane) % 16
  const int e_row = (kq * 32 + lane) >> 4, e_col = (kq * 32 + lane) & 15;

  int64_t it = 0;
  while (any) {
    const int buf = (int)(it & 1);
    const uint32_t vpar = (uint32_t)((it >> 1) & 1);
    const uint32_t ppar = vpar;   // P row-block barriers are double-buffered like V
    const int64_t row0 = cur.tile * K1X_T;
    K1WTile nxt;
    const bool has_next = k1w_tile_at(prm, cid, it + 1, nxt);
    if (cur.rb != a_rb) {
      // a new column block (block-major split only): every warp is past its GEMM1 of the
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

    // ---------------- GEMM1: partial Z[8 rows x 16] over this warp's K-quarter ----------------
    double z[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) z[nt][0] = z[nt][1] = 0.0;
    {
      float fa_n;
      double b_n[NT];
      auto load = [&](int cc, int ks) {   // cc: chunk within the quarter
        const int c = 4 * kq + cc;
        fa_n = k1w_lds_f32(vt + (uint32_t)c * 4096u + v1off[ks]);
        const uint32_t ab = sA_u + 8u * (uint32_t)(((c * 8 + ks) * NT) * 32);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) b_n[nt] = k1w_lds_f64(ab + 256u * nt);
      };
      load(0, 0);
#pragma unroll
      for (int cc = 0; cc < 4; ++cc)
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          const double a = (double)fa_n;
          double b[NT];
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) b[nt] = b_n[nt];
          if (ks < 7) load(cc, ks + 1);
          else if (cc < 3) load(cc + 1, 0);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) dmma884(z[nt], a, b[nt]);
        }
    }

    // ---------------- merge the 4 K-quarters, epilogue on one element per lane ----------------
    {
      double* zm = sZm + (size_t)(rbk * 4 + kq) * 8 * K1X_RB;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
        *reinterpret_cast<double2*>(&zm[g * K1X_RB + 8 * nt + 2 * t]) =
            make_double2(z[nt][0], z[nt][1]);
      k1x_bar_rowblock(rbk);
      const double* zr = sZm + (size_t)rbk * 4 * 8 * K1X_RB + e_row * K1X_RB + e_col;
      double zz = zr[0];
#pragma unroll
      for (int q = 1; q < 4; ++q) zz += zr[q * 8 * K1X_RB];
      if constexpr (CL > 1) {
        // half-Z of this element to the peer CTA, then the peer's half from our own slots;
        // rank 0's half first on both sides
        double* slot = sXz + (size_t)(buf * 4 + rbk) * 128 + kq * 32 + lane;
        const uint32_t peer = crank ^ 1u;
        k1x_st_peer(k1x_peer_addr(slot, peer), zz);
        __syncwarp();
        if (lane == 0) k1x_arrive_peer(k1x_peer_addr(&fullX[buf * 4 + rbk], peer));
        k1x_wait_cluster(&fullX[buf * 4 + rbk], vpar);
        const double o = *slot;
        zz = crank == 0 ? zz + o : o + zz;
      }
      const int lr = 8 * rbk + e_row;
      const double nul = prm.nu ? prm.nu[row0 + lr] : prm.nu_const;
      const double pv = nul * rm_pow(zz, dm1);
      wacc += pv * zz;
      sP[(size_t)buf * K1X_T * SP + lr * SP + e_col] = pv;
      // (the merge slots are rewritten next tile only after GEMM2, which waits for this row
      // block's P barrier -- i.e. for all 4 warps to have read their partials)
      __syncwarp();
      if (lane == 0) mbar_arrive(&fullP[buf * 4 + rbk]);
    }

    // ---------------- GEMM2: Y[32 variables x 16] += V^T P over the 32 tile rows ----------------
    {
      const uint32_t vc = vt + (uint32_t)warp * 4096u;
      const uint32_t pbase = smem_u32(sP + (size_t)buf * K1X_T * SP + 2 * t * SP + g);
      float fa_n[4];
      double b_n[NT];
      auto load = [&](int blk, int p) {
        const uint32_t vb = vc + 1024u * (uint32_t)blk;
        const uint32_t pk = pbase + 8u * (uint32_t)(blk * 8 * SP + p * SP);
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) fa_n[mt] = k1w_lds_f32(vb + v2off[p][mt]);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) b_n[nt] = k1w_lds_f64(pk + 64u * nt);
      };
      mbar_wait(&fullP[buf * 4 + rbk], ppar);
      load(rbk, 0);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int blk = (rbk + i) & 3;
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          double a[4], b[NT];
#pragma unroll
          for (int mt = 0; mt < 4; ++mt) a[mt] = (double)fa_n[mt];
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) b[nt] = b_n[nt];
          if (p == 0) load(blk, 1);
#pragma unroll
          for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) dmma884(y[mt][nt], a[mt], b[nt]);
          if (p == 1 && i < 3) {
            const int nb = (rbk + i + 1) & 3;
            mbar_wait(&fullP[buf * 4 + nb], ppar);
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
          tma_load_3d(sV + (size_t)buf * (K1X_TILE_BYTES / 4), &tmV, 0, (int)(t2.tile * K1X_T),
                      c0, smem_u32(&fullV[buf]));
        }
      }
    }

    // ---------------- end of a segment: flush this CTA's partial ----------------
    if (cur.last_in_seg || !has_next) {
      double* Yp = prm.Ypart + ((size_t)cur.rb * prm.slots + cur.slot) * prm.n_pad * K1X_RB +
                   (size_t)crank * 512 * K1X_RB;
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          *reinterpret_cast<double2*>(
              &Yp[(size_t)(32 * warp + 8 * mt + g) * K1X_RB + 8 * nt + 2 * t]) =
              make_double2(y[mt][nt][0], y[mt][nt][1]);
          y[mt][nt][0] = y[mt][nt][1] = 0.0;
        }
      // (sW aliases the Z merge slots: every warp is past this tile's merge reads)
      k1x_bar_all();
      sW[threadIdx.x] = wacc;
      wacc = 0.0;
      k1x_bar_all();
      if (crank == 0 && threadIdx.x < K1X_RB) {
        // column j's partial sums sit at thread ids with (kq * 32 + lane) % 16 == j, i.e. at
        // every 16th thread: 32 of them, added in thread order
        double s = 0.0;
        for (int q = 0; q < K1X_THREADS / 16; ++q) s += sW[q * 16 + threadIdx.x];
        prm.wpart[((size_t)cur.rb * prm.slots + cur.slot) * K1X_RB + threadIdx.x] = s;
      }
      k1x_bar_all();
    }
    if (!has_next) break;
    cur = nxt;
    ++it;
  }

  k1w_zero_holes<K1X_THREADS, K1X_RB>(prm, cid, (int)crank * 512, 512, crank == 0);
  if constexpr (CL > 1) k1w_cluster_sync();   // the peer may still write into our half-Z slots
}

}  // namespace mcp
