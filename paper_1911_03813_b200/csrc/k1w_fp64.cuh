// K1W (FP64 mode, float32 observations, large n): TMA-staged, barrier-light fused f+grad.
//
// Same arithmetic as the other K1 kernels -- per tile of 64 observations and one 32-column
// block of factors it replaces
//   Z = V^T A                  pkg/src/momentcp/implicit.py:106     (GEMM1, DMMA.8x8x4)
//   P = nu * Z^(d-1)           pkg/src/momentcp/implicit.py:82-91,107 (epilogue, registers)
//   w += sum_l nu_l z_l^d      (= a_j^T y_j, implicit.py:139)
//   Y += V P                   pkg/src/momentcp/implicit.py:107     (GEMM2, DMMA.8x8x4)
// -- organised for the shapes where the FP64 pipe is the bound (c3: n = 512, r = 64; c5 through
// a 2-CTA cluster: n = 1024, r = 256):
//
//  * the whole 64-row tile stays resident in shared memory as n/32 chunk slots of 64 x 32
//    floats, each filled by ONE 2-D TMA (128-byte swizzle) and completing on its own mbarrier;
//    GEMM2 reads the tile GEMM1 read (no reload), and each slot is refilled with the next tile's
//    chunk by the one warp that owns the chunk in GEMM2, right after its GEMM2 pass over it --
//    the other warps' GEMM1 reads of the tile are complete by then (they passed the P barrier);
//  * GEMM1 visits the chunks in release order (every warp's first GEMM2 chunk, then its second),
//    so the next tile's first chunks land while GEMM2 still runs;
//  * the factor block (GEMM1's B operand, fragment order, 8 KB per chunk) streams through a
//    small ring of 1-D TMA copies; the last of the 8 warps to release a slot refills it;
//  * no CTA-wide barrier per tile: warp w computes Z and P for tile rows 8w .. 8w+7 and
//    publishes them on its own mbarrier; in GEMM2 every warp starts with its own rows and
//    rotates through the others, waiting only for the row blocks it has not seen yet -- so the
//    two warps sharing an SM sub-partition never idle at a barrier while the other finishes;
//  * swizzled layouts make every fragment load conflict-free: GEMM1 reads row 8w + g at
//    k = 4 ks + t (16-byte unit ks ^ g); GEMM2 reads column 8 mt + g at tile rows whose residue
//    mod 8 is 2t + (ks & 1) -- DMMA's k index may be any permutation of the 64 tile rows as long
//    as P uses the same one, and this one spreads the swizzled units over all 32 banks; all
//    per-lane offsets are computed once, so the inner loops are loads and DMMAs;
//  * CL = 2: a cluster of two CTAs splits n; each computes its half of Z, the halves are
//    exchanged through distributed shared memory and added in cluster-rank order (bitwise the
//    same Z on both), and each CTA runs GEMM2 on its own half of the tile -- so the Y block stays
//    in registers at n = 1024 with 32 factor columns.
//
// Work split: units = (column block, tile); when the clusters divide evenly among the column
// blocks each cluster keeps one block and strides over tiles (CTAs of different blocks read the
// same tile at about the same time, so it comes from L2); otherwise each cluster takes an equal
// contiguous range of the block-major unit list (at most a few block switches, each flushing the
// Y partial).  Partials go to [rb][slot][n_pad][RB] and are reduced in a fixed order by K3, so
// results are deterministic and exactly linear in nu.
#pragma once

#include <cuda.h>

#include "k1s_fp64.cuh"   // mbarrier helpers
#include "mcp_common.cuh"
#include "pdl.h"
#include "umma.cuh"       // TMA helpers

namespace mcp {

constexpr int K1W_T = 64;          // observations per tile
constexpr int K1W_NK = 32;         // floats per chunk row (one 128-byte swizzle row)
constexpr int K1W_RB_MAX = 32;     // factor columns per block: 16 or 32 (template RB)
constexpr int K1W_THREADS = 256;   // 8 warps
// P row pitch (doubles) RB + 2 == 2 mod 16 -> conflict-free GEMM2 B-fragment loads
__host__ __device__ constexpr int k1w_sp(int rb) { return rb + 2; }
constexpr int K1W_CHUNK_BYTES = K1W_T * K1W_NK * 4;         // 8 KB of V
// factor fragments of one 32-variable chunk: 8 k-steps x RB/8 column tiles x 32 lanes
__host__ __device__ constexpr int k1w_achunk_bytes(int rb) { return 8 * (rb / 8) * 32 * 8; }

struct K1WParams {
  int64_t num_tiles;      // tiles of 64 rows in p_pad
  int n;                  // variables (whole set)
  int n_pad;              // 256 * CPW * CL (Ypart row extent)
  const double* nu;       // p_pad weights or nullptr
  double nu_const;
  const double* Afrag;    // [rbs][n_pad / 4][RB / 8][32]
  int d;
  int rbs;
  int nclusters;          // gridDim.x / CL (<= rbs * num_tiles: no cluster without work)
  int groups;             // G = nclusters / rbs clusters per column block stride the main tiles
  int64_t t_main;         // main region: tiles [0, t_main) of every block (see k1w_tile_at)
  int slots;              // partial slots per column block
  double* Ypart;          // [rbs][slots][n_pad][RB]
  double* wpart;          // [rbs][slots][RB]
};

// factor ring depth: 48 KB (CL = 1) or 24 KB (CL = 2, which also stages the Z exchange)
template <int CPW, int CL, int RB>
__host__ __device__ constexpr int k1w_sa() {
  return (CL == 1 ? 48 * 1024 : 24 * 1024) / k1w_achunk_bytes(RB);
}

template <int CPW, int CL, int RB>
__host__ __device__ constexpr size_t k1w_smem_bytes() {
  return 1024 /*alignment slack*/ + (size_t)8 * CPW * K1W_CHUNK_BYTES +
         (size_t)k1w_sa<CPW, CL, RB>() * k1w_achunk_bytes(RB) +
         2 * (size_t)K1W_T * k1w_sp(RB) * 8 +
         (CL > 1 ? 2 * (size_t)K1W_THREADS * (RB / 4) * 8 : 0) + 8 * (size_t)RB * 8 /*w*/ +
         1024 /*barriers, counters*/;
}

// ---- work split (shared by the host plan and the kernel) --------------------------------
// block-major ranges: cluster c owns units [c U / Nc, (c + 1) U / Nc) of U = rbs * T
__host__ __device__ inline int64_t k1w_u0(int64_t c, int64_t U, int64_t Nc) { return c * U / Nc; }
// first cluster whose range touches column block rb
__host__ __device__ inline int64_t k1w_cfirst(int64_t rb, int64_t T, int64_t U, int64_t Nc) {
  int64_t c = rb * T * Nc / U;
  while (c > 0 && k1w_u0(c, U, Nc) > rb * T) --c;
  while (c + 1 < Nc && k1w_u0(c + 1, U, Nc) <= rb * T) ++c;
  return c;
}
__host__ __device__ inline int64_t k1w_clast(int64_t rb, int64_t T, int64_t U, int64_t Nc) {
  int64_t c = k1w_cfirst(rb, T, U, Nc);
  while (c + 1 < Nc && k1w_u0(c + 1, U, Nc) < (rb + 1) * T) ++c;
  return c;
}

struct K1WTile {
  int rb, slot;
  int64_t tile;
  bool last_in_seg;   // flush the partial after this tile
};

// Work split over (column block, tile) units, shared by the host plan and the kernels:
//  * main region, tiles [0, t_main): the first G * rbs clusters form G groups of one cluster per
//    column block; member j of a group strides over tiles j, j + G, ... -- the rbs clusters that
//    read a tile do so at about the same time, so V comes from HBM once and from L2 rbs - 1
//    times (slot j of the block);
//  * leftover region, tiles [t_main, T): the L = Nc - G rbs remaining clusters take equal
//    contiguous ranges of the block-major unit list (slots G, G + 1, ... of each block they
//    touch); t_main = floor(G rbs T / Nc) equalises the work of both kinds of cluster.
// With Nc <= rbs * T every cluster has work and every slot 0 .. G - 1 + (clusters touching a
// block in the leftover region) is written exactly once; the remaining slots up to `slots` are
// zero-filled.
__host__ __device__ inline void k1w_split(int64_t T, int rbs, int64_t Nc, int& G, int64_t& t_main) {
  G = (int)(Nc / rbs);
  t_main = (Nc % rbs == 0) ? T : (int64_t)G * rbs * T / Nc;
}
__host__ __device__ inline int k1w_used_slots(int rb, int64_t T, int rbs, int64_t Nc, int G,
                                              int64_t t_main) {
  const int64_t L = Nc - (int64_t)G * rbs, T2 = T - t_main, U2 = (int64_t)rbs * T2;
  if (L == 0 || T2 == 0) return G;
  return G + (int)(k1w_clast(rb, T2, U2, L) - k1w_cfirst(rb, T2, U2, L) + 1);
}

// Tile `k` (0-based) of cluster c's work list; returns false past the end.
__device__ __forceinline__ bool k1w_tile_at(const K1WParams& prm, int c, int64_t k, K1WTile& o) {
  const int64_t T = prm.num_tiles;
  const int G = prm.groups;
  if (c < G * prm.rbs) {
    const int slot = c / prm.rbs;
    const int64_t tile = slot + k * G;
    if (tile >= prm.t_main) return false;
    o.rb = c % prm.rbs;
    o.slot = slot;
    o.tile = tile;
    o.last_in_seg = tile + G >= prm.t_main;
    return true;
  }
  const int64_t L = prm.nclusters - (int64_t)G * prm.rbs, T2 = T - prm.t_main;
  const int64_t U2 = (int64_t)prm.rbs * T2, lc = c - (int64_t)G * prm.rbs;
  const int64_t u = k1w_u0(lc, U2, L) + k;
  if (u >= k1w_u0(lc + 1, U2, L)) return false;
  o.rb = (int)(u / T2);
  o.tile = prm.t_main + u % T2;
  o.slot = G + (int)(lc - k1w_cfirst(o.rb, T2, U2, L));
  o.last_in_seg = (u + 1 == k1w_u0(lc + 1, U2, L)) || ((u + 1) % T2 == 0);
  return true;
}

// Zero the partial slots no cluster writes (blocks touched by fewer leftover clusters).
template <int THREADS, int RB>
__device__ __forceinline__ void k1w_zero_holes(const K1WParams& prm, int cid, int var0, int nvars,
                                               bool write_w) {
  for (int rb = 0; rb < prm.rbs; ++rb) {
    const int used = k1w_used_slots(rb, prm.num_tiles, prm.rbs, prm.nclusters, prm.groups,
                                    prm.t_main);
    for (int s = used; s < prm.slots; ++s) {
      if ((rb * prm.slots + s) % prm.nclusters != cid) continue;
      double* Yp = prm.Ypart + ((size_t)rb * prm.slots + s) * prm.n_pad * RB + (size_t)var0 * RB;
      for (int e = threadIdx.x; e < nvars * RB; e += THREADS) Yp[e] = 0.0;
      if (write_w && threadIdx.x < RB) prm.wpart[((size_t)rb * prm.slots + s) * RB + threadIdx.x] = 0.0;
    }
  }
}

__device__ __forceinline__ uint32_t k1w_cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void k1w_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ double k1w_ld_peer(const double* local, uint32_t peer) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n"
               : "=r"(remote)
               : "r"(smem_u32(local)), "r"(peer));
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];\n" : "=d"(v) : "r"(remote) : "memory");
  return v;
}
// Shared-memory operand loads as volatile asm: they stay ahead of the (volatile) DMMAs they are
// written before, so the next step's operands are in flight while the pipe works on this step's
// products (an in-order warp stuck behind a throttled DMMA cannot issue later loads).
__device__ __forceinline__ float k1w_lds_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];\n" : "=f"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ double k1w_lds_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void k1w_named_sync() {
  asm volatile("bar.sync 1, %0;\n" ::"n"(K1W_THREADS) : "memory");
}
__device__ __forceinline__ void k1w_fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

template <int CPW, int CL, int RB>
__global__ void __launch_bounds__(K1W_THREADS, 1)
    k1w_fg_dmma(const __grid_constant__ CUtensorMap tmV, K1WParams prm) {
  constexpr int C = 8 * CPW;           // chunk slots of this CTA's tile (n_local = 32 C)
  constexpr int SA = k1w_sa<CPW, CL, RB>();
  constexpr int NT = RB / 8;           // column tiles
  constexpr int SP = k1w_sp(RB);
  constexpr int ACH = k1w_achunk_bytes(RB);
  extern __shared__ __align__(16) unsigned char k1w_smem_raw[];
  unsigned char* base =
      k1w_smem_raw + ((1024u - (smem_u32(k1w_smem_raw) & 1023u)) & 1023u);
  float* sV = reinterpret_cast<float*>(base);                                  // [C][64][32]
  double* sA = reinterpret_cast<double*>(base + (size_t)C * K1W_CHUNK_BYTES);  // [SA][8][NT][32]
  double* sP = sA + (size_t)SA * (ACH / 8);                       // [2][64][SP]
  double* sZx = sP + 2 * K1W_T * SP;                                           // [2][2NT][256]
  double* sW = sZx + (CL > 1 ? 2 * K1W_THREADS * 2 * NT : 0);                 // [8][RB]
  uint64_t* fullV = reinterpret_cast<uint64_t*>(sW + 8 * RB);              // [C]
  uint64_t* fullA = fullV + C;                                                 // [SA]
  uint64_t* fullP = fullA + SA;                                                // [8] row blocks
  unsigned* cntA = reinterpret_cast<unsigned*>(fullP + 8);                     // [SA]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const uint32_t crank = CL > 1 ? k1w_cluster_rank() : 0;
  const int cid = blockIdx.x / CL;            // cluster index (the unit of the work split)
  const int n0 = (int)crank * 32 * C;         // this CTA's first variable
  const int dm1 = prm.d - 1;

  if (threadIdx.x == 0) {
    for (int i = 0; i < C; ++i) mbar_init(&fullV[i], 1);
    for (int i = 0; i < SA; ++i) {
      mbar_init(&fullA[i], 1);
      cntA[i] = 0;
    }
    for (int i = 0; i < 8; ++i) mbar_init(&fullP[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    tma_prefetch_desc(&tmV);
  }
  __syncthreads();

  K1WTile cur;
  const bool any = k1w_tile_at(prm, cid, 0, cur);
  // V never changes: the first tile's chunks load before waiting for the factor prep kernel
  if (any && threadIdx.x == 0) {
    for (int c = 0; c < C; ++c) {
      mbar_arrive_expect_tx(&fullV[c], K1W_CHUNK_BYTES);
      tma_load_2d(sV + (size_t)c * (K1W_CHUNK_BYTES / 4), &tmV, n0 + 32 * c,
                  (int)(cur.tile * K1W_T), smem_u32(&fullV[c]));
    }
  }
  pdl_enter();   // Afrag comes from the preceding prep kernel

  // factor chunk q of this CTA's GEMM1 sequence: tile q / C, chunk position q % C
  auto a_src = [&](int64_t q, const K1WTile& tq) -> const double* {
    const int j = (int)(q % C);
    const int c = CPW * (j & 7) + (j >> 3);                        // release order
    const int kchunk = (n0 >> 5) + c;                              // 32-variable chunk index
    return prm.Afrag + ((size_t)tq.rb * (prm.n_pad / 4) + (size_t)kchunk * 8) * NT * 32;
  };
  if (any && threadIdx.x == 0) {
    for (int q = 0; q < SA; ++q) {
      K1WTile tq;
      if (!k1w_tile_at(prm, cid, q / C, tq)) break;
      mbar_arrive_expect_tx(&fullA[q], ACH);
      tma_bulk_g2s(sA + (size_t)q * (ACH / 8), a_src(q, tq), ACH,
                   &fullA[q]);
    }
  }

  // per-lane shared-memory offsets, fixed for the whole kernel
  // GEMM1: row 8 warp + g of a chunk, k = 4 ks + t, 16-byte unit ks ^ g (floats)
  int v1off[8];
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) v1off[ks] = (8 * warp + g) * 32 + ((ks ^ g) << 2) + t;
  // GEMM2: column 8 mt + g of a chunk at row 2t + p (+ 8 * row block), p = ks & 1
  int v2off[2][4];
#pragma unroll
  for (int p = 0; p < 2; ++p)
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
      v2off[p][mt] = (2 * t + p) * 32 + (((2 * mt + (g >> 2)) ^ (2 * t + p)) << 2) + (g & 3);
  const int p2off = 2 * t * SP + g;   // P[row 2t (+p) (+ 8 block)][8 nt + g]

  double y[CPW][4][NT][2];
#pragma unroll
  for (int h = 0; h < CPW; ++h)
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) y[h][mt][nt][0] = y[h][mt][nt][1] = 0.0;
  double wacc[NT][2];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) wacc[nt][0] = wacc[nt][1] = 0.0;

  int aslot = 0;            // factor ring position of the next chunk
  uint32_t aphase = 0;
  int64_t it = 0;
  while (any) {
    const uint32_t par = (uint32_t)(it & 1);
    const int pb = (int)(it & 1);
    const int64_t row0 = cur.tile * K1W_T;
    K1WTile nxt;
    const bool has_next = k1w_tile_at(prm, cid, it + 1, nxt);

    // ---------------- GEMM1: Z[8 rows x 32] (partial over this CTA's variables) ----------------
    // flat sequence of C chunks x 8 k-steps; step s + 1's operands are loaded before step s's
    // DMMAs issue (the next chunk's barriers are waited for after the last step's DMMAs)
    double z[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) z[nt][0] = z[nt][1] = 0.0;
    {
      uint32_t vsa, asa;   // shared addresses of the current chunk / factor slot
      auto bind = [&](int jj) {
        const int c = CPW * (jj & 7) + (jj >> 3);
        mbar_wait(&fullV[c], par);
        mbar_wait(&fullA[aslot], aphase);
        vsa = smem_u32(sV + (size_t)c * (K1W_CHUNK_BYTES / 4));
        asa = smem_u32(sA + (size_t)aslot * (ACH / 8) + lane);
      };
      float fa_n;
      double b_n[NT];
      auto load = [&](int ks) {
        fa_n = k1w_lds_f32(vsa + 4u * (uint32_t)v1off[ks]);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) b_n[nt] = k1w_lds_f64(asa + 8u * (uint32_t)((ks * NT + nt) * 32));
      };
      bind(0);
      load(0);
#pragma unroll 1
      for (int j = 0; j < C; ++j) {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          const double a = (double)fa_n;
          double b[NT];
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) b[nt] = b_n[nt];
          if (ks < 7) load(ks + 1);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) dmma884(z[nt], a, b[nt]);
        }
        // release the factor slot; the last of the 8 warps refills it (chunk q + SA)
        __syncwarp();
        if (lane == 0) {
          __threadfence_block();
          if (atomicAdd(&cntA[aslot], 1u) == K1W_THREADS / 32 - 1) {
            cntA[aslot] = 0;
            __threadfence_block();
            const int64_t qn = it * C + j + SA;
            K1WTile tq;
            if (k1w_tile_at(prm, cid, qn / C, tq)) {
              k1w_fence_proxy_async();
              mbar_arrive_expect_tx(&fullA[aslot], ACH);
              tma_bulk_g2s(sA + (size_t)aslot * (ACH / 8), a_src(qn, tq),
                           ACH, &fullA[aslot]);
            }
          }
        }
        if (++aslot == SA) {
          aslot = 0;
          aphase ^= 1u;
        }
        if (j + 1 < C) {
          bind(j + 1);
          load(0);
        }
      }
    }

    if constexpr (CL > 1) {
      // Z halves through distributed shared memory, summed in cluster-rank order on both CTAs
      double* mine = sZx + (size_t)pb * K1W_THREADS * 2 * NT + (size_t)threadIdx.x;
#pragma unroll
      for (int e = 0; e < 2 * NT; ++e) mine[e * K1W_THREADS] = (&z[0][0])[e];
      k1w_cluster_sync();
      const uint32_t peer = crank ^ 1u;
#pragma unroll
      for (int e = 0; e < 2 * NT; ++e) {
        const double o = k1w_ld_peer(mine + e * K1W_THREADS, peer);
        double& zz = (&z[0][0])[e];
        zz = crank == 0 ? zz + o : o + zz;
      }
    }

    // ---------------- epilogue: P = nu z^(d-1), w += P z  (rows 8 warp + g) ----------------
    {
      double* P = sP + (size_t)pb * K1W_T * SP;
      const int lr = 8 * warp + g;
      const double nul = prm.nu ? prm.nu[row0 + lr] : prm.nu_const;
      double zv[2 * NT], pv[2 * NT];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        zv[2 * nt] = z[nt][0];
        zv[2 * nt + 1] = z[nt][1];
      }
      rm_pow_vec<2 * NT>(zv, pv, dm1);
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const double p0 = nul * pv[2 * nt], p1 = nul * pv[2 * nt + 1];
        wacc[nt][0] += p0 * zv[2 * nt];
        wacc[nt][1] += p1 * zv[2 * nt + 1];
        *reinterpret_cast<double2*>(&P[lr * SP + 8 * nt + 2 * t]) = make_double2(p0, p1);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&fullP[warp]);   // this warp's 8 P rows (and its GEMM1) done
    }

    // ---------------- GEMM2: Y[own 32 CPW variables x 32] += V^T P ----------------
    // per half: 8 row blocks (own first, then the others in turn) x 2 k-steps; the next step's
    // operands are loaded before this step's 16 DMMAs issue
    {
      const uint32_t pbase = smem_u32(sP + (size_t)pb * K1W_T * SP + p2off);
#pragma unroll
      for (int h = 0; h < CPW; ++h) {
        const int c = CPW * warp + h;
        const uint32_t vsa = smem_u32(sV + (size_t)c * (K1W_CHUNK_BYTES / 4));
        float fa_n[4];
        double b_n[NT];
        auto load = [&](int blk, int p) {
          const uint32_t vb = vsa + 1024u * (uint32_t)blk;
          const uint32_t pk = pbase + 8u * (uint32_t)(blk * 8 * SP + p * SP);
#pragma unroll
          for (int mt = 0; mt < 4; ++mt) fa_n[mt] = k1w_lds_f32(vb + 4u * (uint32_t)v2off[p][mt]);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) b_n[nt] = k1w_lds_f64(pk + 64u * (uint32_t)nt);
        };
        if (h == 0) mbar_wait(&fullP[warp], par);
        load(warp, 0);
#pragma unroll 1
        for (int i = 0; i < 8; ++i) {
          const int blk = (warp + i) & 7;
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
              for (int nt = 0; nt < NT; ++nt) dmma884(y[h][mt][nt], a[mt], b[nt]);
            if (p == 1 && i < 7) {
              // next row block: its P may still be in flight (waited for after this step's
              // products are queued)
              const int nb = (warp + i + 1) & 7;
              if (h == 0) mbar_wait(&fullP[nb], par);
              load(nb, 0);
            }
          }
        }
        // chunk c is free: refill it with the next tile's chunk.  This warp is its only GEMM2
        // reader, and every warp's GEMM1 reads of it finished before that warp published its P
        // rows, all of which this warp has waited for.
        __syncwarp();
        if (lane == 0 && has_next) {
          k1w_fence_proxy_async();
          mbar_arrive_expect_tx(&fullV[c], K1W_CHUNK_BYTES);
          tma_load_2d(sV + (size_t)c * (K1W_CHUNK_BYTES / 4), &tmV, n0 + 32 * c,
                      (int)(nxt.tile * K1W_T), smem_u32(&fullV[c]));
        }
      }
    }

    // ---------------- end of a segment: flush this CTA's partial ----------------
    if (cur.last_in_seg || !has_next) {
      double* Yp = prm.Ypart + ((size_t)cur.rb * prm.slots + cur.slot) * prm.n_pad * RB;
#pragma unroll
      for (int h = 0; h < CPW; ++h) {
        const int i0 = n0 + 32 * (CPW * warp + h);
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            *reinterpret_cast<double2*>(&Yp[(size_t)(i0 + 8 * mt + g) * RB + 8 * nt + 2 * t]) =
                make_double2(y[h][mt][nt][0], y[h][mt][nt][1]);
            y[h][mt][nt][0] = y[h][mt][nt][1] = 0.0;
          }
      }
      // w: over the 8 row lanes, then the 8 warps (row blocks) in a fixed order (rank 0 writes)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          double v = wacc[nt][e];
          v += __shfl_xor_sync(0xffffffffu, v, 4);
          v += __shfl_xor_sync(0xffffffffu, v, 8);
          v += __shfl_xor_sync(0xffffffffu, v, 16);
          if (g == 0) sW[warp * RB + 8 * nt + 2 * t + e] = v;
          wacc[nt][e] = 0.0;
        }
      k1w_named_sync();
      if (crank == 0 && threadIdx.x < RB) {
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) s += sW[q * RB + threadIdx.x];
        prm.wpart[((size_t)cur.rb * prm.slots + cur.slot) * RB + threadIdx.x] = s;
      }
      k1w_named_sync();   // sW reusable
    }
    if (!has_next) break;
    cur = nxt;
    ++it;
  }

  k1w_zero_holes<K1W_THREADS, RB>(prm, cid, n0, 32 * C, crank == 0);
  if constexpr (CL > 1) k1w_cluster_sync();   // no CTA exits while its peer may read its Z
}

}  // namespace mcp
