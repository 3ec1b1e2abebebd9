// Shared pieces of the TMA-staged fp32-observation FP64 kernels (K1X, k1x_fp64.cuh): launch
// parameters, the work split over (column block, tile) units, and small PTX helpers
// (cluster rank / barrier, async-proxy fence, ordered shared loads).
//
// History: this file held K1W, an 8-warp version of the resident-tile design (one 64-row tile
// per CTA, factor ring, cluster n-split).  Its DMMA inner loops ran at the probe rate, but with
// 2 warps per SM sub-partition every cross-warp dependency left one warp issuing alone; it
// reached 72% of the FP64 pipe at c3 (below the 73% of K1) and 26 TF at n = 256 (K1: 29.5), so
// K1X (16 warps, double-buffered tiles, resident factor block) replaced it (DESIGN.md
// section 4).
#pragma once

#include <cuda.h>

#include "k1s_fp64.cuh"   // mbarrier helpers
#include "mcp_common.cuh"
#include "pdl.h"
#include "umma.cuh"       // TMA helpers

namespace mcp {


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
__device__ __forceinline__ void k1w_fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

}  // namespace mcp
