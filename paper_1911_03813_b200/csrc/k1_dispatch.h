// Shape selection and launch of the K1 fused f+grad kernel variants (host side).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace mcp {


struct K1Variant {
  int dtype = 0;       // MCP_F64 / MCP_F32
  int RB = 8;          // factor columns per CTA
  int MTW = 1;         // compile-time bound on n chunks (register array extent)
  int n_chunks = 1;
  int n_pad = 64;
  int rbs = 1;         // column blocks
  int gp = 1;          // persistent CTAs per column block
  int grid = 1;
  size_t smem = 0;
  int64_t num_tiles = 0;
  size_t afrag_elems = 0, ypart_elems = 0, wpart_elems = 0;
  std::string name;
  int entry = -1;
  int kind = 0;        // 0: k1_fg_dmma (generic, cp.async chunks)  1: k1s_fg_stream (TMA slabs)
                       // 2: k1t_fg_tf32 (tcgen05 fast mode)  3: k1p_fg_pairs (self-fed pairs)
                       // 4: k1q_fg_pairs (warp-specialised pairs)  5: k1g_fg_dmma (Y in L2)
                       // 6: k1r_fg_triads (K1Q with the GEMM1 role split by columns)
                       // 8: k1x_fg_dmma (fp32 V, n <= 512: 16 warps, double-buffered tiles)
  int stages = 0;      // ring depth (kind 1)
  int MT = 0;          // GEMM2 m-tiles (kind 1)
  int MTW2 = 1;        // slabs per TMA copy unit (kind 1)
  int cl = 1;
  int cpw = 1;
  int t_rows = 0;      // kind 8: tile rows (the 3-D TMA box)
  int groups = 0;      // kind 8: work split (k1x_common.cuh k1w_split)
  int64_t t_main = 0;
  bool needs_prep() const { return kind == 0 || kind == 5 || kind == 8; }
  bool needs_tmap() const { return kind == 8; }
};

// Choose the variant for (dtype, n, r, p_pad) on a device with `sms` SMs.
bool k1_select(int dtype, int64_t n, int r, int64_t p_pad, int sms, K1Variant& v, std::string& why);

// Launch K1 on stream s; returns 0 on success.
// tmap: the K1X observation tensor map (CUtensorMap*, fp32 V, 3-D 32 x 32 x 16 boxes, swizzled)
// when v.needs_tmap(), else ignored.
int k1_launch(const K1Variant& v, const void* dV, int64_t ldv, int n, const double* dnu,
              double nu_const, const double* A, int r, const double* Afrag, int d, double* Ypart,
              double* wpart, cudaStream_t s, const void* tmap = nullptr);

// Raise a kernel's dynamic shared-memory limit (per device, once per new maximum).
bool ensure_dyn_smem(const void* fn, size_t smem);

// True when the evaluation can end with the one-kernel reduce + finish K3F (prep-free FP64 K1,
// r <= 32, every w in K3F's w block).
bool k1_fuses_tail(const K1Variant& v, int64_t n, int r);

// Row pitch (elements) the observation upload uses for dtype / n.
int64_t obs_pitch(int dtype, int64_t n);

}  // namespace mcp
