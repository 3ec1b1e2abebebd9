// Instantiations of the K1 FP64 kernel family and the host-side variant selection.
#include <atomic>
#include <map>
#include <mutex>
#include <utility>
#include <cstdlib>

#include "momentcp_b200.h"
#include "tuning.h"
#include "k1_dispatch.h"
#include "k1_fp64.cuh"
#include "tail_pieces.cuh"
#include "k1s_fp64.cuh"
#include "k1p_fp64.cuh"
#include "k1q_fp64.cuh"
#include "k1x_common.cuh"
#include "k1x_fp64.cuh"
#if MCP_WITH_K1R
#include "k1r_fp64.cuh"
#endif

namespace mcp_internal {
// abi.cu: 2-D fp64 tensor map (inner x outer, row pitch in bytes)
bool make_tmap_f64(CUtensorMap* m, const void* gaddr, uint64_t inner, uint64_t outer,
                   uint64_t pitch, uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle sw);
}  // namespace mcp_internal

namespace mcp {

// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-device maximum: raise it once per
// (kernel, device) to the largest size requested so far instead of on every plan (a driver call
// on the host path of every evaluation).
bool ensure_dyn_smem(const void* fn, size_t smem) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    (void)cudaGetLastError();
    return false;
  }
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> have;
  std::lock_guard<std::mutex> lk(mu);
  int& h = have[{fn, dev}];
  if ((int)smem <= h) return true;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess) {
    (void)cudaGetLastError();
    return false;
  }
  h = (int)smem;
  return true;
}

namespace {

template <typename VT, int RB, int MTW>
void launch_t(const K1Params& prm, int grid, size_t smem, cudaStream_t s) {
  launch_pdl(k1_fg_dmma<VT, RB, MTW>, dim3(grid), dim3(K1_THREADS), smem, s, prm);
}

using LaunchFn = void (*)(const K1Params&, int, size_t, cudaStream_t);

struct Entry {
  int dtype, RB, MTW;
  LaunchFn launch;
  const void* fn;
  size_t smem;
};

#define MCP_K1_E(VT, DT, RB, MTW) \
  {DT, RB, MTW, &launch_t<VT, RB, MTW>, (const void*)&k1_fg_dmma<VT, RB, MTW>, k1_smem_bytes<VT, RB>()}
#define MCP_K1_ROW(VT, DT)                                                                   \
  MCP_K1_E(VT, DT, 8, 1), MCP_K1_E(VT, DT, 16, 1), MCP_K1_E(VT, DT, 32, 1),                   \
      MCP_K1_E(VT, DT, 64, 1), MCP_K1_E(VT, DT, 8, 2), MCP_K1_E(VT, DT, 16, 2),               \
      MCP_K1_E(VT, DT, 32, 2), MCP_K1_E(VT, DT, 64, 2), MCP_K1_E(VT, DT, 8, 4),               \
      MCP_K1_E(VT, DT, 16, 4), MCP_K1_E(VT, DT, 32, 4), MCP_K1_E(VT, DT, 64, 4),              \
      MCP_K1_E(VT, DT, 8, 8), MCP_K1_E(VT, DT, 16, 8), MCP_K1_E(VT, DT, 32, 8),               \
      MCP_K1_E(VT, DT, 8, 16), MCP_K1_E(VT, DT, 16, 16), MCP_K1_E(VT, DT, 8, 32)

const Entry kTable[] = {MCP_K1_ROW(double, MCP_F64), MCP_K1_ROW(float, MCP_F32)};

// K1G (Y partial in global memory): column blocks of RB in {16, 32, 64}
// (Entry::MTW: 0 = Y partial in L2 (8 warps), 1 = K1GT with 8 warps, 2 = K1GT with 16 warps)
// K1G's launch takes the partial's tensor map (K1GT's bulk reduce-adds) through a file-scope
// slot set by k1_launch right before the call (the table's launchers share one signature)
thread_local const CUtensorMap* g_k1g_tmap = nullptr;
template <typename VT, int RB, bool TM, int NW>
void launch_g(const K1Params& prm, int grid, size_t smem, cudaStream_t s) {
  launch_pdl(k1g_fg_dmma<VT, RB, TM, NW>, dim3(grid), dim3(NW * 32), smem, s, prm, *g_k1g_tmap);
}
#define MCP_K1G_E(VT, DT, RB, TM, NW)                                                        \
  {DT, RB, TM ? NW / 8 : 0, &launch_g<VT, RB, TM, NW>, (const void*)&k1g_fg_dmma<VT, RB, TM, NW>, \
   k1g_smem_bytes<VT, RB, TM>()}
const Entry kTableG[] = {
    MCP_K1G_E(double, MCP_F64, 16, false, 8), MCP_K1G_E(double, MCP_F64, 32, false, 8),
    MCP_K1G_E(double, MCP_F64, 64, false, 8), MCP_K1G_E(float, MCP_F32, 16, false, 8),
    MCP_K1G_E(float, MCP_F32, 32, false, 8),  MCP_K1G_E(float, MCP_F32, 64, false, 8),
    MCP_K1G_E(double, MCP_F64, 16, true, 8),  MCP_K1G_E(double, MCP_F64, 32, true, 8),
    MCP_K1G_E(float, MCP_F32, 16, true, 8),   MCP_K1G_E(float, MCP_F32, 32, true, 8),
    MCP_K1G_E(double, MCP_F64, 64, true, 8),  MCP_K1G_E(float, MCP_F32, 64, true, 8),
#if MCP_CFG_K1GT_NW == 16
    MCP_K1G_E(double, MCP_F64, 32, true, 16), MCP_K1G_E(float, MCP_F32, 32, true, 16),
#endif
};
constexpr int kEntriesG = sizeof(kTableG) / sizeof(kTableG[0]);
constexpr int kEntries = sizeof(kTable) / sizeof(kTable[0]);

int max_rb_for(int mtw) {
  switch (mtw) {
    case 1: case 2: case 4: return 64;
    case 8: return 32;
    case 16: return 16;
    default: return 8;
  }
}

// Resident CTAs per SM of K1 table entry e on the current device, cached per (entry, device);
// the dynamic shared-memory limit is raised per device through ensure_dyn_smem.
int occupancy(int e) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    (void)cudaGetLastError();
    return 0;
  }
  static std::mutex mu;
  static std::map<std::pair<int, int>, int> cache;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find({e, dev});
    if (it != cache.end()) return it->second;
  }
  const Entry& en = kTable[e];
  if (!ensure_dyn_smem(en.fn, en.smem)) return 0;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, en.fn, K1_THREADS, en.smem) !=
      cudaSuccess) {
    (void)cudaGetLastError();
    return 0;
  }
  std::lock_guard<std::mutex> lk(mu);
  cache[{e, dev}] = occ;
  return occ;
}

// ---------------- K1S (TMA-streamed slabs, fp64, n <= 128) ----------------
template <int NTM, int TAIL, int MTH, int KH>
void launch_s(const K1SParams& prm, int grid, size_t smem, cudaStream_t s) {
  k1s_fg_stream<NTM, TAIL, MTH, KH><<<grid, K1S_THREADS, smem, s>>>(prm);
}
using LaunchS = void (*)(const K1SParams&, int, size_t, cudaStream_t);
struct EntryS {
  int NTM, TAIL, MTH, KH;
  LaunchS launch;
  const void* fn;
};
#define MCP_K1S_E(NTM, TAIL, MTH, KH) \
  {NTM, TAIL, MTH, KH, &launch_s<NTM, TAIL, MTH, KH>, \
   (const void*)&k1s_fg_stream<NTM, TAIL, MTH, KH>}
#define MCP_K1S_COLS(MTH, KH) \
  MCP_K1S_E(1, 0, MTH, KH), MCP_K1S_E(1, 1, MTH, KH), MCP_K1S_E(1, 2, MTH, KH), \
      MCP_K1S_E(2, 0, MTH, KH)
// (MTH, KH) groups by n (KH = ldv / 4 with ldv == 4 mod 16): n <= 4, <= 20, <= 36, <= 68,
// <= 100, <= 116, <= 128
const EntryS kTableS[] = {MCP_K1S_COLS(1, 1),  MCP_K1S_COLS(2, 5),  MCP_K1S_COLS(3, 9),
                          MCP_K1S_COLS(5, 17), MCP_K1S_COLS(7, 25), MCP_K1S_COLS(8, 29),
                          MCP_K1S_COLS(8, 33)};
constexpr int kEntriesS = sizeof(kTableS) / sizeof(kTableS[0]);

// ---------------- K1P (self-fed pairs, fp64, n <= 128) ----------------
template <int NTM, int TAIL, int MTH, int KH>
void launch_p(const K1SParams& prm, int grid, size_t smem, cudaStream_t s) {
  k1p_fg_pairs<NTM, TAIL, MTH, KH><<<grid, K1P_THREADS, smem, s>>>(prm);
}
#define MCP_K1P_E(NTM, TAIL, MTH, KH) \
  {NTM, TAIL, MTH, KH, &launch_p<NTM, TAIL, MTH, KH>, \
   (const void*)&k1p_fg_pairs<NTM, TAIL, MTH, KH>}
#define MCP_K1P_COLS(MTH, KH) \
  MCP_K1P_E(1, 0, MTH, KH), MCP_K1P_E(1, 1, MTH, KH), MCP_K1P_E(1, 2, MTH, KH), \
      MCP_K1P_E(2, 0, MTH, KH)
const EntryS kTableP[] = {MCP_K1P_COLS(1, 1),  MCP_K1P_COLS(2, 5),  MCP_K1P_COLS(3, 9),
                          MCP_K1P_COLS(5, 17), MCP_K1P_COLS(7, 25), MCP_K1P_COLS(8, 29),
                          MCP_K1P_COLS(8, 33)};

// ---------------- K1Q (warp-specialised pairs, fp64, n <= 128) ----------------
template <int NTM, int TAIL, int MT2, int KH>
void launch_q(const K1SParams& prm, int grid, size_t smem, cudaStream_t s) {
  // programmatic dependent launch: the V-only prologue overlaps the previous kernel
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(K1Q_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k1q_fg_pairs<NTM, TAIL, MT2, KH>, prm);
}
#define MCP_K1Q_E(NTM, TAIL, MT2, KH) \
  {NTM, TAIL, MT2, KH, &launch_q<NTM, TAIL, MT2, KH>, \
   (const void*)&k1q_fg_pairs<NTM, TAIL, MT2, KH>}
#define MCP_K1Q_COLS(MT2, KH) \
  MCP_K1Q_E(1, 0, MT2, KH), MCP_K1Q_E(1, 1, MT2, KH), MCP_K1Q_E(1, 2, MT2, KH), \
      MCP_K1Q_E(2, 0, MT2, KH)
// (MT2, KH) groups by n: n <= 4, <= 20, <= 36, <= 68, <= 100, <= 116, <= 128 (MTH field = MT2)
const EntryS kTableQ[] = {MCP_K1Q_COLS(1, 1),  MCP_K1Q_COLS(3, 5),  MCP_K1Q_COLS(5, 9),
                          MCP_K1Q_COLS(9, 17), MCP_K1Q_COLS(13, 25), MCP_K1Q_COLS(15, 29),
                          MCP_K1Q_COLS(16, 33)};

#if MCP_WITH_K1R
// ---------------- K1R (warp triads: the GEMM1 role split by columns; r mod 8 in 1..2) ----------
template <int NTM, int TAIL, int MT2, int KH>
void launch_r(const K1SParams& prm, int grid, size_t smem, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(K1R_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k1r_fg_triads<NTM, TAIL, MT2, KH>, prm);
}
#define MCP_K1R_E(NTM, TAIL, MT2, KH) \
  {NTM, TAIL, MT2, KH, &launch_r<NTM, TAIL, MT2, KH>, \
   (const void*)&k1r_fg_triads<NTM, TAIL, MT2, KH>}
#define MCP_K1R_COLS(MT2, KH) MCP_K1R_E(1, 1, MT2, KH), MCP_K1R_E(1, 2, MT2, KH)
const EntryS kTableR[] = {MCP_K1R_COLS(1, 1),  MCP_K1R_COLS(3, 5),  MCP_K1R_COLS(5, 9),
                          MCP_K1R_COLS(9, 17), MCP_K1R_COLS(13, 25), MCP_K1R_COLS(15, 29),
                          MCP_K1R_COLS(16, 33)};
constexpr int kEntriesR = sizeof(kTableR) / sizeof(kTableR[0]);
#endif

bool select_stream(int64_t n, int r, int64_t p_pad, int64_t ldv, int sms, K1Variant& v) {
  if (n > 128) return false;
  const int MT = (int)ceil_div(n, 8);
  const int kst = (int)(ldv / 4);
  const int mth_need = (MT + 1) / 2, kh_need = kst;
  int ntm, tail;
  if (r <= 8) { ntm = 1; tail = 0; }
  else if (r <= 10 && MCP_CFG_DFMA_TAIL) { ntm = 1; tail = r - 8; }
  else { ntm = 2; tail = 0; }          // r > 16: several 16-column blocks, one per CTA
  int e = -1;
  for (int i = 0; i < kEntriesS && e < 0; ++i)
    if (kTableS[i].NTM == ntm && kTableS[i].TAIL == tail && kTableS[i].MTH >= mth_need &&
        kTableS[i].KH >= kh_need && 2 * kTableS[i].MTH >= MT + (8 * MT > n ? 0 : 0))
      e = i;
  if (e < 0) return false;
  const int mtm = kTableS[e].MTH;
  const int cw = 8 * ntm + tail;
  // Copy units of spc slabs: the bulk-copy engine costs ~660 cycles per copy per SM whatever
  // its size (tools/probe_tma.cu), so units must be >= ~24 KB to reach HBM bandwidth.  Every
  // ring stage must be consumed by a fixed set of pairs (mbarrier parity waits cannot tell
  // phase u from u + 2): spc in {7, 14} puts every pair in every unit, spc in {1, 2} needs a
  // ring depth that is a multiple of K1S_PAIRS.
  const size_t slab = (size_t)K1S_SR * ldv * 8;
  const size_t fixed = k1s_fixed_bytes(kTableS[e].KH, ntm, cw, K1S_PAIRS);
  const size_t budget = 227 * 1024 - 1024 - fixed;
  int spc = 0, S = 0;
  for (int cand : {1, 2, 7, 14}) {   // smallest unit >= 24 KB, else the largest that fits
    int st = (int)(budget / (cand * slab + 16));
    if (cand < K1S_PAIRS) {
      if (st > 4 * K1S_PAIRS) st = 4 * K1S_PAIRS;
      st -= st % K1S_PAIRS;
      if (st < K1S_PAIRS) continue;
    } else {
      if (st > 8) st = 8;
      if (st < 2) continue;
    }
    spc = cand;
    S = st;
    if (cand * slab >= 24 * 1024) break;
  }
  if (spc == 0) return false;
  if ((p_pad / K1S_SR) % spc != 0) return false;
  const size_t stage = (size_t)spc * slab;
  const size_t stage_need =
      (size_t)K1S_PAIRS * MT * 8 * cw * 8 + (size_t)2 * K1S_PAIRS * cw * 8;
  if ((size_t)S * stage < stage_need) return false;
  const size_t smem = (size_t)S * stage + fixed + 16 * (size_t)S;
  if (!ensure_dyn_smem(kTableS[e].fn, smem)) return false;
  v.kind = 1;
  v.dtype = MCP_F64;
  v.RB = cw;
  v.MTW = mtm;
  v.MT = MT;
  v.n_chunks = 0;
  v.n_pad = MT * 8;
  v.rbs = (int)ceil_div(r, cw);
  v.num_tiles = p_pad / K1S_SR;
  int64_t G = sms;
  if (G < v.rbs) G = v.rbs;
  G -= G % v.rbs;
  int64_t gp = G / v.rbs;
  if (gp > v.num_tiles / spc) gp = v.num_tiles / spc;
  if (gp < 1) gp = 1;
  v.gp = (int)gp;
  v.grid = v.gp * v.rbs;
  v.stages = S;
  v.MTW2 = spc;
  v.smem = smem;
  v.entry = e;
  v.afrag_elems = 0;
  v.ypart_elems = (size_t)v.rbs * v.gp * v.n_pad * cw;
  v.wpart_elems = (size_t)v.rbs * v.gp * cw;
  v.name = "k1s_fg_stream<f64,DMMA=" + std::to_string(8 * ntm) + ",DFMA=" +
           std::to_string(tail) + ",MTH=" + std::to_string(mtm) + ",KH=" +
           std::to_string(kTableS[e].KH) + ",S=" + std::to_string(S) + ">";
  return true;
}

// K1P: same column / m-tile split as K1S, a private ring of SP >= 2 slabs per pair.
// flavor 0: K1P, 1: K1Q, 2: K1R
bool select_pairs(int64_t n, int r, int64_t p_pad, int64_t ldv, int sms, K1Variant& v,
                  int flavor) {
  if (n > 128) return false;
  const bool specialised = flavor >= 1;
#if MCP_WITH_K1R
  const EntryS* table = flavor == 2 ? kTableR : specialised ? kTableQ : kTableP;
  const int n_entries = flavor == 2 ? kEntriesR : kEntriesS;
#else
  if (flavor == 2) return false;
  const EntryS* table = specialised ? kTableQ : kTableP;
  const int n_entries = kEntriesS;
#endif
  const int MT = (int)ceil_div(n, 8);
  const int kst = (int)(ldv / 4);
  const int mth_need = (MT + 1) / 2, kh_need = kst;
  int ntm, tail;
  if (r <= 8) { ntm = 1; tail = 0; }
  else if (r <= 10 && MCP_CFG_DFMA_TAIL) { ntm = 1; tail = r - 8; }
  else { ntm = 2; tail = 0; }
  if (flavor == 2 && tail == 0) return false;   // triads only pay off with DFMA tail columns
  int e = -1;
  for (int i = 0; i < n_entries && e < 0; ++i)
    if (table[i].NTM == ntm && table[i].TAIL == tail &&
        table[i].MTH >= (specialised ? MT : mth_need) && table[i].KH >= kh_need)
      e = i;
  if (e < 0) return false;
  const int cw = 8 * ntm + tail;
  const size_t slab = (size_t)K1S_SR * ldv * 8;
#if MCP_WITH_K1R
  const int NPR = flavor == 2 ? K1R_TRIADS : specialised ? K1Q_PAIRS : K1P_PAIRS;
#else
  const int NPR = specialised ? K1Q_PAIRS : K1P_PAIRS;
#endif
#if MCP_WITH_K1R
  const size_t fixed = flavor == 2    ? k1r_fixed_bytes(table[e].KH, ntm, cw)
                       : specialised ? k1q_fixed_bytes(table[e].KH, ntm, cw)
                                     : k1p_fixed_bytes(table[e].KH, ntm, cw);
#else
  const size_t fixed = specialised ? k1q_fixed_bytes(table[e].KH, ntm, cw)
                                   : k1p_fixed_bytes(table[e].KH, ntm, cw);
#endif
  const size_t budget = 227 * 1024 - 1024 - fixed;
  int SP = (int)(budget / ((size_t)NPR * (slab + 8)));
  if (SP > 4) SP = 4;
  if (SP < 2) return false;
  const size_t ring_bytes = (size_t)NPR * SP * slab;
  const size_t stage_need = ((size_t)NPR * MT * 8 * cw + (size_t)2 * NPR * cw) * 8;
  if (ring_bytes < stage_need) return false;
  size_t smem = ring_bytes + fixed + 8 * (size_t)NPR * (SP + 4);
  if (!ensure_dyn_smem(table[e].fn, smem)) return false;
  v.kind = flavor == 2 ? 6 : specialised ? 4 : 3;
  v.dtype = MCP_F64;
  v.RB = cw;
  v.MTW = table[e].MTH;
  v.MT = MT;
  v.n_chunks = 0;
  v.n_pad = MT * 8;
  v.rbs = (int)ceil_div(r, cw);
  v.num_tiles = p_pad / K1S_SR;
  int64_t G = sms;
  if (G < v.rbs) G = v.rbs;
  G -= G % v.rbs;
  int64_t gp = G / v.rbs;
  if (gp > v.num_tiles) gp = v.num_tiles;
  if (gp < 1) gp = 1;
  v.gp = (int)gp;
  v.grid = v.gp * v.rbs;
  v.stages = SP;
  v.MTW2 = 1;
  v.smem = smem;
  v.entry = e;
  v.afrag_elems = 0;
  v.ypart_elems = (size_t)v.rbs * v.gp * v.n_pad * cw;
  v.wpart_elems = (size_t)v.rbs * v.gp * cw;
  v.name = std::string(flavor == 2 ? "k1r_fg_triads" : specialised ? "k1q_fg_pairs" : "k1p_fg_pairs") + "<f64,DMMA=" +
           std::to_string(8 * ntm) + ",DFMA=" + std::to_string(tail) +
           (specialised ? ",MT2=" : ",MTH=") + std::to_string(table[e].MTH) + ",KH=" +
           std::to_string(table[e].KH) + ",SP=" + std::to_string(SP) + ">";
  return true;
}

template <int NL, int T, int RB>
void launch_x(const K1WParams& prm, const CUtensorMap* tm, int grid, size_t smem, cudaStream_t s) {
  launch_pdl(k1x_fg_dmma<NL, T, RB>, dim3(grid), dim3(K1X_THREADS), smem, s, *tm, prm);
}

// K1X: fp32 sets with a chunk-aligned pitch (one 3-D TMA per tile): 384 < n <= 512 (NL = 512,
// T = 32, RB = 16) or, with K1X_1024, 768 < n <= 1024 (NL = 1024, T = 16, RB = 8)
bool select_x(int dtype, int64_t n, int r, int64_t p_pad, int64_t ldv, int sms, K1Variant& v) {
  if (dtype != MCP_F32 || ldv % 32 != 0) return false;
  int nl = 0, tt = 0, rb = 0;
  const void* fn = nullptr;
  size_t smem = 0;
  if (n > 384 && n <= 512 && r >= 12) {
    nl = 512, tt = 32, rb = 16;
    fn = (const void*)k1x_fg_dmma<512, 32, 16>;
    smem = k1x_smem_bytes<512, 32, 16>();
#if MCP_CFG_K1X_1024
  } else if (n > 768 && n <= 1024 && r >= 6) {
    nl = 1024, tt = 16, rb = 8;
    fn = (const void*)k1x_fg_dmma<1024, 16, 8>;
    smem = k1x_smem_bytes<1024, 16, 8>();
#endif
  } else {
    return false;
  }
  if (!ensure_dyn_smem(fn, smem)) return false;
  const int64_t T = p_pad / tt;
  v.kind = 8;
  v.dtype = dtype;
  v.RB = rb;
  v.cl = 1;
  v.cpw = 1;
  v.t_rows = tt;
  v.n_pad = nl;
  v.n_chunks = v.n_pad / 64;
  v.rbs = (int)ceil_div(r, rb);
  v.num_tiles = T;
  const int Nc = (int)std::min<int64_t>(sms, (int64_t)v.rbs * T);
  k1w_split(T, v.rbs, Nc, v.groups, v.t_main);
  int mx = 1;
  for (int b = 0; b < v.rbs; ++b)
    mx = std::max(mx, k1w_used_slots(b, T, v.rbs, Nc, v.groups, v.t_main));
  v.gp = mx;
  v.grid = Nc;
  v.smem = smem;
  v.entry = 0;
  v.afrag_elems = (size_t)v.rbs * v.n_chunks * 16 * (rb / 8) * 32;
  v.ypart_elems = (size_t)v.rbs * v.gp * v.n_pad * rb;
  v.wpart_elems = (size_t)v.rbs * v.gp * rb;
  v.name = std::string("k1x_fg_dmma<f32,NL=") + std::to_string(nl) + ",T=" + std::to_string(tt) +
           ",RB=" + std::to_string(rb) + ",16 warps,G=" + std::to_string(v.groups) +
           (v.t_main < T ? ",+ranges" : "") + ">";
  return true;
}

}  // namespace

// The one-kernel reduce + finish (K3F) applies when its w block holds every w and the factor
// Gram fits its shared memory; it forms the tail pieces itself, so any K1 that needs no prep
// launch qualifies.
bool k1_fuses_tail(const K1Variant& v, int64_t n, int r) {
  (void)n;
  return (v.kind == 1 || v.kind == 3 || v.kind == 4 || v.kind == 6) && r <= K3F_MAXR &&
         v.rbs * v.RB <= K3W_X;
}

int64_t obs_pitch(int dtype, int64_t n) {
  if (dtype == MCP_F64) {
    // == 4 (mod 16) doubles: conflict-free fragment loads straight from the TMA-staged rows
    int64_t ldv = n < 4 ? 4 : n;
    while (ldv % 16 != 4) ++ldv;
    return ldv;
  }
  // fp32: whole 32-float chunks for n > 128 (the 3-D chunk tensor maps of K1X and the fast
  // mode need ldv % 32 == 0), else 16-byte rows
  return n > 128 ? round_up(n, 32) : round_up(n, 4);
}

bool k1_select(int dtype, int64_t n, int r, int64_t p_pad, int sms, K1Variant& v,
               std::string& why) {
  v = K1Variant();
  // K1R is opt-in (MCP_K1R=1): at c2 it measured 5% slower than K1Q
#if MCP_WITH_K1R
  if (dtype == MCP_F64 && select_pairs(n, r, p_pad, obs_pitch(dtype, n), sms, v, 2)) return true;
#endif
  v = K1Variant();
  if (dtype == MCP_F64 && MCP_CFG_K1Q &&
      select_pairs(n, r, p_pad, obs_pitch(dtype, n), sms, v, 1))
    return true;
  v = K1Variant();
  if (dtype == MCP_F64 && MCP_CFG_K1P &&
      select_pairs(n, r, p_pad, obs_pitch(dtype, n), sms, v, 0))
    return true;
  v = K1Variant();
  if (dtype == MCP_F64 && MCP_CFG_K1S &&
      select_stream(n, r, p_pad, obs_pitch(dtype, n), sms, v))
    return true;
  v = K1Variant();
  if (MCP_CFG_K1X && select_x(dtype, n, r, p_pad, obs_pitch(dtype, n), sms, v)) return true;
  v = K1Variant();
  // K1G when registers cap K1's column block at a quarter (or less) of K1G's: e.g. n = 1024,
  // r = 256 (c5): K1 RB = 16 vs K1G RB = 64 -> 4x fewer passes over V (measured 18% faster);
  // at n = 512, r = 64 (c3) K1's RB = 32 keeps Y in registers and wins by 4%.
  int rb_k1 = 8;
  {
    int mtw1 = 1;
    while (mtw1 < (int)ceil_div(n, K1_NK)) mtw1 *= 2;
    const int r8_ = (int)round_up(r, 8);
    while (rb_k1 < r8_ && rb_k1 < 64) rb_k1 *= 2;
    if (mtw1 <= 32 && rb_k1 > max_rb_for(mtw1)) rb_k1 = max_rb_for(mtw1);
  }
  int rb_g = 16;
  while (rb_g < (int)round_up(r, 8) && rb_g < 64) rb_g *= 2;
  const bool use_g = MCP_CFG_FORCE_K1G ? true : (rb_g >= 4 * rb_k1 || n > 2048);
  if (MCP_CFG_K1G && use_g && n > 128) {   // any n: Y lives in L2 (or TMEM)
    int rb = rb_g;
    int tm = 0;
    // K1GT: the Y partial fits TMEM when n_chunks * RB <= 512 (RB 16 or 32)
    const int nch = (int)ceil_div(n, K1_NK);
    if (MCP_CFG_K1GT_HALF && rb_g == 64 && nch * 32 <= 512) {
      tm = 1;   // RB = 64 with the first half of the partial in TMEM, the rest in L2
    } else if (MCP_CFG_K1GT && nch * 16 <= 512) {
      tm = 1;
      rb = (nch * 32 <= 512 && rb_g >= 32) ? 32 : 16;
      // 16 warps (column halves, 128 TMEM columns per thread) when RB = 32 and n <= 1024
      if (MCP_CFG_K1GT_NW == 16 && rb == 32 && nch <= 16) tm = 2;
    }
    int e = -1;
    for (int i = 0; i < kEntriesG; ++i)
      if (kTableG[i].dtype == dtype && kTableG[i].RB == rb && kTableG[i].MTW == tm) e = i;
    if (e >= 0) {
      if (ensure_dyn_smem(kTableG[e].fn, kTableG[e].smem)) {
        const int n_chunks = (int)ceil_div(n, K1_NK);
        v.kind = 5;
        v.dtype = dtype;
        v.RB = rb;
        v.MTW = 0;
        v.n_chunks = n_chunks;
        v.n_pad = n_chunks * K1_NK;
        v.rbs = (int)ceil_div(r, rb);
        v.num_tiles = p_pad / K1_TP;
        // every SM busy: K1X's split (groups striding the main tiles + leftover tail ranges)
        const int64_t T = v.num_tiles;
        const int Nc = (int)std::min<int64_t>(sms, (int64_t)v.rbs * T);
        k1w_split(T, v.rbs, Nc, v.groups, v.t_main);
        int mx = 1;
        for (int b = 0; b < v.rbs; ++b)
          mx = std::max(mx, k1w_used_slots(b, T, v.rbs, Nc, v.groups, v.t_main));
        v.gp = mx;
        v.grid = Nc;
        v.smem = kTableG[e].smem;
        v.entry = e;
        v.afrag_elems = (size_t)v.rbs * v.n_chunks * 16 * (rb / 8) * 32;
        v.ypart_elems = (size_t)v.rbs * v.gp * v.n_pad * rb;
        v.wpart_elems = (size_t)v.rbs * v.gp * rb;
        v.name = std::string(tm ? "k1gt_fg_dmma<" : "k1g_fg_dmma<") +
                 (dtype == MCP_F64 ? "f64" : "f32") + ",RB=" + std::to_string(rb) +
                 (tm == 2 ? ",16 warps" : "") + ">";
        return true;
      }
    }
  }
  v = K1Variant();
  const int n_chunks = (int)ceil_div(n, K1_NK);
  int mtw = 1;
  while (mtw < n_chunks) mtw *= 2;
  if (mtw > 32) {
    why = "n = " + std::to_string(n) + " exceeds this build's FP64 kernel limit (2048)";
    return false;
  }
  const int r8 = (int)round_up(r, 8);
  int rb = 8;
  while (rb < r8 && rb < 64) rb *= 2;
  if (rb > max_rb_for(mtw)) rb = max_rb_for(mtw);
  int e = -1;
  for (int i = 0; i < kEntries; ++i)
    if (kTable[i].dtype == dtype && kTable[i].RB == rb && kTable[i].MTW == mtw) e = i;
  if (e < 0) {
    why = "no K1 variant for this shape";
    return false;
  }
  const int occ = occupancy(e);
  if (occ < 1) {
    why = "K1 variant cannot be resident on this device";
    return false;
  }
  v.dtype = dtype;
  v.RB = rb;
  v.MTW = mtw;
  v.n_chunks = n_chunks;
  v.n_pad = n_chunks * K1_NK;
  v.rbs = (int)ceil_div(r, rb);
  v.num_tiles = p_pad / K1_TP;
  int64_t G = (int64_t)sms * occ;
  if (G < v.rbs) G = v.rbs;
  G -= G % v.rbs;
  int64_t gp = G / v.rbs;
  if (gp > v.num_tiles) gp = v.num_tiles;
  if (gp < 1) gp = 1;
  v.gp = (int)gp;
  v.grid = v.gp * v.rbs;
  v.smem = kTable[e].smem;
  v.entry = e;
  v.afrag_elems = (size_t)v.rbs * v.n_chunks * 16 * (rb / 8) * 32;
  v.ypart_elems = (size_t)v.rbs * v.gp * v.n_pad * rb;
  v.wpart_elems = (size_t)v.rbs * v.gp * rb;
  v.name = std::string("k1_fg_dmma<") + (dtype == MCP_F64 ? "f64" : "f32") + ",RB=" +
           std::to_string(rb) + ",MTW=" + std::to_string(mtw) + ">";
  return true;
}

int k1_launch(const K1Variant& v, const void* dV, int64_t ldv, int n, const double* dnu,
              double nu_const, const double* A, int r, const double* Afrag, int d, double* Ypart,
              double* wpart, cudaStream_t s, const void* tmap) {
  if (v.entry < 0) return 1;
  if (v.kind == 8) {
    if (!tmap) return 1;
    K1WParams wp;
    wp.num_tiles = v.num_tiles;
    wp.n = n;
    wp.n_pad = v.n_pad;
    wp.nu = dnu;
    wp.nu_const = nu_const;
    wp.Afrag = Afrag;
    wp.d = d;
    wp.rbs = v.rbs;
    wp.nclusters = v.grid / v.cl;
    wp.groups = v.groups;
    wp.t_main = v.t_main;
    wp.slots = v.gp;
    wp.Ypart = Ypart;
    wp.wpart = wpart;
#if MCP_CFG_K1X_1024
    if (v.n_pad == 1024)
      launch_x<1024, 16, 8>(wp, static_cast<const CUtensorMap*>(tmap), v.grid, v.smem, s);
    else
#endif
      launch_x<512, 32, 16>(wp, static_cast<const CUtensorMap*>(tmap), v.grid, v.smem, s);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 1;
  }
  if (v.kind == 1 || v.kind == 3 || v.kind == 4 || v.kind == 6) {
    K1SParams sp;
    sp.V = static_cast<const double*>(dV);
    sp.ldv = ldv;
    sp.num_slabs = v.num_tiles;
    sp.n = n;
    sp.MT = v.MT;
    sp.nu = dnu;
    sp.nu_const = nu_const;
    sp.A = A;
    sp.r = r;
    sp.d = d;
    sp.rbs = v.rbs;
    sp.gp = v.gp;
    sp.stages = v.stages;
    sp.spc = v.MTW2;
    sp.Ypart = Ypart;
    sp.wpart = wpart;
#if MCP_WITH_K1R
    if (v.kind == 6) {
      kTableR[v.entry].launch(sp, v.grid, v.smem, s);
      return cudaPeekAtLastError() == cudaSuccess ? 0 : 1;
    }
#endif
    (v.kind == 1 ? kTableS : v.kind == 3 ? kTableP : kTableQ)[v.entry].launch(sp, v.grid, v.smem, s);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 1;
  }
  K1Params prm;
  prm.V = dV;
  prm.ldv = ldv;
  prm.num_tiles = v.num_tiles;
  prm.n = n;
  prm.n_chunks = v.n_chunks;
  prm.n_pad = v.n_pad;
  prm.nu = dnu;
  prm.nu_const = nu_const;
  prm.Afrag = Afrag;
  prm.d = d;
  prm.rbs = v.rbs;
  prm.gp = v.gp;
  prm.groups = v.groups;
  prm.t_main = v.t_main;
  prm.Ypart = Ypart;
  prm.wpart = wpart;
  CUtensorMap tm_y;
  if (v.kind == 5) {
    // the Y partial as rows of RB doubles; box = one warp's 8 x RB GEMM2 chunk result
    if (!mcp_internal::make_tmap_f64(&tm_y, Ypart, (uint64_t)v.RB,
                                     (uint64_t)v.rbs * v.gp * v.n_pad, 8 * (uint64_t)v.RB,
                                     (uint32_t)v.RB, 8, CU_TENSOR_MAP_SWIZZLE_NONE))
      return 1;
    g_k1g_tmap = &tm_y;
  }
  (v.kind == 5 ? kTableG : kTable)[v.entry].launch(prm, v.grid, v.smem, s);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace mcp
