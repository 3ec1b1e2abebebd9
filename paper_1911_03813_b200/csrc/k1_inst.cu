// Instantiations of the K1 FP64 kernel family and the host-side variant selection.
#include <atomic>

#include "momentcp_b200.h"
#include "k1_dispatch.h"
#include "k1_fp64.cuh"

namespace mcp {
namespace {

template <typename VT, int RB, int MTW>
void launch_t(const K1Params& prm, int grid, size_t smem, cudaStream_t s) {
  k1_fg_dmma<VT, RB, MTW><<<grid, K1_THREADS, smem, s>>>(prm);
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
constexpr int kEntries = sizeof(kTable) / sizeof(kTable[0]);
std::atomic<int> g_occ[kEntries];
std::atomic<bool> g_occ_init{false};

int max_rb_for(int mtw) {
  switch (mtw) {
    case 1: case 2: case 4: return 64;
    case 8: return 32;
    case 16: return 16;
    default: return 8;
  }
}

int occupancy(int e) {
  if (!g_occ_init.exchange(true))
    for (int i = 0; i < kEntries; ++i) g_occ[i].store(-1);
  int o = g_occ[e].load();
  if (o >= 0) return o;
  const Entry& en = kTable[e];
  if (cudaFuncSetAttribute(en.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)en.smem) !=
      cudaSuccess) {
    (void)cudaGetLastError();
    return 0;
  }
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, en.fn, K1_THREADS, en.smem) !=
      cudaSuccess) {
    (void)cudaGetLastError();
    return 0;
  }
  g_occ[e].store(occ);
  return occ;
}

}  // namespace

bool k1_select(int dtype, int64_t n, int r, int64_t p_pad, int sms, K1Variant& v,
               std::string& why) {
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
              double nu_const, const double* Afrag, int d, double* Ypart, double* wpart,
              cudaStream_t s) {
  if (v.entry < 0) return 1;
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
  prm.Ypart = Ypart;
  prm.wpart = wpart;
  kTable[v.entry].launch(prm, v.grid, v.smem, s);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace mcp
