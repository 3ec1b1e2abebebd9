// Internal view of a momentcp context shared by the C-ABI translation units (abi.cu, lbfgs.cu).
// Not part of the public ABI (include/momentcp_b200.h): the struct layout may change freely.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "momentcp_b200.h"
#include "k1_dispatch.h"
#include "tail_pieces.cuh"

namespace mcp_internal {

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

struct GraphEntry {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
};

}  // namespace mcp_internal

struct mcp_ctx {
  int device = 0;
  int sms = 0;
  cudaStream_t stream = nullptr;
  mutable std::mutex mu;
  std::string err;

  bool loaded = false;
  int dtype = MCP_F64;
  int64_t n = 0, p = 0, p_pad = 0, ldv = 0;
  void* dV = nullptr;
  double* dnu = nullptr;  // nullptr => uniform nu_const
  double nu_const = 0.0;

  mcp_internal::DevBuf dx, dout, dYw, dAfrag, dYpart, dwpart, dG, dC, dpart, dscalar, dflag;
  mcp_internal::DevBuf dticket;  // K3 last-block ticket of the fused peer publication
  mcp_internal::DevBuf dzbar;    // K1Z grid barrier: arrivals, generation, error flag (zeroed)
  void* hx = nullptr;
  size_t hx_bytes = 0;
  void* hout = nullptr;
  size_t hout_bytes = 0;

  // fast mode (tcgen05 TF32): fp32 copy of V when the set is fp64, tensor maps, prepared A^T
  float* dV32 = nullptr;       // == dV when dtype is fp32
  bool own_v32 = false;
  int64_t ldv32 = 0;
  bool tm_v_ready = false;
  CUtensorMap tm_v1, tm_v2, tm_a;
  float* dVlo32 = nullptr;     // fast mode K1T2: V - tf32(V), same layout as dV32
  CUtensorMap tm_l1, tm_l2;
  CUtensorMap tm_v3, tm_l3;    // K1T2 GEMM2: 3-D chunk maps over V / V_lo (ld % 32 == 0)
  bool tm_c_ready = false;
  bool tm_l3_ready = false;   // the V_lo chunk map (tm_l3) matches dVlo32
  CUtensorMap tm_w;            // K1X observation map (3-D, 32 x 32 x 16 boxes, 128-byte swizzle)
  int tm_w_kind = 0;           // tile rows of the K1X shape tm_w was encoded for (0: none)
  void* tm_a_addr = nullptr;
  int tm_a_rows = 0, tm_a_kpad = 0, tm_a_rb = 0;
  mcp_internal::DevBuf dAt;

  std::map<std::tuple<int, int, int>, mcp_internal::GraphEntry> graphs;
  bool timing = false;
  int timing_every = 1;      // time one K1/K5 launch in every timing_every (sampling)
  int64_t timing_seen = 0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> timed, event_pool;
  int last_launches = 0;
  std::string variant = "none";
  // run-time options (mcp_set_option)
  bool opt_fused_tail = true;   // MCP_OPT_FUSED_TAIL: K1 -> fused reduce+finish when eligible
  bool opt_small_kernel = true; // MCP_OPT_SMALL_KERNEL: small problems in one launch (K1Z)

  // optional row indirection of a view (stochastic path): row l of this view is row
  // gidx[*git * p + l] of gV (the parent's resident set); K1Z reads the rows in place and the
  // gathered copy in dV is only made for the other kernels
  const void* gV = nullptr;
  int64_t gldv = 0;
  int gdtype = MCP_F64;
  const int64_t* gidx = nullptr;
  const int* git = nullptr;
  // optional Adam update fused into K1Z's finish (mcp::K1ZAdam owned by the stochastic-path
  // workspace; applied only when the evaluation's x is the Adam variables)
  const void* z_adam = nullptr;

  // cached device-resident L-BFGS workspace (lbfgs.cu); freed with the graphs
  void* lbfgs_ws = nullptr;
  void (*lbfgs_ws_free)(void*) = nullptr;
  // cached stochastic-path workspace (adam.cu); freed with the graphs
  void* adam_ws = nullptr;
  void (*adam_ws_free)(void*) = nullptr;

  int fail(int code, const std::string& msg) {
    err = msg;
    return code;
  }
};

#define CUDA_TRY(ctx, expr)                                                               \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess) {                                                              \
      (void)cudaGetLastError();                                                           \
      return (ctx)->fail(MCP_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
    }                                                                                     \
  } while (0)

namespace mcp_internal {

// Shape of the fast-mode (K1T) launch.
struct K1TPlan {
  int RB = 0, rbs = 0, gp = 0, stages = 0, nkb = 0, mt2 = 0, r_pad = 0, kpad = 0;
  bool v2 = false;   // K1T2 (precomputed V_lo) instead of K1T (in-kernel split)
  bool zcat = false; // K1T2 concatenated GEMM1 (Z in two TMEM halves)
  bool serial = false;  // K1T2 tile order GEMM1(u), GEMM2(u) (one Z buffer)
  bool hint = false;    // K1T2 L2 eviction policy on the V reads
  int flush = 8;        // K1T2 tiles per fp64 flush of the fp32 TMEM Y
  bool g2_3d = false;   // K1T2 GEMM2 V loads as one 3-D TMA per operand and stage
  int wide = 0;         // K1T2 GEMM2 m-tiles with the N = 2 RB [P_hi | P_lo] product
  bool insplit = false; // K1T2 V_lo formed in shared memory (no V_lo copy in HBM)
  int mt_tr = 0;        // K1T2 transient GEMM2 m-tiles (accumulate in Z's columns)
  bool tr_wide = false; // K1T2: the transient m-tile is wide (all m-tiles wide at c3)
  bool drain_tma = false; // K1T2: partial adds by bulk tensor reduce-add (16 KB staging)
  int64_t num_tiles = 0;
  size_t smem = 0;
};

// Shape of the single-launch small-problem evaluation (K1Z, csrc/k1z_small.cuh).
struct K1ZPlan {
  bool on = false;
  bool pdl = false;   // launch with the programmatic-serialization attribute as well
  int G = 0, Gp = 0, rows_per_cta = 0, R = 0, ns = 0, np = 0, RP = 0, MT1 = 1, PS = 0;
  size_t smem = 0;
  std::string name;
};

// Shape of one evaluation's K1 launch.
struct EvalPlan {
  mcp::K1Variant k1;
  K1TPlan t;
  K1ZPlan z;
  int mode = MCP_MODE_FP64;
  int d = 0, r = 0;
};

// NVTX range over an entry point or a kernel role's enqueue (header-only NVTX3: a no-op unless
// a profiler injects itself)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define MCP_NVTX_CAT2(a, b) a##b
#define MCP_NVTX_CAT(a, b) MCP_NVTX_CAT2(a, b)
#define MCP_NVTX(name) mcp_internal::NvtxRange MCP_NVTX_CAT(_mcp_nvtx_, __LINE__)(name)

struct Guard {
  mcp_ctx* c;
  std::unique_lock<std::mutex> lk;
  explicit Guard(mcp_ctx* ctx) : c(ctx), lk(ctx->mu) { cudaSetDevice(ctx->device); }
};


void drop_graphs(mcp_ctx* c);
int ensure(mcp_ctx* c, DevBuf& b, size_t bytes);
int ensure_host(mcp_ctx* c, void*& p, size_t& have, size_t bytes);
int plan_eval(mcp_ctx* c, int d, int r, int mode, EvalPlan& pl);
// prep -> K1 -> K3 : dYw = [vec_F(Y) ; w] for the loaded rows (stream-ordered, capturable).
// signal: K3 also publishes the reduced piece to the peers' flags (multi-GPU exchange) once
// all of it is written.
int enqueue_partial(mcp_ctx* c, const EvalPlan& pl, const double* dx, double* dYw,
                    cudaStream_t s, const mcp::K3Signal* signal = nullptr);
// K4 : out = [f ; g_lam ; vec_F(g_A)] from x = [lam ; vec_F(A)] and [Y ; w]
int enqueue_finish(mcp_ctx* c, int d, int r, const double* dx, const double* dYw,
                   const double* alpha_dev, double alpha, double* dout, cudaStream_t s);
// Tails of k evaluations that shared one pass over V: run s has x = xs + s*sx (packed,
// [lam; vec_F(A)]), its Y block Y + s*n*r, w + s*r, output out + s*so (alpha on the host).
int enqueue_tails_batched(mcp_ctx* c, int d, int r, int k, const double* xs, int64_t sx,
                          const double* Y, const double* w, double alpha, double* out, int64_t so,
                          cudaStream_t s);
// A whole single-device evaluation x -> out: K1P + fused reduce/finish when available, else
// partial (K1 -> K3) + finish (K4).  Scratch [Y ; w] in c->dYw.
int enqueue_fg_full(mcp_ctx* c, const EvalPlan& pl, const double* dx, const double* alpha_dev,
                    double alpha, double* dout, cudaStream_t s);

// A context over rows gathered elsewhere (stochastic path): shares the parent's device and
// stream, V (p_pad = round_up(p, 896) rows of pitch ldv, zero padded) is owned by the caller,
// uniform weights 1/p.  Destroy with destroy_view_ctx.
mcp_ctx* make_view_ctx(const mcp_ctx* parent, void* dV, int dtype, int64_t p, int64_t ldv);
void destroy_view_ctx(mcp_ctx* v);
void release_ctx(mcp_ctx* c);

inline int grid_for(int64_t total, int threads, int cap) {
  int64_t b = (total + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return (int)b;
}

}  // namespace mcp_internal
