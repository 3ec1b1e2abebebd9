// C ABI of the momentcp B200 path (see include/momentcp_b200.h for the reference mapping).
//
// A context owns: the observation set resident in HBM (observation-major, padded), the
// per-evaluation workspaces, pinned staging for the host entry points and one CUDA graph per
// (d, r, mode) that replays  H2D(x) -> prep -> K1 -> K3 -> K4 -> D2H(f, g)  with one sync.
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

#include "momentcp_b200.h"
#include "k1_fp64.cuh"
#include "k5_gram.cuh"
#include "k_aux.cuh"
#include "pdl.h"
#include "k1_dispatch.h"
#include "k1t_tf32.cuh"
#include "k1z_small.cuh"
#include "ctx.h"

#include <cuda.h>
#include <cudaTypedefs.h>

using namespace mcp;

namespace {

thread_local std::string g_create_error;

// Transpose a variable-major n x ld source (row i = variable) into the observation-major
// p_pad x ldv device layout, zero padding included (dst pre-zeroed).
template <typename T>
__global__ void k_transpose_in(const T* __restrict__ src, int64_t n, int64_t p, int64_t ld,
                               T* __restrict__ dst, int64_t ldv) {
  __shared__ T tile[32][33];
  const int64_t l0 = (int64_t)blockIdx.x * 32, i0 = (int64_t)blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t i = i0 + k, l = l0 + threadIdx.x;
    if (i < n && l < p) tile[k][threadIdx.x] = src[i * ld + l];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t l = l0 + k, i = i0 + threadIdx.x;
    if (i < n && l < p) dst[l * ldv + i] = tile[threadIdx.x][k];
  }
}

template <typename T>
__global__ void k_count_nonfinite(const T* __restrict__ V, int64_t total, unsigned long long* bad) {
  unsigned long long local = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x)
    local += isfinite((double)V[i]) ? 0ull : 1ull;
  if (local) atomicAdd(bad, local);
}

__global__ void k_copy_f64(const double* __restrict__ src, double* __restrict__ dst, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

__global__ void k_check_nu(const double* __restrict__ nu, int64_t p, unsigned long long* bad) {
  unsigned long long local = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p;
       i += (int64_t)gridDim.x * blockDim.x)
    local += (isfinite(nu[i]) && nu[i] > 0.0) ? 0ull : 1ull;
  if (local) atomicAdd(bad, local);
}

}  // namespace

namespace mcp_internal {

void drop_graphs(mcp_ctx* c) {
  for (auto& kv : c->graphs) {
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    if (kv.second.graph) cudaGraphDestroy(kv.second.graph);
  }
  c->graphs.clear();
  if (c->lbfgs_ws) {
    c->lbfgs_ws_free(c->lbfgs_ws);
    c->lbfgs_ws = nullptr;
  }
  if (c->adam_ws) {
    c->adam_ws_free(c->adam_ws);
    c->adam_ws = nullptr;
  }
}

// Event pair bracketing one timed kernel launch (only when timing is on and not capturing).
std::pair<cudaEvent_t, cudaEvent_t>* timing_begin(mcp_ctx* c, cudaStream_t s) {
  if (!c->timing) return nullptr;
  if ((c->timing_seen++ % c->timing_every) != 0) return nullptr;
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &st) != cudaSuccess || st != cudaStreamCaptureStatusNone)
    return nullptr;
  std::pair<cudaEvent_t, cudaEvent_t> ev;
  if (!c->event_pool.empty()) {
    ev = c->event_pool.back();
    c->event_pool.pop_back();
  } else {
    cudaEventCreate(&ev.first);
    cudaEventCreate(&ev.second);
  }
  c->timed.push_back(ev);
  cudaEventRecord(ev.first, s);
  return &c->timed.back();
}

void timing_end(std::pair<cudaEvent_t, cudaEvent_t>* ev, cudaStream_t s) {
  if (ev) cudaEventRecord(ev->second, s);
}

int ensure(mcp_ctx* c, DevBuf& b, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (b.bytes >= bytes) return MCP_OK;
  drop_graphs(c);  // graphs hold raw pointers into the old buffer
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.bytes = 0;
  CUDA_TRY(c, cudaMalloc(&b.p, bytes));
  b.bytes = bytes;
  return MCP_OK;
}

int ensure_host(mcp_ctx* c, void*& p, size_t& have, size_t bytes) {
  if (have >= bytes) return MCP_OK;
  drop_graphs(c);
  if (p) cudaFreeHost(p);
  p = nullptr;
  have = 0;
  CUDA_TRY(c, cudaMallocHost(&p, bytes));
  have = bytes;
  return MCP_OK;
}

PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    else
      (void)cudaGetLastError();
  }
  return fn;
}

// 2-D fp64 tensor map (K53's V tiles): inner dim (contiguous) x outer dim, row pitch in bytes.
bool make_tmap_f64(CUtensorMap* m, const void* gaddr, uint64_t inner, uint64_t outer,
                   uint64_t pitch, uint32_t box_inner, uint32_t box_outer,
                   CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
  auto enc = tmap_encoder();
  if (!enc) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {pitch};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(gaddr), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 2-D fp32 tensor map: inner dim (contiguous) x outer dim, row pitch in bytes.
bool make_tmap_f32(CUtensorMap* m, void* gaddr, uint64_t inner, uint64_t outer, uint64_t pitch,
                   uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle sw) {
  auto enc = tmap_encoder();
  if (!enc) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {pitch};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, gaddr, dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 3-D fp32 tensor map over row-major rows of `ld` floats viewed as (32 floats, rows, ld / 32
// column chunks): one box of 32 x box_rows x box_chunks loads box_chunks bricks of
// box_rows x 128 B, chunk-major (the layout four 2-D boxes would produce), in ONE TMA.
bool make_tmap_f32_chunks(CUtensorMap* m, void* gaddr, uint64_t ld, uint64_t rows,
                          uint32_t box_rows, uint32_t box_chunks, CUtensorMapSwizzle sw) {
  auto enc = tmap_encoder();
  if (!enc || ld % 32) return false;
  cuuint64_t dims[3] = {32, rows, ld / 32};
  cuuint64_t strides[2] = {4 * ld, 128};
  cuuint32_t box[3] = {32, box_rows, box_chunks};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, gaddr, dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// an experiment build's forced column block disables the transient-m-tile widening
static bool forced_rb_ok(int forced) { return !(forced >= 16 && forced <= 64); }

int plan_tf32(mcp_ctx* c, int r, EvalPlan& pl) {
  K1TPlan& t = pl.t;
  const int64_t n = c->n;
  t.nkb = (int)ceil_div(n, 32);
  t.mt2 = (int)ceil_div(n, 128);
  // fp32 copy of V (fp64 sets), tensor maps over it
  if (!c->dV32) {
    if (c->dtype == MCP_F32) {
      c->dV32 = (float*)c->dV;
      c->ldv32 = c->ldv;
      c->own_v32 = false;
    } else {
      c->ldv32 = round_up(n, 4);
      CUDA_TRY(c, cudaMalloc(&c->dV32, sizeof(float) * (size_t)c->p_pad * c->ldv32));
      c->own_v32 = true;
      k_f64_to_f32<<<grid_for(c->p_pad * c->ldv32, 256, 16 * c->sms), 256, 0, c->stream>>>(
          (const double*)c->dV, c->dV32, c->p_pad, c->ldv, c->ldv32, n);
      CUDA_TRY(c, cudaGetLastError());
      CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    }
    c->tm_v_ready = false;
    c->tm_c_ready = false;
    c->tm_l3_ready = false;
  }
  if (!c->tm_v_ready) {
    if (!make_tmap_f32(&c->tm_v1, c->dV32, c->ldv32, c->p_pad, 4 * c->ldv32, 32, 128,
                       CU_TENSOR_MAP_SWIZZLE_128B) ||
        !make_tmap_f32(&c->tm_v2, c->dV32, c->ldv32, c->p_pad, 4 * c->ldv32, 32, 32,
                       CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B))
      return c->fail(MCP_ERR_CUDA, "cuTensorMapEncodeTiled failed for V");
    c->tm_v_ready = true;
  }
  // K1T2: V_lo formed in shared memory by splitter warps (MCP_CFG_K1T2_INSPLIT), else
  // precomputed once per set (falling back to K1T's in-kernel split if it does not fit)
  // The split pays where the UMMAs are compute-bound enough to spare shared-memory bandwidth:
  // measured c3 (RB = 64: N = 128 / 64 products) 5.46 -> 5.11 ms, c5 (RB = 48: N = 96 / 48)
  // 220 -> 238 ms -- so only when K1T2's column block is 64 (same formula as below).
  // transient GEMM2 m-tiles (serial order, zcat): tr m-tiles accumulate in Z's 2 RB columns,
  // so RB fits when 2 RB + (mt2 - tr) RB <= 512 with tr RB <= 2 RB
  auto transient_tr = [&](int rbv) -> int {
    if (!MCP_CFG_K1T2_TRANSIENT || !MCP_CFG_K1T2_SERIAL || !MCP_CFG_K1T_ZCAT || 2 * rbv > 256)
      return 0;
    for (int tr = 1; tr <= 2 && tr <= t.mt2; ++tr)
      if (2 * rbv + (t.mt2 - tr) * rbv <= 512) return tr;
    return 0;
  };
  const int rb_v2 = [&] {
    const int want = (int)std::min<int64_t>(64, round_up(r, 16));
    int rbv = want;
    while (rbv > 16 && ((MCP_CFG_K1T2_SERIAL ? 1 : 2) + t.mt2) * rbv > 512) rbv -= 16;
    if (rbv < want && transient_tr(want) > 0) rbv = want;
    return rbv;
  }();
  t.v2 = false;
  t.insplit = !MCP_CFG_K1T_V1 && MCP_CFG_K1T2_INSPLIT && rb_v2 >= 64;
  if (t.insplit) {
    t.v2 = true;
  } else if (!MCP_CFG_K1T_V1) {
    if (!c->dVlo32) {
      const size_t bytes = sizeof(float) * (size_t)c->p_pad * c->ldv32;
      if (cudaMalloc(&c->dVlo32, bytes) == cudaSuccess) {
        k_split_lo<<<grid_for(c->p_pad * c->ldv32, 256, 16 * c->sms), 256, 0, c->stream>>>(
            c->dV32, c->dVlo32, c->p_pad * c->ldv32);
        CUDA_TRY(c, cudaGetLastError());
        CUDA_TRY(c, cudaStreamSynchronize(c->stream));
        if (!make_tmap_f32(&c->tm_l1, c->dVlo32, c->ldv32, c->p_pad, 4 * c->ldv32, 32, 128,
                           CU_TENSOR_MAP_SWIZZLE_128B) ||
            !make_tmap_f32(&c->tm_l2, c->dVlo32, c->ldv32, c->p_pad, 4 * c->ldv32, 32, 32,
                           CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B))
          return c->fail(MCP_ERR_CUDA, "cuTensorMapEncodeTiled failed for V_lo");
      } else {
        (void)cudaGetLastError();
        c->dVlo32 = nullptr;
      }
    }
    t.v2 = c->dVlo32 != nullptr;
  }
  // K1T2's GEMM2 V reads: one 3-D TMA per 16 KB stage half when rows are whole 32-float chunks
  t.g2_3d = false;
  if (t.v2 && c->ldv32 % 32 == 0 && c->ldv32 >= 128 && MCP_CFG_K1T2_G2_3D) {
    if (!c->tm_c_ready)
      c->tm_c_ready = make_tmap_f32_chunks(&c->tm_v3, c->dV32, c->ldv32, c->p_pad, 32, 4,
                                           CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    if (!t.insplit && !c->tm_l3_ready)
      c->tm_l3_ready = make_tmap_f32_chunks(&c->tm_l3, c->dVlo32, c->ldv32, c->p_pad, 32, 4,
                                            CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    t.g2_3d = c->tm_c_ready && (t.insplit || c->tm_l3_ready);
  }
  // column block RB (the UMMA N): as wide as TMEM allows -- Z (K1T2: double-buffered) plus
  // Y[mt] for the n / 128 m-tiles -- since the 3xTF32 UMMAs are shared-memory-bandwidth bound
  // and the operand bytes per MAC fall with N.  K1T2 takes any multiple of 16 up to 64, K1T
  // powers of two.
  const bool v1 = !t.v2;
  t.serial = !v1 && MCP_CFG_K1T2_SERIAL != 0;
  t.hint = !v1 && MCP_CFG_K1T2_HINT != 0;
  t.flush = std::max(1, MCP_CFG_K1T2_FLUSH);
  const int zbufs = (v1 || t.serial) ? 1 : 2;
  int RB = 16;
  if (v1) {
    while (RB < r && RB < 64) RB *= 2;
    while (RB > 16 && (zbufs + t.mt2) * RB > 512) RB /= 2;
  } else {
    const int want = (int)std::min<int64_t>(64, round_up(r, 16));
    RB = want;
    while (RB > 16 && (zbufs + t.mt2) * RB > 512) RB -= 16;
    // prefer the widest block that does not add a column block over the narrowest
    const int rbs_w = (int)ceil_div(r, RB);
    while (RB > 16 && ceil_div(r, RB - 16) == rbs_w && (RB - 16) >= r / rbs_w) RB -= 16;
    const int forced = MCP_CFG_K1T2_RB;   // experiment builds only
    if (forced >= 16 && forced <= 64 && forced % 16 == 0 && (zbufs + t.mt2) * forced <= 512)
      RB = forced;
  }
  // transient m-tiles when they widen the column block (c5: 48 -> 64, four blocks instead of six)
  t.mt_tr = 0;
  if (!v1 && t.serial && forced_rb_ok(MCP_CFG_K1T2_RB)) {
    const int want = (int)std::min<int64_t>(64, round_up(r, 16));
    const int tr = transient_tr(want);
    if (want > RB && tr > 0) {
      RB = want;
      t.mt_tr = tr;
    }
  }
  // K1T2 with the concatenated GEMM1 when TMEM has room for two 2 RB-wide Z buffers
  t.zcat = !v1 && MCP_CFG_K1T_ZCAT && 2 * RB <= 256 && (2 * zbufs + t.mt2) * RB <= 512;
  if (t.mt_tr) t.zcat = true;   // transient m-tiles live in the concatenated Z's columns
  // every GEMM2 m-tile wide when one wide transient m-tile in Z's columns makes room for the
  // rest: 2 RB + (mt2 - 1) 2 RB <= 512 (c3: 4 m-tiles at RB = 64)
  t.tr_wide = false;
  if (!v1 && t.serial && t.zcat && !t.mt_tr && MCP_CFG_K1T2_TRANSIENT && MCP_CFG_K1T2_WIDE &&
      MCP_CFG_K1T2_TRWIDE && t.mt2 >= 2 && 2 * RB + (t.mt2 - 1) * 2 * RB <= 512) {
    const int spare_now = 512 - 2 * RB - t.mt2 * RB;
    if (spare_now / RB < t.mt2) {   // not all wide today
      t.mt_tr = 1;
      t.tr_wide = true;
    }
  }
  if ((zbufs + t.mt2 - t.mt_tr) * RB > 512)
    return c->fail(MCP_ERR_ARG, "n = " + std::to_string(n) + " exceeds the tf32x3 kernel limit");
  // GEMM2 m-tiles that get a second RB-column accumulator half from the spare TMEM columns
  t.wide = 0;
  if (!v1 && MCP_CFG_K1T2_WIDE != 0) {
    const int zw = t.zcat ? 2 * RB : RB;
    const int spare = 512 - zbufs * zw - (t.mt2 - t.mt_tr) * RB;
    t.wide = std::max(0, std::min(t.mt2 - t.mt_tr, spare / RB));
  }
  t.RB = RB;
  t.rbs = (int)ceil_div(r, RB);
  t.r_pad = t.rbs * RB;
  t.kpad = t.nkb * 32;
  const size_t budget = 227 * 1024;
  // the fp64 partial's adds (flushes, transient drains) by bulk tensor reduce-add need a 16 KB
  // staging area: taken unless it would cost a stage of the ring (transient m-tiles: always)
  bool drain_tma = !v1 && MCP_K1T2_DRAIN_TMA;
  if (drain_tma && !t.mt_tr &&
      (budget - k1t_smem_bytes(RB, 0, true)) / k1t_stage_bytes(RB) <
          (budget - k1t_smem_bytes(RB, 0, false)) / k1t_stage_bytes(RB))
    drain_tma = false;
  t.drain_tma = drain_tma;
  int ns = (int)((budget - k1t_smem_bytes(RB, 0, drain_tma)) / k1t_stage_bytes(RB));
  if (ns > 8) ns = 8;
  if (ns < 2) return c->fail(MCP_ERR_ARG, "tf32x3 stage ring does not fit");
  t.stages = ns;
  t.smem = k1t_smem_bytes(RB, ns, drain_tma);
  t.num_tiles = c->p_pad / K1T_TP;
  int64_t G = c->sms;
  if (G < t.rbs) G = t.rbs;
  G -= G % t.rbs;
  int64_t gp = G / t.rbs;
  if (gp > t.num_tiles) gp = t.num_tiles;
  t.gp = (int)std::max<int64_t>(gp, 1);
  int rc;
  if ((rc = ensure(c, c->dAt, sizeof(float) * 2 * (size_t)t.r_pad * t.kpad))) return rc;
  if (c->tm_a_addr != c->dAt.p || c->tm_a_rows != 2 * t.r_pad || c->tm_a_kpad != t.kpad ||
      c->tm_a_rb != RB) {
    if (!make_tmap_f32(&c->tm_a, c->dAt.p, t.kpad, 2 * t.r_pad, 4 * (uint64_t)t.kpad, 32, RB,
                       CU_TENSOR_MAP_SWIZZLE_128B))
      return c->fail(MCP_ERR_CUDA, "cuTensorMapEncodeTiled failed for A");
    c->tm_a_addr = c->dAt.p;
    c->tm_a_rows = 2 * t.r_pad;
    c->tm_a_kpad = t.kpad;
    c->tm_a_rb = RB;
  }
  if (!ensure_dyn_smem(!t.v2        ? (const void*)k1t_fg_tf32
                       : t.mt_tr ? (const void*)k1t2_fg_tf32<true>
                                 : (const void*)k1t2_fg_tf32<false>,
                       t.smem))
    return c->fail(MCP_ERR_CUDA, "cudaFuncSetAttribute failed for the tf32x3 kernel");
  pl.k1 = K1Variant();
  pl.k1.kind = 2;
  pl.k1.RB = RB;
  pl.k1.rbs = t.rbs;
  pl.k1.gp = t.gp;
  pl.k1.n_pad = t.mt2 * 128;
  pl.k1.ypart_elems = (size_t)t.rbs * t.gp * t.mt2 * 128 * RB;
  pl.k1.wpart_elems = 0;
  pl.k1.afrag_elems = 0;
  pl.k1.name = std::string(t.v2 ? "k1t2_fg_tf32" : "k1t_fg_tf32") + "<3xTF32,RB=" +
                std::to_string(RB) + ",S=" + std::to_string(ns) +
                (t.v2 ? std::string(t.serial ? ",serial" : ",lookahead") + (t.zcat ? ",zcat" : "") +
                             (t.hint ? ",l2hint" : "") +  (t.g2_3d ? ",g2tma3d" : "") + (t.wide ? ",wide=" + std::to_string(t.wide) : std::string()) + (MCP_CFG_K1T2_G2X2 ? ",g2x2" : "") + (t.insplit ? ",insplit" : "") + (t.drain_tma ? ",tmadrain" : "") + (t.mt_tr ? ",transient=" + std::to_string(t.mt_tr) + (t.tr_wide ? "w" : "") : std::string()) + ",flush=" + std::to_string(t.flush)
                      : std::string()) +
                ">";
  return MCP_OK;
}

// K1Z shape for (dtype, n, r, p): a function of those and the SM count only (the summation
// order -- and so the result bits -- must not depend on where the rows came from).
static bool k1z_pdl_ok(mcp_ctx* c);
static bool plan_k1z(const mcp_ctx* c, int r, K1ZPlan& z) {
  z = K1ZPlan();
  if (!MCP_CFG_K1Z || !c->opt_small_kernel) return false;
  const int64_t n = c->n, p = c->p;
  if (r > K1Z_MAXR || n > K1Z_MAXN || p < 1) return false;
  if (ceil_div(p, (int64_t)c->sms) > MCP_CFG_K1Z_MAX_ROWS) return false;
  const int dtype = c->gV ? c->gdtype : c->dtype;
  const size_t esz = dtype == MCP_F64 ? 8 : 4;
  z.RP = r <= 8 ? 8 : (r <= 16 ? 16 : 32);
  // staged rows: conflict-free 8 x 4 DMMA fragment loads (== 4 mod 16 doubles / mod 32 floats)
  const int64_t n4 = round_up(n, (int64_t)4);
  const int64_t mod = dtype == MCP_F64 ? 16 : 32;
  int64_t ns = n4;
  while (ns % mod != 4) ++ns;
  z.ns = (int)ns;
  z.np = (int)(n4 | 1);
  const int64_t max_g = MCP_CFG_K1Z_MAXG > 0 ? std::min<int64_t>(MCP_CFG_K1Z_MAXG, c->sms) : c->sms;
  // GEMM1 pass height: 8, 16 or 32 rows (1, 2 or 4 DMMA row tiles sharing the factor fragments)
  const int64_t rpc0 = ceil_div(p, max_g);
  const size_t budget = 226 * 1024;
  const size_t per_row = ns * esz + sizeof(double) * z.RP;
  // (32 columns: at most 16-row passes -- the Y_b tiles already take 128 registers)
  for (z.MT1 = rpc0 <= 8 ? 1 : ((rpc0 <= 16 || z.RP == 32) ? 2 : 4); z.MT1 >= 1; z.MT1 /= 2) {
    const int64_t RS = 8 * z.MT1;
    const size_t fixed =
        sizeof(double) * ((size_t)z.np * z.RP + (size_t)k1z_sz_elems(z.RP, z.MT1) + 3 * K1Z_T +
                          2 * (size_t)z.RP * z.RP + 3 * z.RP) + 8 * esz;
    if (fixed + (size_t)RS * per_row > budget) continue;   // a lower pass height may fit
    z.rows_per_cta = (int)round_up(rpc0, RS);
    z.Gp = (int)ceil_div(p, (int64_t)z.rows_per_cta);
    // tiny batches: extra CTAs without rows so that no CTA finishes more than 256 outputs
    z.G = (int)std::max<int64_t>(z.Gp, std::min<int64_t>(max_g, ceil_div(n * r + r, (int64_t)K1Z_T)));
    const int64_t Rmax = (int64_t)((budget - fixed) / per_row) / RS * RS;
    z.R = (int)std::min<int64_t>(z.rows_per_cta, Rmax);
    z.smem = fixed + (size_t)z.R * per_row;
    break;
  }
  if (z.MT1 < 1) return false;
  z.PS = (int)round_up(n * r + r, (int64_t)2);
  z.name = std::string("k1z_fg_small<") + (dtype == MCP_F64 ? "f64" : "f32") +
           ",RP=" + std::to_string(z.RP) + ",MT1=" + std::to_string(z.MT1) +
           ",G=" + std::to_string(z.G) + (z.G != z.Gp ? "/" + std::to_string(z.Gp) : std::string()) +
           ",R=" + std::to_string(z.R) + ">";
  z.on = true;
  return true;
}

int plan_eval(mcp_ctx* c, int d, int r, int mode, EvalPlan& pl) {
  if (!c->loaded) return c->fail(MCP_ERR_STATE, "no observation set loaded (call mcp_load_obs)");
  if (d < 2) return c->fail(MCP_ERR_ARG, "order must be >= 2, got " + std::to_string(d));
  if (r < 1) return c->fail(MCP_ERR_ARG, "rank must be >= 1, got " + std::to_string(r));
  if (mode != MCP_MODE_FP64 && mode != MCP_MODE_TF32X3)
    return c->fail(MCP_ERR_ARG, "unknown mode " + std::to_string(mode));
  pl.d = d;
  pl.r = r;
  pl.mode = mode;
  if (mode == MCP_MODE_TF32X3) {
    int rc = plan_tf32(c, r, pl);
    if (rc) return rc;
    const int64_t n = c->n;
    if ((rc = ensure(c, c->dx, sizeof(double) * (r + n * r + 1)))) return rc;
    if ((rc = ensure(c, c->dout, sizeof(double) * (1 + r + n * r)))) return rc;
    if ((rc = ensure(c, c->dYw, sizeof(double) * (n * r + r)))) return rc;
    if ((rc = ensure(c, c->dYpart, sizeof(double) * pl.k1.ypart_elems))) return rc;
    if ((rc = ensure(c, c->dG, sizeof(double) * (size_t)r * r))) return rc;
    if ((rc = ensure(c, c->dC, sizeof(double) * (size_t)r * r))) return rc;
    return MCP_OK;
  }
  std::string why;
  if (!k1_select(c->dtype, c->n, r, c->p_pad, c->sms, pl.k1, why))
    return c->fail(MCP_ERR_ARG, why);
  if (pl.k1.needs_tmap() && c->tm_w_kind != pl.k1.t_rows) {
    // K1X: one box = a whole tile (t_rows rows x n_pad / 32 chunks of 32 floats)
    if (!make_tmap_f32_chunks(&c->tm_w, c->dV, c->ldv, c->p_pad, pl.k1.t_rows,
                              (uint32_t)(pl.k1.n_pad / 32), CU_TENSOR_MAP_SWIZZLE_128B))
      return c->fail(MCP_ERR_CUDA, "cuTensorMapEncodeTiled failed for the K1X observation map");
    c->tm_w_kind = pl.k1.t_rows;
  }
  int rc;
  const int64_t n = c->n;
  if ((rc = ensure(c, c->dx, sizeof(double) * (r + n * r + 1)))) return rc;
  if ((rc = ensure(c, c->dout, sizeof(double) * (1 + r + n * r)))) return rc;
  if ((rc = ensure(c, c->dYw, sizeof(double) * (n * r + r)))) return rc;
  if ((rc = ensure(c, c->dAfrag, sizeof(double) * pl.k1.afrag_elems))) return rc;
  if ((rc = ensure(c, c->dYpart, sizeof(double) * pl.k1.ypart_elems))) return rc;
  if ((rc = ensure(c, c->dwpart, sizeof(double) * pl.k1.wpart_elems))) return rc;
  if ((rc = ensure(c, c->dG, sizeof(double) * (size_t)r * r))) return rc;
  if ((rc = ensure(c, c->dC, sizeof(double) * (size_t)r * r))) return rc;
  // K1Z only where the general chain is the 4-6 launch one (prep -> K1 -> K3 -> tail): the
  // two-launch pairs / stream kernels of n <= 128 fp64 sets measured faster than K1Z
  // (tools/sweep_small.py, profiles/r02/sweep_small.txt)
  if (pl.k1.needs_prep() && plan_k1z(c, r, pl.z)) {
    pl.z.pdl = k1z_pdl_ok(c);
    if ((rc = ensure(c, c->dYpart, sizeof(double) * (size_t)pl.z.G * pl.z.PS))) return rc;
    if (!c->dzbar.p) {
      if ((rc = ensure(c, c->dzbar, 4 * sizeof(unsigned)))) return rc;
      CUDA_TRY(c, cudaMemset(c->dzbar.p, 0, 4 * sizeof(unsigned)));
    }
  }
  return MCP_OK;
}

// fast mode: prep A^T hi/lo -> K1T -> K3 (Y) -> w from Y
int enqueue_partial_tf32(mcp_ctx* c, const EvalPlan& pl, const double* dx, double* dYw,
                         cudaStream_t s) {
  MCP_NVTX("K1T2 fast-mode partial");
  const K1TPlan& t = pl.t;
  const int n = (int)c->n, r = pl.r;
  k_prep_at_tf32<<<grid_for((int64_t)t.r_pad * t.kpad, 256, 4 * c->sms), 256, 0, s>>>(
      dx + r, n, r, t.r_pad, t.kpad, (float*)c->dAt.p,
      (t.insplit && MCP_K1T2_ASPLIT && t.serial) ? 1 : 0);
  K1TParams prm;
  prm.n = n;
  prm.r = r;
  prm.d = pl.d;
  prm.nkb = t.nkb;
  prm.mt2 = t.mt2;
  prm.RB = t.RB;
  prm.rbs = t.rbs;
  prm.gp = t.gp;
  prm.r_pad = t.r_pad;
  prm.stages = t.stages;
  prm.num_tiles = t.num_tiles;
  prm.nu = c->dnu;
  prm.nu_const = c->nu_const;
  prm.Ypart = (double*)c->dYpart.p;
  prm.zcat = t.zcat ? 1 : 0;
  prm.serial = t.serial ? 1 : 0;
  prm.hint = t.hint ? 1 : 0;
  prm.flush = t.flush;
  prm.g2_3d = t.g2_3d ? 1 : 0;
  prm.wide = t.wide;
  prm.insplit = t.insplit ? 1 : 0;
  prm.mt_tr = t.mt_tr;
  // the transient drain's bulk tensor reduce-add target: the fp64 partial as rows of RB
  CUtensorMap tm_y;
  prm.drain_tma = 0;
  if (t.drain_tma) {
    if (!make_tmap_f64(&tm_y, c->dYpart.p, (uint64_t)t.RB,
                       (uint64_t)t.rbs * t.gp * t.mt2 * 128, 8 * (uint64_t)t.RB, 8, 32,
                       CU_TENSOR_MAP_SWIZZLE_NONE))
      return c->fail(MCP_ERR_CUDA, "cuTensorMapEncodeTiled failed for the fast-mode partial");
    prm.drain_tma = 1;
  } else {
    tm_y = c->tm_a;   // unused
  }
  prm.tr_wide = t.tr_wide ? 1 : 0;
  // opt-in: GEMM2 as V P_hi with P_hi rounded to nearest (8-9% faster at c3 / c5, but normwise
  // error up to 7e-5 at reduced p -- too close to the stated 1e-4 to be the default)
  prm.g2x2 = MCP_CFG_K1T2_G2X2 ? 1 : 0;
  auto* ev = timing_begin(c, s);
  if (t.v2)
    (t.mt_tr ? k1t2_fg_tf32<true> : k1t2_fg_tf32<false>)<<<t.gp * t.rbs, t.insplit ? K1T2_THREADS_S : K1T2_THREADS, t.smem, s>>>(
        c->tm_v1, t.g2_3d ? c->tm_v3 : c->tm_v2, t.insplit ? c->tm_v1 : c->tm_l1,
        t.insplit ? (t.g2_3d ? c->tm_v3 : c->tm_v2) : (t.g2_3d ? c->tm_l3 : c->tm_l2), c->tm_a,
        tm_y, prm);
  else
    k1t_fg_tf32<<<t.gp * t.rbs, K1T_THREADS, t.smem, s>>>(c->tm_v1, c->tm_v2, c->tm_a, prm);
  timing_end(ev, s);
  const int64_t red_blocks = (int64_t)t.rbs * ceil_div((int64_t)n * t.RB, K3_X);
  k_reduce_partials<<<(int)std::min<int64_t>(red_blocks, 16 * c->sms), K3_T, 0, s>>>(
      (const double*)c->dYpart.p, nullptr, n, r, t.mt2 * 128, t.RB, t.rbs, t.gp, dYw);
  k_w_from_y<<<(int)ceil_div((int64_t)r * 32, 256), 256, 0, s>>>(dx + r, n, r, dYw);
  CUDA_TRY(c, cudaGetLastError());
  c->last_launches = 4;
  c->variant = pl.k1.name;
  return MCP_OK;
}

// prep -> K1 -> K3 : dYw = [vec_F(Y) ; w] for the loaded rows.
int enqueue_partial(mcp_ctx* c, const EvalPlan& pl, const double* dx, double* dYw,
                    cudaStream_t s, const K3Signal* signal) {
  if (pl.mode == MCP_MODE_TF32X3) {
    int rc = enqueue_partial_tf32(c, pl, dx, dYw, s);
    if (rc || !signal) return rc;
    k_publish<<<1, 32, 0, s>>>(*signal);
    CUDA_TRY(c, cudaGetLastError());
    return MCP_OK;
  }
  const K1Variant& v = pl.k1;
  const int n = (int)c->n, r = pl.r;
  int launches = 2;
  if (v.needs_prep()) {
    CUDA_TRY(c, launch_pdl(k_prep_afrag, dim3(grid_for(v.afrag_elems, 256, 4 * c->sms)), dim3(256),
                           0, s, dx + r, n, r, v.RB, v.rbs, v.n_chunks * 16,
                           (double*)c->dAfrag.p));
    ++launches;
  }
  auto* ev = timing_begin(c, s);
  int rc;
  {
    MCP_NVTX("K1 f+grad partial");
    rc = k1_launch(v, c->dV, c->ldv, n, c->dnu, c->nu_const, dx + r, r,
                   (const double*)c->dAfrag.p, pl.d, (double*)c->dYpart.p, (double*)c->dwpart.p,
                   s, &c->tm_w);
  }
  timing_end(ev, s);
  if (rc) {
    const cudaError_t e = cudaGetLastError();
    return c->fail(MCP_ERR_CUDA, std::string("K1 launch failed (") + v.name + "): " +
                                     cudaGetErrorString(e));
  }
  const int64_t red_blocks = (int64_t)v.rbs * ceil_div((int64_t)n * v.RB, K3_X) +
                             ceil_div((int64_t)v.rbs * v.RB, K3W_X);
  {
    // K3 under programmatic dependent launch (its launch overlaps K1's drain); with a signal it
    // also publishes the reduced piece to the peers (one launch instead of two)
    K3Signal sig;
    if (signal) {
      if (!c->dticket.p) {
        if ((rc = ensure(c, c->dticket, sizeof(unsigned)))) return rc;
        CUDA_TRY(c, cudaMemsetAsync(c->dticket.p, 0, sizeof(unsigned), s));
      }
      sig = *signal;
      sig.ticket = (unsigned*)c->dticket.p;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)std::min<int64_t>(red_blocks, 16 * c->sms));
    cfg.blockDim = dim3(K3_T);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CUDA_TRY(c, cudaLaunchKernelEx(&cfg, k_reduce_partials, (const double*)c->dYpart.p,
                                   (const double*)c->dwpart.p, n, r, v.n_pad, v.RB, v.rbs, v.gp,
                                   dYw, sig));
  }
  CUDA_TRY(c, cudaGetLastError());
  c->last_launches = launches;
  c->variant = v.name;
  return MCP_OK;
}

// k_tail_fused stages A in dynamic shared memory (beyond the 48 KB default for large n r)
static bool k4s_ready(int64_t nr) {
  if (ensure_dyn_smem((const void*)k_tail_fused, k4s_smem_bytes(K4S_MAX_NR))) return true;
  return k4s_smem_bytes(nr) <= 48 * 1024;
}

// one-CTA tail for small factor blocks; else the three-kernel tail (measured: at n r = 5000 the
// single CTA is ~10 us slower than the three parallel kernels)
static bool k4s_fits(int64_t n, int r) {
  const int64_t nr = n * r;
  return nr <= K4S_MAX_NR && r <= K4S_MAX_R && k4s_ready(nr);
}

// K4: tail from (x, Y, w) -> out = [f ; g_lam ; vec_F(g_A)].
int enqueue_finish_yw(mcp_ctx* c, int d, int r, const double* dx, const double* dY,
                      const double* dw, const double* alpha_dev, double alpha, double* dout,
                      cudaStream_t s) {
  MCP_NVTX("K4 tail");
  const int n = (int)c->n;
  if (k4s_fits(n, r)) {
    CUDA_TRY(c, launch_pdl(k_tail_fused, dim3(1), dim3(K4S_THREADS), k4s_smem_bytes((int64_t)n * r),
                           s, dx, dY, dw, n, r, d, alpha_dev, alpha, dout, (int64_t)0, (int64_t)0,
                           (int64_t)0, (int64_t)0));
    CUDA_TRY(c, cudaGetLastError());
    c->last_launches += 1;
    return MCP_OK;
  }
  CUDA_TRY(c, launch_pdl(k_tail_gram, dim3(grid_for((int64_t)r * r, K4A_WARPS, 16 * c->sms)),
                         dim3(32 * K4A_WARPS), 0, s, dx, n, r, d, (double*)c->dG.p,
                         (double*)c->dC.p));
  CUDA_TRY(c, launch_pdl(k_tail_vec, dim3(1), dim3(256), sizeof(double) * r, s, dx, dw,
                         (const double*)c->dG.p, (const double*)c->dC.p, n, r, alpha_dev, alpha,
                         dout));
  CUDA_TRY(c, launch_pdl(k_tail_ga, dim3(grid_for((int64_t)n * r, 256, 8 * c->sms)), dim3(256), 0,
                         s, dx, dY, (const double*)c->dC.p, n, r, d, dout));
  CUDA_TRY(c, cudaGetLastError());
  c->last_launches += 3;
  return MCP_OK;
}

int enqueue_finish(mcp_ctx* c, int d, int r, const double* dx, const double* dYw,
                   const double* alpha_dev, double alpha, double* dout, cudaStream_t s) {
  return enqueue_finish_yw(c, d, r, dx, dYw, dYw + c->n * r, alpha_dev, alpha, dout, s);
}

int enqueue_tails_batched(mcp_ctx* c, int d, int r, int k, const double* xs, int64_t sx,
                          const double* Y, const double* w, double alpha, double* out, int64_t so,
                          cudaStream_t s) {
  const int64_t n = c->n, nr = n * r;
  if (k4s_fits(n, r)) {
    k_tail_fused<<<k, K4S_THREADS, k4s_smem_bytes(nr), s>>>(xs, Y, w, (int)n, r, d, nullptr, alpha,
                                                            out, sx, nr, r, so);
    CUDA_TRY(c, cudaGetLastError());
    c->last_launches += 1;
    return MCP_OK;
  }
  for (int i = 0; i < k; ++i) {
    int rc = enqueue_finish_yw(c, d, r, xs + (int64_t)i * sx, Y + (int64_t)i * nr, w + (int64_t)i * r,
                               nullptr, alpha, out + (int64_t)i * so, s);
    if (rc) return rc;
  }
  return MCP_OK;
}

// Can a kernel be launched with the cooperative AND the programmatic-serialization attribute?
// Probed once per process with an empty kernel on the context's stream (never while capturing).
__global__ void k_k1z_probe() { pdl_wait(); }
static std::atomic<int> g_k1z_pdl{-1};   // -1 unknown, 0 no, 1 yes
static bool k1z_pdl_ok(mcp_ctx* c) {
  if (!MCP_CFG_K1Z_PDL || !pdl_enabled()) return false;
  int st = g_k1z_pdl.load();
  if (st >= 0) return st == 1;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(c->stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
    (void)cudaGetLastError();
    return false;   // decide at the next plan outside a capture
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2);
  cfg.blockDim = dim3(32);
  cfg.stream = c->stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_k1z_probe);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) (void)cudaGetLastError();
  g_k1z_pdl.store(e == cudaSuccess ? 1 : 0);
  return e == cudaSuccess;
}

// The whole evaluation in one cooperative launch (small problems, csrc/k1z_small.cuh).
static int enqueue_fg_small(mcp_ctx* c, const EvalPlan& pl, const double* dx,
                            const double* alpha_dev, double alpha, double* dout, cudaStream_t s) {
  MCP_NVTX("K1Z single-launch f+grad");
  const K1ZPlan& z = pl.z;
  K1ZParams prm;
  prm.V = c->gV ? c->gV : c->dV;
  prm.ldv = c->gV ? c->gldv : c->ldv;
  prm.idx = c->gV ? c->gidx : nullptr;
  prm.it_dev = c->gV ? c->git : nullptr;
  prm.nu = c->dnu;
  prm.nu_const = c->nu_const;
  prm.x = dx;
  prm.alpha_dev = alpha_dev;
  prm.alpha_host = alpha;
  prm.part = (double*)c->dYpart.p;
  prm.bar = (unsigned*)c->dzbar.p;
  prm.out = dout;
  prm.p = c->p;
  prm.n = (int)c->n;
  prm.r = pl.r;
  prm.d = pl.d;
  prm.rows_per_cta = z.rows_per_cta;
  prm.R = z.R;
  prm.ns = z.ns;
  prm.np = z.np;
  prm.PS = z.PS;
  prm.Gp = z.Gp;
  if (c->z_adam && static_cast<const K1ZAdam*>(c->z_adam)->x == dx)
    prm.adam = *static_cast<const K1ZAdam*>(c->z_adam);
  const bool f64 = (c->gV ? c->gdtype : c->dtype) == MCP_F64;
  void (*fn)(const K1ZParams) = nullptr;
#define MCP_K1Z_PICK(TV, RP_)                                                    \
  fn = z.MT1 == 1 ? k1z_fg_small<TV, RP_, 1>                                     \
                  : (z.MT1 == 2 ? k1z_fg_small<TV, RP_, 2> : k1z_fg_small<TV, RP_, 4>)
  if (f64) {
    if (z.RP == 8) MCP_K1Z_PICK(double, 8);
    else if (z.RP == 16) MCP_K1Z_PICK(double, 16);
    else fn = z.MT1 == 1 ? k1z_fg_small<double, 32, 1> : k1z_fg_small<double, 32, 2>;
  } else {
    if (z.RP == 8) MCP_K1Z_PICK(float, 8);
    else if (z.RP == 16) MCP_K1Z_PICK(float, 16);
    else fn = z.MT1 == 1 ? k1z_fg_small<float, 32, 1> : k1z_fg_small<float, 32, 2>;
  }
#undef MCP_K1Z_PICK
  if (!ensure_dyn_smem((const void*)fn, z.smem))
    return c->fail(MCP_ERR_CUDA, "K1Z: cannot raise the dynamic shared-memory limit");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)z.G);
  cfg.blockDim = dim3(K1Z_T);
  cfg.dynamicSmemBytes = z.smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;   // every CTA resident: the grid barrier is safe
  attr[0].val.cooperative = MCP_CFG_K1Z_COOP;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = z.pdl ? 2 : 1;
  auto* ev = timing_begin(c, s);
  cudaError_t e = cudaLaunchKernelEx(&cfg, fn, prm);
  timing_end(ev, s);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    return c->fail(MCP_ERR_CUDA, std::string("K1Z launch failed: ") + cudaGetErrorString(e));
  }
  c->last_launches = 1;
  c->variant = z.name;
  return MCP_OK;
}

int enqueue_fg_full(mcp_ctx* c, const EvalPlan& pl, const double* dx, const double* alpha_dev,
                    double alpha, double* dout, cudaStream_t s) {
  const int r = pl.r;
  if (pl.mode == MCP_MODE_FP64 && pl.z.on)
    return enqueue_fg_small(c, pl, dx, alpha_dev, alpha, dout, s);
  if (pl.mode != MCP_MODE_FP64 || !k1_fuses_tail(pl.k1, c->n, r) || !c->opt_fused_tail) {
    int rc = enqueue_partial(c, pl, dx, (double*)c->dYw.p, s);
    if (rc) return rc;
    return enqueue_finish(c, pl.d, r, dx, (const double*)c->dYw.p, alpha_dev, alpha, dout, s);
  }
  const K1Variant& v = pl.k1;
  const int n = (int)c->n;
  auto* ev = timing_begin(c, s);
  // the tail pieces (G, C, M, u) are formed by K3F itself, overlapping K1's drain
  int rc = k1_launch(v, c->dV, c->ldv, n, c->dnu, c->nu_const, dx + r, r, nullptr, pl.d,
                     (double*)c->dYpart.p, (double*)c->dwpart.p, s);
  timing_end(ev, s);
  if (rc) {
    const cudaError_t e = cudaGetLastError();
    return c->fail(MCP_ERR_CUDA, std::string("K1 launch failed (") + v.name + "): " +
                                     cudaGetErrorString(e));
  }
  const int64_t red_blocks = (int64_t)v.rbs * ceil_div((int64_t)n * v.RB, K3_X) + 1;
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)std::min<int64_t>(red_blocks, 16 * c->sms));
    cfg.blockDim = dim3(K3_T);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CUDA_TRY(c, cudaLaunchKernelEx(&cfg, k_reduce_finish, (const double*)c->dYpart.p,
                                   (const double*)c->dwpart.p, n, r, v.n_pad, v.RB, v.rbs, v.gp,
                                   dx, pl.d,
                                   alpha_dev, alpha, dout));
  }
  CUDA_TRY(c, cudaGetLastError());
  c->last_launches = 2;
  c->variant = v.name;
  return MCP_OK;
}

// Host entry: x (r + n r doubles) + alpha -> out (1 + r + n r doubles), through a cached graph.
int run_host_eval(mcp_ctx* c, int d, int r, int mode, const double* lam, const double* A,
                  double alpha) {
  EvalPlan pl;
  int rc = plan_eval(c, d, r, mode, pl);
  if (rc) return rc;
  const int64_t n = c->n;
  const size_t xin = sizeof(double) * (r + n * r + 1);
  const size_t xout = sizeof(double) * (1 + r + n * r);
  if ((rc = ensure_host(c, c->hx, c->hx_bytes, xin))) return rc;
  if ((rc = ensure_host(c, c->hout, c->hout_bytes, xout))) return rc;
  double* hx = (double*)c->hx;
  // copy into the pinned staging, checking finiteness on the way (objective.py:45-47)
  bool finite = true;
  for (int j = 0; j < r; ++j) {
    hx[j] = lam[j];
    finite &= std::isfinite(lam[j]);
  }
  for (int64_t e = 0; e < n * r; ++e) {
    hx[r + e] = A[e];
    finite &= std::isfinite(A[e]);
  }
  if (!finite) return c->fail(MCP_ERR_ARG, "model variables and alpha must be finite");
  hx[r + n * r] = alpha;

  auto key = std::make_tuple(d, r, mode);
  auto it = c->graphs.find(key);
  if (it == c->graphs.end()) {
    GraphEntry ge;
    CUDA_TRY(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    double* dx = (double*)c->dx.p;
    int rc2;
    if (MCP_CFG_HOST_MEMCPY) {
      cudaMemcpyAsync(dx, hx, xin, cudaMemcpyHostToDevice, c->stream);
      rc2 = enqueue_fg_full(c, pl, dx, dx + r + n * r, 0.0, (double*)c->dout.p, c->stream);
      cudaMemcpyAsync(c->hout, c->dout.p, xout, cudaMemcpyDeviceToHost, c->stream);
    } else {
      // zero-copy staging (pinned memory is device-mapped under UVA): one small kernel pulls x
      // over PCIe and the finishing kernel stores [f ; g] straight into host memory -- no copy
      // engine round trips in the per-evaluation latency
      const int64_t nx = r + n * r + 1;
      k_copy_f64<<<grid_for(nx, 256, 8), 256, 0, c->stream>>>(hx, dx, nx);
      rc2 = enqueue_fg_full(c, pl, dx, dx + r + n * r, 0.0, (double*)c->hout, c->stream);
    }
    cudaError_t ce = cudaStreamEndCapture(c->stream, &ge.graph);
    if (rc2) {
      if (ge.graph) cudaGraphDestroy(ge.graph);
      return rc2;
    }
    CUDA_TRY(c, ce);
    CUDA_TRY(c, cudaGraphInstantiate(&ge.exec, ge.graph, 0));
    it = c->graphs.emplace(key, ge).first;
  } else if (pl.mode == MCP_MODE_FP64 && pl.z.on) {
    c->last_launches = 1;
    c->variant = pl.z.name;
  } else {
    c->last_launches =
        (pl.mode == MCP_MODE_FP64 && k1_fuses_tail(pl.k1, c->n, r) && c->opt_fused_tail)
            ? 2
            : (pl.mode == MCP_MODE_TF32X3 ? 4 : (pl.k1.needs_prep() ? 3 : 2)) +
                  (k4s_fits(n, r) ? 1 : 3);
    c->variant = pl.k1.name;
  }
  CUDA_TRY(c, cudaGraphLaunch(it->second.exec, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return MCP_OK;  // results in c->hout = [f ; g_lam ; vec_F(g_A)]
}

template <typename T>
int upload_obs(mcp_ctx* c, const T* V, bool on_device, int layout, int64_t n, int64_t p,
               int64_t ld) {
  const int64_t ldv = obs_pitch(sizeof(T) == 8 ? MCP_F64 : MCP_F32, n);
  // rows padded with zeros to a multiple of 3584 = lcm(K1 tile 64, K1S copy unit 14 x 16, K1T 128)
  const int64_t p_pad = round_up(p, (int64_t)3584);  // also a multiple of the K1T 128-row tile
  const size_t bytes = sizeof(T) * (size_t)p_pad * ldv;
  if (c->dV) cudaFree(c->dV);
  c->dV = nullptr;
  c->loaded = false;
  CUDA_TRY(c, cudaMalloc(&c->dV, bytes));
  CUDA_TRY(c, cudaMemsetAsync(c->dV, 0, bytes, c->stream));
  if (layout == MCP_OBS_MAJOR) {
    CUDA_TRY(c, cudaMemcpy2DAsync(c->dV, sizeof(T) * ldv, V, sizeof(T) * ld, sizeof(T) * n, p,
                                  on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                  c->stream));
  } else {
    const T* src = V;
    void* staging = nullptr;
    if (!on_device) {
      CUDA_TRY(c, cudaMalloc(&staging, sizeof(T) * (size_t)n * ld));
      CUDA_TRY(c, cudaMemcpyAsync(staging, V, sizeof(T) * (size_t)n * ld, cudaMemcpyHostToDevice,
                                  c->stream));
      src = (const T*)staging;
    }
    dim3 grid((unsigned)ceil_div(p, 32), (unsigned)ceil_div(n, 32));
    k_transpose_in<T><<<grid, dim3(32, 8), 0, c->stream>>>(src, n, p, ld, (T*)c->dV, ldv);
    cudaError_t e = cudaGetLastError();
    if (staging) {
      cudaStreamSynchronize(c->stream);
      cudaFree(staging);
    }
    CUDA_TRY(c, e);
  }
  // finiteness of V (dense.py:87-88)
  int rc = ensure(c, c->dflag, sizeof(unsigned long long));
  if (rc) return rc;
  CUDA_TRY(c, cudaMemsetAsync(c->dflag.p, 0, sizeof(unsigned long long), c->stream));
  k_count_nonfinite<T><<<grid_for(p_pad * ldv, 256, 16 * c->sms), 256, 0, c->stream>>>(
      (const T*)c->dV, p_pad * ldv, (unsigned long long*)c->dflag.p);
  unsigned long long bad = 0;
  CUDA_TRY(c, cudaMemcpyAsync(&bad, c->dflag.p, sizeof(bad), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (bad) {
    cudaFree(c->dV);
    c->dV = nullptr;
    return c->fail(MCP_ERR_ARG, "V contains non-finite entries");
  }
  c->ldv = ldv;
  c->p_pad = p_pad;
  return MCP_OK;
}

int load_nu(mcp_ctx* c, const double* nu, bool on_device, double nu_const) {
  if (c->dnu) cudaFree(c->dnu);
  c->dnu = nullptr;
  if (!nu) {
    c->nu_const = nu_const > 0.0 ? nu_const : 1.0 / (double)c->p;
    if (!std::isfinite(c->nu_const) || !(c->nu_const > 0.0))
      return c->fail(MCP_ERR_ARG, "nu entries must be finite and strictly positive");
    return MCP_OK;
  }
  c->nu_const = 0.0;
  CUDA_TRY(c, cudaMalloc(&c->dnu, sizeof(double) * c->p_pad));
  CUDA_TRY(c, cudaMemsetAsync(c->dnu, 0, sizeof(double) * c->p_pad, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(c->dnu, nu, sizeof(double) * c->p,
                              on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                              c->stream));
  int rc = ensure(c, c->dflag, sizeof(unsigned long long));
  if (rc) return rc;
  CUDA_TRY(c, cudaMemsetAsync(c->dflag.p, 0, sizeof(unsigned long long), c->stream));
  k_check_nu<<<grid_for(c->p, 256, 4 * c->sms), 256, 0, c->stream>>>(
      c->dnu, c->p, (unsigned long long*)c->dflag.p);
  unsigned long long bad = 0;
  CUDA_TRY(c, cudaMemcpyAsync(&bad, c->dflag.p, sizeof(bad), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (bad) return c->fail(MCP_ERR_ARG, "nu entries must be finite and strictly positive");
  return MCP_OK;
}

int load_obs_impl(mcp_ctx* c, const void* V, bool on_device, int dtype, int layout, int64_t n,
                  int64_t p, int64_t ld, const double* nu, double nu_const) {
  if (!V) return c->fail(MCP_ERR_ARG, "V is NULL");
  if (dtype != MCP_F64 && dtype != MCP_F32) return c->fail(MCP_ERR_ARG, "unknown dtype");
  if (layout != MCP_VAR_MAJOR && layout != MCP_OBS_MAJOR)
    return c->fail(MCP_ERR_ARG, "unknown layout");
  if (n < 1 || p < 1)
    return c->fail(MCP_ERR_ARG, "V must be at least 1x1, got shape (" + std::to_string(n) + ", " +
                                    std::to_string(p) + ")");
  const int64_t minld = layout == MCP_OBS_MAJOR ? n : p;
  if (ld < minld) return c->fail(MCP_ERR_ARG, "leading dimension too small");
  c->loaded = false;
  if (on_device) {
    // V / nu in device memory were produced on the caller's streams (e.g. torch's), which this
    // context's non-blocking stream does not order against: wait for all of them first.
    CUDA_TRY(c, cudaDeviceSynchronize());
  }
  drop_graphs(c);
  if (c->own_v32 && c->dV32) cudaFree(c->dV32);
  c->dV32 = nullptr;
  if (c->dVlo32) cudaFree(c->dVlo32);
  c->dVlo32 = nullptr;
  c->own_v32 = false;
  c->tm_v_ready = false;
  c->tm_c_ready = false;
  c->tm_l3_ready = false;
  c->tm_w_kind = 0;
  int rc = dtype == MCP_F64
               ? upload_obs<double>(c, (const double*)V, on_device, layout, n, p, ld)
               : upload_obs<float>(c, (const float*)V, on_device, layout, n, p, ld);
  if (rc) return rc;
  c->dtype = dtype;
  c->n = n;
  c->p = p;
  if ((rc = load_nu(c, nu, on_device, nu_const))) return rc;
  c->loaded = true;
  return MCP_OK;
}

// Everything a context owns except V, nu and the stream (shared with views).
void release_ctx(mcp_ctx* c) {
  drop_graphs(c);
  DevBuf* bufs[] = {&c->dx, &c->dout, &c->dYw, &c->dAfrag, &c->dYpart, &c->dwpart,
                    &c->dG, &c->dC, &c->dpart, &c->dscalar, &c->dflag, &c->dAt,
                    &c->dticket, &c->dzbar};
  for (DevBuf* b : bufs)
    if (b->p) cudaFree(b->p);
  if (c->own_v32 && c->dV32) cudaFree(c->dV32);
  c->dV32 = nullptr;
  if (c->dVlo32) cudaFree(c->dVlo32);
  c->dVlo32 = nullptr;
  if (c->hx) cudaFreeHost(c->hx);
  if (c->hout) cudaFreeHost(c->hout);
  c->hx = c->hout = nullptr;
  for (auto* v : {&c->timed, &c->event_pool})
    for (auto& ev : *v) {
      cudaEventDestroy(ev.first);
      cudaEventDestroy(ev.second);
    }
  c->timed.clear();
  c->event_pool.clear();
}

mcp_ctx* make_view_ctx(const mcp_ctx* parent, void* dV, int dtype, int64_t p, int64_t ldv) {
  mcp_ctx* v = new mcp_ctx();
  v->device = parent->device;
  v->sms = parent->sms;
  v->stream = parent->stream;
  v->dtype = dtype;
  v->n = parent->n;
  v->p = p;
  v->p_pad = round_up(p, 896);  // lcm of the K1 (64), K1S (224) and K1T (128) row units
  v->ldv = ldv;
  v->dV = dV;
  v->dnu = nullptr;
  v->nu_const = 1.0 / (double)p;
  v->opt_fused_tail = parent->opt_fused_tail;
  v->opt_small_kernel = parent->opt_small_kernel;
  v->loaded = true;
  return v;
}

void destroy_view_ctx(mcp_ctx* v) {
  if (!v) return;
  release_ctx(v);
  delete v;
}

}  // namespace mcp_internal

using namespace mcp_internal;

extern "C" {

int mcp_abi_version(void) { return MCP_ABI_VERSION; }

const char* mcp_last_error(const mcp_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_create_error.c_str();
}

int mcp_create(mcp_ctx** out, int device) {
  if (!out) {
    g_create_error = "out is NULL";
    return MCP_ERR_ARG;
  }
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    g_create_error = std::string("no CUDA device available: ") + cudaGetErrorString(e);
    (void)cudaGetLastError();
    return MCP_ERR_CUDA;
  }
  if (device < 0 || device >= count) {
    g_create_error = "device index out of range";
    return MCP_ERR_ARG;
  }
  cudaDeviceProp prop;
  if ((e = cudaSetDevice(device)) != cudaSuccess ||
      (e = cudaGetDeviceProperties(&prop, device)) != cudaSuccess) {
    g_create_error = cudaGetErrorString(e);
    return MCP_ERR_CUDA;
  }
  if (prop.major != 10 || prop.minor != 0) {
    g_create_error = std::string("device ") + prop.name + " is not sm_100 (B200); this build targets sm_100a only";
    return MCP_ERR_CUDA;
  }
  mcp_ctx* c = new mcp_ctx();
  c->device = device;
  c->sms = prop.multiProcessorCount;
  if ((e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking)) != cudaSuccess) {
    g_create_error = cudaGetErrorString(e);
    delete c;
    return MCP_ERR_CUDA;
  }
  *out = c;
  return MCP_OK;
}

int mcp_destroy(mcp_ctx* c) {
  if (!c) return MCP_OK;
  {
    Guard gd(c);
    cudaStreamSynchronize(c->stream);
    release_ctx(c);
    if (c->dV) cudaFree(c->dV);
    if (c->dnu) cudaFree(c->dnu);
    cudaStreamDestroy(c->stream);
  }
  delete c;
  return MCP_OK;
}

int mcp_device_sms(const mcp_ctx* c) { return c ? c->sms : 0; }

int mcp_load_obs(mcp_ctx* c, const void* V, int dtype, int layout, int64_t n, int64_t p,
                 int64_t ld, const double* nu, double nu_const) {
  if (!c) return MCP_ERR_ARG;
  Guard gd(c);
  MCP_NVTX("mcp_load_obs");
  return load_obs_impl(c, V, false, dtype, layout, n, p, ld, nu, nu_const);
}

int mcp_load_obs_device(mcp_ctx* c, const void* dV, int dtype, int layout, int64_t n, int64_t p,
                        int64_t ld, const double* dnu, double nu_const) {
  if (!c) return MCP_ERR_ARG;
  Guard gd(c);
  MCP_NVTX("mcp_load_obs_device");
  return load_obs_impl(c, dV, true, dtype, layout, n, p, ld, dnu, nu_const);
}

int mcp_obs_shape(const mcp_ctx* c, int64_t* n, int64_t* p) {
  if (!c || !c->loaded) return MCP_ERR_STATE;
  if (n) *n = c->n;
  if (p) *p = c->p;
  return MCP_OK;
}


int mcp_fg(mcp_ctx* c, int d, int r, const double* lam, const double* A, double alpha, int mode,
           double* f, double* g_lam, double* g_A) {
  if (!c) return MCP_ERR_ARG;
  Guard gd(c);
  MCP_NVTX("mcp_fg");
  if (!lam || !A || !f || !g_lam || !g_A) return c->fail(MCP_ERR_ARG, "NULL argument");
  if (!std::isfinite(alpha))
    return c->fail(MCP_ERR_ARG, "model variables and alpha must be finite");
  int rc = run_host_eval(c, d, r, mode, lam, A, alpha);
  if (rc) return rc;
  const double* out = (const double*)c->hout;
  *f = out[0];
  std::memcpy(g_lam, out + 1, sizeof(double) * r);
  std::memcpy(g_A, out + 1 + r, sizeof(double) * (size_t)c->n * r);
  return MCP_OK;
}

int mcp_fg_packed(mcp_ctx* c, int d, int r, const double* x, double alpha, int mode, double* f,
                  double* g) {
  if (!c) return MCP_ERR_ARG;
  Guard gd(c);
  MCP_NVTX("mcp_fg_packed");
  if (!x || !f || !g) return c->fail(MCP_ERR_ARG, "NULL argument");
  if (!std::isfinite(alpha))
    return c->fail(MCP_ERR_ARG, "model variables and alpha must be finite");
  if (!c->loaded) return c->fail(MCP_ERR_STATE, "no observation set loaded (call mcp_load_obs)");
  int rc = run_host_eval(c, d, r, mode, x, x + r, alpha);
  if (rc) return rc;
  const double* out = (const double*)c->hout;
  *f = out[0];
  std::memcpy(g, out + 1, sizeof(double) * (r + (size_t)c->n * r));
  return MCP_OK;
}

int mcp_ttsv_batch(mcp_ctx* c, int d, int r, const double* A, int mode, double* Y) {
  if (!c) return MCP_ERR_ARG;
  Guard gd(c);
  MCP_NVTX("mcp_ttsv_batch");
  if (!A || !Y) return c->fail(MCP_ERR_ARG, "NULL argument");
  EvalPlan pl;
  int rc = plan_eval(c, d, r, mode, pl);
  if (rc) return rc;
  const int64_t n = c->n;
  double* dx = (double*)c->dx.p;
  // dx = [lam ; A]; lam is unused by the partial, leave it as is
  CUDA_TRY(c, cudaMemcpyAsync(dx + r, A, sizeof(double) * n * r, cudaMemcpyHostToDevice, c->stream));
  if ((rc = enqueue_partial(c, pl, dx, (double*)c->dYw.p, c->stream))) return rc;
  CUDA_TRY(c, cudaMemcpyAsync(Y, c->dYw.p, sizeof(double) * n * r, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return MCP_OK;
}

// ||X||^2 partial sums.  cross == nullptr: tile-pair slice [part / nparts] of the upper triangle
// of this context's own Gram.  cross != nullptr: slice of the TI x TJ rectangle between this
// context's rows (I) and another row shard of the same set (J, device memory in this context's
// layout), every tile counted twice (sharded ||X||^2, distributed.data_norm_sq_sharded).
struct CrossShard {
  const void* dV;
  int64_t p_pad;
  const double* dnu;
  double nu_const;
  int colmajor;   // tile-pair order of the rectangle: 0 row-major (I outer), 1 column-major
};

static int data_norm_part(mcp_ctx* c, int d, int mode, int part, int nparts, const CrossShard* cross,
                          double* out) {
  if (!c->loaded) return c->fail(MCP_ERR_STATE, "no observation set loaded (call mcp_load_obs)");
  if (d < 2) return c->fail(MCP_ERR_ARG, "order must be >= 2, got " + std::to_string(d));
  // ||X||^2 is a one-time constant: both modes run the FP64 DMMA kernel (exact superset of the
  // fast mode's stated 1e-4 tolerance).
  if (mode != MCP_MODE_FP64 && mode != MCP_MODE_TF32X3)
    return c->fail(MCP_ERR_ARG, "unknown mode " + std::to_string(mode));
  if (nparts < 1 || part < 0 || part >= nparts) return c->fail(MCP_ERR_ARG, "bad part/nparts");
  if (!out) return c->fail(MCP_ERR_ARG, "NULL argument");
  if (cross && (!cross->dV || cross->p_pad < 0 || cross->p_pad % K52_T != 0))
    return c->fail(MCP_ERR_ARG, "cross shard must be a padded row block (multiple of 128 rows)");
  // K53 (fp64, TMA ring) / K5 v2 (fp32) on 128 x 128 tiles for n >= 32 and every cross-shard
  // rectangle; the 64 x 64 variant for narrow observations
  const bool big = (c->n >= 32 || cross) && (c->p_pad % K52_T) == 0;
  const bool f64 = c->dtype == MCP_F64;
  const bool k53 = big && f64 && MCP_CFG_K53;
  const int64_t TT = big ? K52_T : K5_T;
  const int64_t T = c->p_pad / TT;
  const int64_t TJ = cross ? cross->p_pad / K52_T : T;
  const int64_t pairs = cross ? T * TJ : T * (T + 1) / 2;
  const int64_t b = pairs * part / nparts, e = pairs * (part + 1) / nparts;
  const int n_chunks = (int)ceil_div(c->n, k53 ? K53_NK : big ? K52_NK : K5_NK);
  const bool k53h = k53 && MCP_CFG_K53_HALF;   // 64-row I halves, two CTAs per SM
  const int k53ti = !k53 ? 128 : !k53h ? 128 : MCP_CFG_K53_TI;   // I-tile rows per CTA
  const size_t smem = k53 ? (k53ti == 32 ? k53_smem_bytes<32>()
                             : k53ti == 64 ? k53_smem_bytes<64>() : k53_smem_bytes<128>())
                          : big ? (f64 ? k52_smem_bytes<double>() : k52_smem_bytes<float>())
                                : (f64 ? k5_smem_bytes<double>() : k5_smem_bytes<float>());
  const void* fn = k53 ? (k53ti == 32 ? (const void*)k53_gram_power<32>
                         : k53ti == 64 ? (const void*)k53_gram_power<64> : (const void*)k53_gram_power<128>)
                       : big ? (f64 ? (const void*)k52_gram_power<double> : (const void*)k52_gram_power<float>)
                             : (f64 ? (const void*)k5_gram_power<double> : (const void*)k5_gram_power<float>);
  const int threads = k53 ? 4 * k53ti
                          : big ? K52_THREADS : K5_THREADS;
  if (!ensure_dyn_smem(fn, smem))
    return c->fail(MCP_ERR_CUDA, "cannot raise the Gram-power kernel's shared-memory limit");
  int occ = 1;
  CUDA_TRY(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem));
  if (occ < 1) occ = 1;
  int64_t grid = (int64_t)c->sms * occ;
  const int64_t work_units = (e - b) * (k53 ? 128 / k53ti : 1);
  if (grid > work_units) grid = work_units;
  if (grid < 1) grid = 1;
  int rc;
  if ((rc = ensure(c, c->dpart, sizeof(double) * grid))) return rc;
  if ((rc = ensure(c, c->dscalar, sizeof(double)))) return rc;
  CUtensorMap tmI, tmJ;
  if (k53) {
    if (!make_tmap_f64(&tmI, c->dV, c->ldv, c->p_pad, 8 * c->ldv, K53_NK, (uint32_t)k53ti) ||
        !make_tmap_f64(&tmJ, cross ? cross->dV : c->dV, c->ldv, cross ? cross->p_pad : c->p_pad,
                       8 * c->ldv, K53_NK, K53_T))
      return c->fail(MCP_ERR_CUDA, "cuTensorMapEncodeTiled failed for the Gram-power tiles");
  }
  auto* ev = timing_begin(c, c->stream);
  MCP_NVTX("K5 Gram power");
  if (k53) {
    (k53ti == 32 ? k53_gram_power<32> : k53ti == 64 ? k53_gram_power<64> : k53_gram_power<128>)<<<(int)grid, threads, smem, c->stream>>>(
        tmI, tmJ, n_chunks, c->dnu, c->nu_const, cross ? cross->dnu : nullptr,
        cross ? cross->nu_const : 0.0, d, T, TJ, cross ? 1 : 0, cross ? cross->colmajor : 0, b, e,
        (double*)c->dpart.p);
  } else if (big && f64) {
    K52Cross<double> cr;
    if (cross) {
      cr.VJ = (const double*)cross->dV;
      cr.nuJ = cross->dnu;
      cr.nu_constJ = cross->nu_const;
      cr.TJ = TJ;
      cr.colmajor = cross->colmajor;
    }
    k52_gram_power<double><<<(int)grid, threads, smem, c->stream>>>(
        (const double*)c->dV, c->ldv, n_chunks, c->dnu, c->nu_const, d, T, b, e,
        (double*)c->dpart.p, cr);
  } else if (big) {
    K52Cross<float> cr;
    if (cross) {
      cr.VJ = (const float*)cross->dV;
      cr.nuJ = cross->dnu;
      cr.nu_constJ = cross->nu_const;
      cr.TJ = TJ;
      cr.colmajor = cross->colmajor;
    }
    k52_gram_power<float><<<(int)grid, threads, smem, c->stream>>>(
        (const float*)c->dV, c->ldv, n_chunks, c->dnu, c->nu_const, d, T, b, e,
        (double*)c->dpart.p, cr);
  } else if (f64) {
    k5_gram_power<double><<<(int)grid, threads, smem, c->stream>>>(
        (const double*)c->dV, c->ldv, n_chunks, c->dnu, c->nu_const, d, T, b, e,
        (double*)c->dpart.p);
  } else {
    k5_gram_power<float><<<(int)grid, threads, smem, c->stream>>>(
        (const float*)c->dV, c->ldv, n_chunks, c->dnu, c->nu_const, d, T, b, e,
        (double*)c->dpart.p);
  }
  timing_end(ev, c->stream);
  k_ordered_sum<<<1, 32, 0, c->stream>>>((const double*)c->dpart.p, (int)grid,
                                         (double*)c->dscalar.p);
  CUDA_TRY(c, cudaGetLastError());
  CUDA_TRY(c, cudaMemcpyAsync(out, c->dscalar.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  c->last_launches = 2;
  c->variant = std::string(k53 ? "k53_gram_dmma" + std::to_string(k53ti) + "x128_tma" : big ? "k52_gram_dmma128" : "k5_gram_dmma64") +
               (f64 ? "<f64>" : "<f32>") +
               (cross ? "[cross]" : "");
  return MCP_OK;
}

int mcp_data_norm_sq(mcp_ctx* c, int d, int mode, double* out) {
  if (!c) return MCP_ERR_ARG;
  Guard gd(c);
  MCP_NVTX("mcp_data_norm_sq");
  return data_norm_part(c, d, mode, 0, 1, nullptr, out);
}

int mcp_data_norm_sq_part(mcp_ctx* c, int d, int mode, int part, int nparts, double* out) {
  if (!c) return MCP_ERR_ARG;
  Guard gd(c);
  MCP_NVTX("mcp_data_norm_sq_part");
  return data_norm_part(c, d, mode, part, nparts, nullptr, out);
}

int mcp_data_norm_sq_cross(mcp_ctx* c, const void* dVJ, int64_t p_pad_J, const double* dnuJ,
                           double nu_const_J, int d, int mode, int pair_order, int part, int nparts,
                           double* out) {
  if (!c) return MCP_ERR_ARG;
  Guard gd(c);
  MCP_NVTX("mcp_data_norm_sq_cross");
  if (pair_order != 0 && pair_order != 1) return c->fail(MCP_ERR_ARG, "pair_order must be 0 or 1");
  CrossShard cs{dVJ, p_pad_J, dnuJ, nu_const_J, pair_order};
  return data_norm_part(c, d, mode, part, nparts, &cs, out);
}

int mcp_obs_device_view(const mcp_ctx* c, void** dV, int64_t* ldv, int64_t* p_pad, int* dtype,
                        const double** dnu, double* nu_const) {
  if (!c || !c->loaded) return MCP_ERR_STATE;
  if (dV) *dV = c->dV;
  if (ldv) *ldv = c->ldv;
  if (p_pad) *p_pad = c->p_pad;
  if (dtype) *dtype = c->dtype;
  if (dnu) *dnu = c->dnu;
  if (nu_const) *nu_const = c->nu_const;
  return MCP_OK;
}

int mcp_fg_partial_device(mcp_ctx* c, int d, int r, const double* dx, int mode, double* dYw,
                          void* stream) {
  if (!c) return MCP_ERR_ARG;
  Guard gd(c);
  MCP_NVTX("mcp_fg_partial_device");
  if (!dx || !dYw) return c->fail(MCP_ERR_ARG, "NULL argument");
  EvalPlan pl;
  int rc = plan_eval(c, d, r, mode, pl);
  if (rc) return rc;
  cudaStream_t s = stream ? (cudaStream_t)stream : c->stream;
  return enqueue_partial(c, pl, dx, dYw, s);
}

int mcp_fg_partial_signal_device(mcp_ctx* c, int d, int r, const double* dx, int mode,
                                 double* dYw, const void* flag_ptrs, int rank, int world,
                                 int64_t epoch, void* stream) {
  if (!c) return MCP_ERR_ARG;
  Guard gd(c);
  MCP_NVTX("mcp_fg_partial_signal_device");
  if (!dx || !dYw || !flag_ptrs) return c->fail(MCP_ERR_ARG, "NULL argument");
  if (world < 1 || rank < 0 || rank >= world) return c->fail(MCP_ERR_ARG, "bad peer arguments");
  EvalPlan pl;
  int rc = plan_eval(c, d, r, mode, pl);
  if (rc) return rc;
  cudaStream_t s = stream ? (cudaStream_t)stream : c->stream;
  K3Signal sig;
  sig.flags = (int64_t* const*)flag_ptrs;
  sig.rank = rank;
  sig.world = world;
  sig.epoch = epoch;
  return enqueue_partial(c, pl, dx, dYw, s, &sig);
}

int mcp_fg_finish_device(mcp_ctx* c, int d, int r, const double* dx, const double* dYw,
                         double alpha, double* dout, void* stream) {
  if (!c) return MCP_ERR_ARG;
  Guard gd(c);
  MCP_NVTX("mcp_fg_finish_device");
  if (!dx || !dYw || !dout) return c->fail(MCP_ERR_ARG, "NULL argument");
  if (!c->loaded) return c->fail(MCP_ERR_STATE, "no observation set loaded (call mcp_load_obs)");
  if (d < 2) return c->fail(MCP_ERR_ARG, "order must be >= 2, got " + std::to_string(d));
  if (r < 1) return c->fail(MCP_ERR_ARG, "rank must be >= 1, got " + std::to_string(r));
  int rc;
  if ((rc = ensure(c, c->dG, sizeof(double) * (size_t)r * r))) return rc;
  if ((rc = ensure(c, c->dC, sizeof(double) * (size_t)r * r))) return rc;
  cudaStream_t s = stream ? (cudaStream_t)stream : c->stream;
  c->last_launches = 0;
  return enqueue_finish(c, d, r, dx, dYw, nullptr, alpha, dout, s);
}

int mcp_fg_device(mcp_ctx* c, int d, int r, const double* dx, double alpha, int mode,
                  double* dout, void* stream) {
  if (!c) return MCP_ERR_ARG;
  Guard gd(c);
  MCP_NVTX("mcp_fg_device");
  if (!dx || !dout) return c->fail(MCP_ERR_ARG, "NULL argument");
  EvalPlan pl;
  int rc = plan_eval(c, d, r, mode, pl);
  if (rc) return rc;
  cudaStream_t s = stream ? (cudaStream_t)stream : c->stream;
  return enqueue_fg_full(c, pl, dx, nullptr, alpha, dout, s);
}

int mcp_set_option(mcp_ctx* c, int key, int64_t value) {
  if (!c) return MCP_ERR_ARG;
  Guard gd(c);
  switch (key) {
    case MCP_OPT_FUSED_TAIL:
      if (c->opt_fused_tail != (value != 0)) drop_graphs(c);
      c->opt_fused_tail = value != 0;
      return MCP_OK;
    case MCP_OPT_SMALL_KERNEL:
      if (c->opt_small_kernel != (value != 0)) drop_graphs(c);
      c->opt_small_kernel = value != 0;
      return MCP_OK;
    default:
      return c->fail(MCP_ERR_ARG, "unknown option " + std::to_string(key));
  }
}

int mcp_set_kernel_timing(mcp_ctx* c, int enable) {
  if (!c) return MCP_ERR_ARG;
  Guard gd(c);
  c->timing = enable != 0;
  c->timing_every = enable > 1 ? enable : 1;
  c->timing_seen = 0;
  return MCP_OK;
}

int mcp_kernel_time_ms(mcp_ctx* c, double* total_ms, int* launches, int reset) {
  if (!c) return MCP_ERR_ARG;
  Guard gd(c);
  double tot = 0.0;
  for (auto& ev : c->timed) {
    CUDA_TRY(c, cudaEventSynchronize(ev.second));
    float ms = 0.f;
    CUDA_TRY(c, cudaEventElapsedTime(&ms, ev.first, ev.second));
    tot += ms;
  }
  if (total_ms) *total_ms = tot;
  if (launches) *launches = (int)c->timed.size();
  if (reset) {
    for (auto& ev : c->timed) c->event_pool.push_back(ev);
    c->timed.clear();
  }
  return MCP_OK;
}

int mcp_fg_batch(mcp_ctx* c, int d, int r, int k, const double* X, double alpha, int mode,
                 double* F, double* G) {
  if (!c) return MCP_ERR_ARG;
  Guard gd(c);
  MCP_NVTX("mcp_fg_batch");
  if (!X || !F || !G) return c->fail(MCP_ERR_ARG, "NULL argument");
  if (k < 1) return c->fail(MCP_ERR_ARG, "batch size must be >= 1");
  if (!std::isfinite(alpha))
    return c->fail(MCP_ERR_ARG, "model variables and alpha must be finite");
  if (!c->loaded) return c->fail(MCP_ERR_STATE, "no observation set loaded (call mcp_load_obs)");
  const int64_t n = c->n;
  const int64_t rows = r + n * r;             // one packed start
  const int R = k * r;                        // columns of the shared pass
  EvalPlan pl;
  int rc = plan_eval(c, d, R, mode, pl);
  if (rc) return rc;
  // staging: [lam_all (R) ; A_all (n x R, col-major) ; alpha] for the pass, then the k starts
  const size_t xin = sizeof(double) * ((size_t)R + n * R + 1 + (size_t)k * rows);
  const size_t xout = sizeof(double) * (size_t)k * (1 + rows);
  if ((rc = ensure_host(c, c->hx, c->hx_bytes, xin))) return rc;
  if ((rc = ensure_host(c, c->hout, c->hout_bytes, xout))) return rc;
  if ((rc = ensure(c, c->dx, xin))) return rc;
  if ((rc = ensure(c, c->dout, xout))) return rc;
  double* hx = (double*)c->hx;
  for (int sidx = 0; sidx < k; ++sidx) {
    const double* xs = X + (size_t)sidx * rows;
    std::memcpy(hx + (size_t)sidx * r, xs, sizeof(double) * r);
    std::memcpy(hx + R + (size_t)sidx * n * r, xs + r, sizeof(double) * n * r);
  }
  hx[R + n * R] = alpha;
  std::memcpy(hx + R + n * R + 1, X, sizeof(double) * (size_t)k * rows);
  double* dx = (double*)c->dx.p;
  CUDA_TRY(c, cudaMemcpyAsync(dx, hx, xin, cudaMemcpyHostToDevice, c->stream));
  if ((rc = enqueue_partial(c, pl, dx, (double*)c->dYw.p, c->stream))) return rc;
  const int launches = c->last_launches;
  const double* dY = (const double*)c->dYw.p;
  const double* dW = dY + n * R;
  const double* dXs = dx + R + n * R + 1;
  if (k4s_fits(n, r)) {
    // all k tails in one launch, one CTA per start
    k_tail_fused<<<k, K4S_THREADS, k4s_smem_bytes(n * r), c->stream>>>(dXs, dY, dW, (int)n, r, d, dx + R + n * R, 0.0,
                                                   (double*)c->dout.p, rows, n * r, r, 1 + rows);
    CUDA_TRY(c, cudaGetLastError());
    c->last_launches = 1;
  } else {
    for (int sidx = 0; sidx < k; ++sidx) {
      if ((rc = enqueue_finish_yw(c, d, r, dXs + (size_t)sidx * rows, dY + (size_t)sidx * n * r,
                                  dW + (size_t)sidx * r, dx + R + n * R, 0.0,
                                  (double*)c->dout.p + (size_t)sidx * (1 + rows), c->stream)))
        return rc;
    }
  }
  c->last_launches += launches;
  CUDA_TRY(c, cudaMemcpyAsync(c->hout, c->dout.p, xout, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  const double* out = (const double*)c->hout;
  for (int sidx = 0; sidx < k; ++sidx) {
    F[sidx] = out[(size_t)sidx * (1 + rows)];
    std::memcpy(G + (size_t)sidx * rows, out + (size_t)sidx * (1 + rows) + 1,
                sizeof(double) * rows);
  }
  return MCP_OK;
}

int mcp_last_launch_count(const mcp_ctx* c) { return c ? c->last_launches : 0; }

const char* mcp_last_variant(const mcp_ctx* c) { return c ? c->variant.c_str() : ""; }

}  // extern "C"
