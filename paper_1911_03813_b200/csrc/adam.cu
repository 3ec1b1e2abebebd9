// Stochastic path on the device: row sampling + epoch-based Adam.
//
// Reference: sample_observations (pkg/src/momentcp/objective.py:97-113) and adam_minimize
// (pkg/src/momentcp/optimize.py:365-451).
//
// The observation set stays resident; a mini-batch is a gather of `batch` rows of V into a
// small zero-padded buffer that a view context (ctx.h make_view_ctx, uniform weights 1/batch)
// evaluates with the same K1 -> K3 -> K4 chain as a full evaluation.  One Adam iteration is
//     gather(idx[it]) -> fg(batch view, x) -> adam update of x, m1, m2 (it += 1)
// captured once as a CUDA graph and replayed epoch_len times per epoch without host syncs; the
// epoch's indices (drawn by the caller's numpy Generator exactly as the reference draws them)
// and bias corrections 1 - beta^t (host pow, as in the reference) are uploaded per epoch.  The
// function estimate on the fixed estimate subset is one more graph; the host reads back only f.
// The update uses explicit round-to-nearest operations in the reference's evaluation order, so
// given the same gradient it reproduces numpy's m1, m2 and x bit for bit.
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "ctx.h"
#include "mcp_common.cuh"
#include "pdl.h"
#include "k1z_small.cuh"

using namespace mcp;
using namespace mcp_internal;

namespace {

constexpr int AD_T = 256;

// rows idx[it * batch + l] of the resident set -> row l of the batch buffer (pitch ldo)
template <typename Tin, typename Tout>
__global__ void k_gather_rows(const Tin* __restrict__ V, int64_t ldv, int64_t n,
                              const int64_t* __restrict__ idx, const int* __restrict__ it_dev,
                              int64_t batch, Tout* __restrict__ out, int64_t ldo) {
  const int64_t base = it_dev ? (int64_t)(*it_dev) * batch : 0;
  for (int64_t l = blockIdx.y; l < batch; l += gridDim.y) {
    const Tin* src = V + idx[base + l] * ldv;
    Tout* dst = out + l * ldo;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
      dst[i] = (Tout)src[i];
  }
}

struct AdamScalars {
  double lr, b1, omb1, b2, omb2, eps;
};

// m1 = b1 m1 + (1-b1) g ; m2 = b2 m2 + ((1-b2) g) g ; x -= (lr (m1/bc1)) / (sqrt(m2/bc2) + eps)
// (optimize.py:425-430).  bc[2 it], bc[2 it + 1] = 1 - b1^t, 1 - b2^t.  The last block advances
// the iteration counter.
__global__ void k_adam_step(int64_t N, const double* __restrict__ out, double* __restrict__ x,
                            double* __restrict__ m1, double* __restrict__ m2,
                            const double* __restrict__ bc, const double* __restrict__ lr_dev,
                            AdamScalars sc, int* __restrict__ it_dev, unsigned* counter) {
  pdl_enter();   // the gradient comes from the preceding finish kernel
  const int it = *it_dev;
  const double bc1 = bc[2 * it], bc2 = bc[2 * it + 1];
  const double lr = *lr_dev;
  const double* g = out + 1;
  for (int64_t j = blockIdx.x * (int64_t)AD_T + threadIdx.x; j < N;
       j += (int64_t)gridDim.x * AD_T) {
    const double gj = g[j];
    const double a = __dadd_rn(__dmul_rn(sc.b1, m1[j]), __dmul_rn(sc.omb1, gj));
    const double b = __dadd_rn(__dmul_rn(sc.b2, m2[j]), __dmul_rn(__dmul_rn(sc.omb2, gj), gj));
    m1[j] = a;
    m2[j] = b;
    const double mh = __ddiv_rn(a, bc1);
    const double vh = __ddiv_rn(b, bc2);
    x[j] = __dsub_rn(x[j], __ddiv_rn(__dmul_rn(lr, mh), __dadd_rn(__dsqrt_rn(vh), sc.eps)));
  }
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
    if (last) {
      *counter = 0u;
      *it_dev = it + 1;
    }
  }
}

struct AdamRun {
  mcp_ctx* c = nullptr;
  mcp_ctx* vb = nullptr;   // batch view
  mcp_ctx* ve = nullptr;   // estimate view
  int d = 0, r = 0, mode = 0;
  int64_t N = 0, batch = 0, epoch_len = 0, n_est = 0;
  int nb = 1;
  EvalPlan plb, ple;
  std::vector<void*> dev;
  void *Vb = nullptr, *Ve = nullptr;
  double *X = nullptr, *XB = nullptr, *M1 = nullptr, *M2 = nullptr, *OB = nullptr, *OE = nullptr;
  double *bc = nullptr, *lr_dev = nullptr;
  int64_t *idx = nullptr, *eidx = nullptr;
  int* it_dev = nullptr;
  unsigned* counter = nullptr;
  int64_t* h_idx = nullptr;    // two staging halves: the running epoch and the one sampled ahead
  int64_t h_idx_half = 0;
  double* h_bc = nullptr;
  double* h_scal = nullptr;  // [lr, f_est]
  K1ZAdam zadam;   // the update fused into K1Z's finish when the batch plans to K1Z
  GraphEntry g_iter, g_chunk, g_est;   // one iteration, ITER_CHUNK iterations, the estimate
  int64_t chunk_iters = 0;
  AdamScalars sc{};

  ~AdamRun() {
    for (GraphEntry* g : {&g_iter, &g_chunk, &g_est}) {
      if (g->exec) cudaGraphExecDestroy(g->exec);
      if (g->graph) cudaGraphDestroy(g->graph);
    }
    destroy_view_ctx(vb);
    destroy_view_ctx(ve);
    for (void* p : dev) cudaFree(p);
    if (h_idx) cudaFreeHost(h_idx);
    if (h_bc) cudaFreeHost(h_bc);
    if (h_scal) cudaFreeHost(h_scal);
  }

  template <typename T>
  int alloc(T*& p, size_t elems) {
    void* q = nullptr;
    CUDA_TRY(c, cudaMalloc(&q, sizeof(T) * (elems ? elems : 1)));
    dev.push_back(q);
    p = (T*)q;
    return MCP_OK;
  }

  // gather view dtype: the set's own, except fp32 rows for tcgen05 fast mode on an fp64 set
  int view_dtype() const { return mode == MCP_MODE_TF32X3 ? MCP_F32 : c->dtype; }

  int enqueue_gather(void* dst, int64_t rows, const int64_t* ix, const int* itp, int64_t ldo) {
    const int64_t n = c->n;
    dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>((n + AD_T - 1) / AD_T, 4)),
              (unsigned)std::min<int64_t>(rows, 4096));
    cudaStream_t s = c->stream;
    if (c->dtype == MCP_F64 && view_dtype() == MCP_F64)
      k_gather_rows<double, double><<<grid, AD_T, 0, s>>>((const double*)c->dV, c->ldv, n, ix,
                                                           itp, rows, (double*)dst, ldo);
    else if (c->dtype == MCP_F64)
      k_gather_rows<double, float><<<grid, AD_T, 0, s>>>((const double*)c->dV, c->ldv, n, ix, itp,
                                                          rows, (float*)dst, ldo);
    else
      k_gather_rows<float, float><<<grid, AD_T, 0, s>>>((const float*)c->dV, c->ldv, n, ix, itp,
                                                         rows, (float*)dst, ldo);
    CUDA_TRY(c, cudaGetLastError());
    return MCP_OK;
  }

  int make_view(mcp_ctx** out, void** buf, int64_t rows) {
    const int dt = view_dtype();
    const int64_t ldo = obs_pitch(dt, c->n);
    const size_t esz = dt == MCP_F64 ? 8 : 4;
    const size_t bytes = esz * (size_t)round_up(rows, (int64_t)896) * ldo;
    void* q = nullptr;
    CUDA_TRY(c, cudaMalloc(&q, bytes));
    dev.push_back(q);
    CUDA_TRY(c, cudaMemset(q, 0, bytes));
    *buf = q;
    *out = make_view_ctx(c, q, dt, rows, ldo);
    return MCP_OK;
  }

  int capture(GraphEntry& ge, const std::function<int()>& body) {
    CUDA_TRY(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    int rc = body();
    cudaError_t ce = cudaStreamEndCapture(c->stream, &ge.graph);
    if (rc) return rc;
    CUDA_TRY(c, ce);
    CUDA_TRY(c, cudaGraphInstantiate(&ge.exec, ge.graph, 0));
    return MCP_OK;
  }

  int fg_on(mcp_ctx* v, const EvalPlan& pl, const double* x, double* out) {
    int rc = enqueue_fg_full(v, pl, x, nullptr, 0.0, out, c->stream);
    if (rc) return c->fail(rc, v->err);
    return MCP_OK;
  }

  bool matches(int d_, int r_, int mode_, int64_t batch_, int64_t epoch_len_, int64_t n_est_,
               const AdamScalars& sc_) const {
    return d == d_ && r == r_ && mode == mode_ && batch == batch_ && epoch_len == epoch_len_ &&
           n_est == n_est_ && c->n == n && std::memcmp(&sc, &sc_, sizeof(sc)) == 0;
  }
  int64_t n = 0;

  int setup() {
    n = c->n;
    N = r + n * r;
    nb = grid_for(N, AD_T, 2 * c->sms);
    int rc;
    if ((rc = make_view(&vb, &Vb, batch)) || (rc = make_view(&ve, &Ve, n_est))) return rc;
    if ((rc = alloc(idx, epoch_len * batch)) || (rc = alloc(it_dev, 1))) return rc;
    if (mode == MCP_MODE_FP64) {
      // K1Z (when the batch plans to it) reads the batch rows in place through the index list
      vb->gV = c->dV;
      vb->gldv = c->ldv;
      vb->gdtype = c->dtype;
      vb->gidx = idx;
      vb->git = it_dev;
    }
    if ((rc = plan_eval(vb, d, r, mode, plb))) return c->fail(rc, vb->err);
    if ((rc = plan_eval(ve, d, r, mode, ple))) return c->fail(rc, ve->err);
    if ((rc = alloc(X, N)) || (rc = alloc(XB, N)) || (rc = alloc(M1, N)) || (rc = alloc(M2, N)) ||
        (rc = alloc(OB, N + 1)) || (rc = alloc(OE, N + 1)) || (rc = alloc(bc, 2 * epoch_len)) ||
        (rc = alloc(lr_dev, 1)) || (rc = alloc(eidx, n_est)) || (rc = alloc(counter, 1)))
      return rc;
    CUDA_TRY(c, cudaMemset(counter, 0, sizeof(unsigned)));
    h_idx_half = std::max(epoch_len * batch, n_est);
    CUDA_TRY(c, cudaMallocHost(&h_idx, sizeof(int64_t) * 2 * h_idx_half));
    CUDA_TRY(c, cudaMallocHost(&h_bc, sizeof(double) * 2 * epoch_len));
    CUDA_TRY(c, cudaMallocHost(&h_scal, sizeof(double) * 4));
    cudaStream_t s = c->stream;
    const bool fused_step = mode == MCP_MODE_FP64 && plb.z.on && MCP_CFG_ADAM_FUSED_STEP;
    if (fused_step) {
      zadam.x = X;
      zadam.m1 = M1;
      zadam.m2 = M2;
      zadam.bc = bc;
      zadam.lr = lr_dev;
      zadam.it = it_dev;
      zadam.b1 = sc.b1;
      zadam.omb1 = sc.omb1;
      zadam.b2 = sc.b2;
      zadam.omb2 = sc.omb2;
      zadam.eps = sc.eps;
      vb->z_adam = &zadam;
    }
    auto one_iteration = [&]() -> int {
      int e = MCP_OK;
      // no gathered copy when the single-launch kernel reads the rows through the index
      if (!(mode == MCP_MODE_FP64 && plb.z.on)) e = enqueue_gather(Vb, batch, idx, it_dev, vb->ldv);
      if (e) return e;
      if ((e = fg_on(vb, plb, X, OB))) return e;
      if (fused_step) return MCP_OK;   // gather, f+grad and the update were one launch
      CUDA_TRY(c, launch_pdl(k_adam_step, dim3(nb), dim3(AD_T), 0, s, N, (const double*)OB, X, M1,
                             M2, (const double*)bc, (const double*)lr_dev, sc, it_dev, counter));
      return MCP_OK;
    };
    if ((rc = capture(g_iter, one_iteration))) return rc;
    // the iteration cursor lives on the device, so iterations are identical graph nodes: an epoch
    // replays a graph of up to ITER_CHUNK iterations (one host launch instead of one per
    // iteration) plus single iterations for the remainder
    chunk_iters = std::min<int64_t>(epoch_len, MCP_CFG_ADAM_ITER_CHUNK);
    if (chunk_iters > 1) {
      if ((rc = capture(g_chunk, [&]() -> int {
             for (int64_t k = 0; k < chunk_iters; ++k) {
               int e = one_iteration();
               if (e) return e;
             }
             return MCP_OK;
           })))
        return rc;
    }
    if ((rc = capture(g_est, [&]() -> int {
           int e = fg_on(ve, ple, X, OE);
           if (e) return e;
           CUDA_TRY(c, cudaMemcpyAsync(h_scal + 1, OE, sizeof(double), cudaMemcpyDeviceToHost, s));
           return MCP_OK;
         })))
      return rc;
    return MCP_OK;
  }

  // the estimate subset of this run, gathered once
  int load_estimate_rows(const int64_t* est_idx) {
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    std::memcpy(h_idx, est_idx, sizeof(int64_t) * n_est);
    CUDA_TRY(c, cudaMemcpyAsync(eidx, h_idx, sizeof(int64_t) * n_est, cudaMemcpyHostToDevice,
                                c->stream));
    int rc = enqueue_gather(Ve, n_est, eidx, nullptr, ve->ldv);
    if (rc) return rc;
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return MCP_OK;
  }

  int estimate(double* f) {
    CUDA_TRY(c, cudaGraphLaunch(g_est.exec, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    *f = h_scal[1];
    return MCP_OK;
  }
};

}  // namespace

extern "C" int mcp_gather_rows(mcp_ctx* c, const int64_t* idx, int64_t s, void* dst,
                               int64_t ld_dst, int dst_dtype) {
  if (!c) return MCP_ERR_ARG;
  Guard gd(c);
  if (!c->loaded) return c->fail(MCP_ERR_STATE, "no observation set loaded (call mcp_load_obs)");
  if (!idx || !dst || s < 1) return c->fail(MCP_ERR_ARG, "sample size must be >= 1");
  if (ld_dst < c->n) return c->fail(MCP_ERR_ARG, "leading dimension too small");
  if (dst_dtype != c->dtype && !(c->dtype == MCP_F64 && dst_dtype == MCP_F32))
    return c->fail(MCP_ERR_ARG, "unsupported destination dtype");
  for (int64_t l = 0; l < s; ++l)
    if (idx[l] < 0 || idx[l] >= c->p) return c->fail(MCP_ERR_ARG, "row index out of range");
  // dst belongs to the caller (e.g. a fresh torch allocation whose memory earlier work on the
  // caller's streams may still touch): order the gather after everything on the device
  CUDA_TRY(c, cudaDeviceSynchronize());
  int64_t* didx = nullptr;
  CUDA_TRY(c, cudaMalloc(&didx, sizeof(int64_t) * s));
  cudaError_t e = cudaMemcpyAsync(didx, idx, sizeof(int64_t) * s, cudaMemcpyHostToDevice,
                                  c->stream);
  if (e == cudaSuccess) {
    dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>((c->n + AD_T - 1) / AD_T, 4)),
              (unsigned)std::min<int64_t>(s, 4096));
    if (c->dtype == MCP_F64 && dst_dtype == MCP_F64)
      k_gather_rows<double, double><<<grid, AD_T, 0, c->stream>>>(
          (const double*)c->dV, c->ldv, c->n, didx, nullptr, s, (double*)dst, ld_dst);
    else if (c->dtype == MCP_F64)
      k_gather_rows<double, float><<<grid, AD_T, 0, c->stream>>>(
          (const double*)c->dV, c->ldv, c->n, didx, nullptr, s, (float*)dst, ld_dst);
    else
      k_gather_rows<float, float><<<grid, AD_T, 0, c->stream>>>(
          (const float*)c->dV, c->ldv, c->n, didx, nullptr, s, (float*)dst, ld_dst);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  }
  cudaFree(didx);
  CUDA_TRY(c, e);
  return MCP_OK;
}

extern "C" int mcp_adam(mcp_ctx* c, int d, int r, int mode, const double* x0, const double* opts,
                        const int64_t* est_idx, int64_t n_est, mcp_sample_fn sample, void* user,
                        double* x_out, double* g_out, double* f_out, double* trace_f,
                        double* trace_t, int64_t trace_cap, int64_t* info) {
  if (!c) return MCP_ERR_ARG;
  Guard gd(c);
  MCP_NVTX("mcp_adam");
  if (!x0 || !opts || !est_idx || !sample || !x_out || !g_out || !f_out || !info)
    return c->fail(MCP_ERR_ARG, "NULL argument");
  if (!c->loaded) return c->fail(MCP_ERR_STATE, "no observation set loaded (call mcp_load_obs)");
  const double step_size = opts[0], reduced = opts[1];
  const int64_t epoch_len = (int64_t)opts[2], batch = (int64_t)opts[3];
  const double beta1 = opts[4], beta2 = opts[5], eps = opts[6];
  const int64_t max_epochs = (int64_t)opts[7];
  if (epoch_len < 1) return c->fail(MCP_ERR_ARG, "epoch_len must be >= 1");
  if (batch < 1) return c->fail(MCP_ERR_ARG, "batch must be >= 1");
  if (n_est < 1) return c->fail(MCP_ERR_ARG, "estimate subset is empty");
  for (int64_t l = 0; l < n_est; ++l)
    if (est_idx[l] < 0 || est_idx[l] >= c->p) return c->fail(MCP_ERR_ARG, "row index out of range");
  const auto t_start = std::chrono::steady_clock::now();
  auto seconds = [&]() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  };
  const AdamScalars sc{step_size, beta1, 1.0 - beta1, beta2, 1.0 - beta2, eps};
  AdamRun* ws = (AdamRun*)c->adam_ws;
  if (!ws || !ws->matches(d, r, mode, batch, epoch_len, n_est, sc)) {
    if (ws) {
      c->adam_ws_free(ws);
      c->adam_ws = nullptr;
    }
    ws = new AdamRun();
    ws->c = c;
    ws->d = d;
    ws->r = r;
    ws->mode = mode;
    ws->batch = batch;
    ws->epoch_len = epoch_len;
    ws->n_est = n_est;
    ws->sc = sc;
    int rc0 = ws->setup();
    if (rc0) {
      delete ws;
      return rc0;
    }
    c->adam_ws = ws;
    c->adam_ws_free = [](void* p) { delete (AdamRun*)p; };
  }
  AdamRun& R = *ws;
  int rc = R.load_estimate_rows(est_idx);
  if (rc) return rc;
  const int64_t N = R.N;
  cudaStream_t s = c->stream;
  CUDA_TRY(c, cudaMemcpyAsync(R.X, x0, sizeof(double) * N, cudaMemcpyHostToDevice, s));
  CUDA_TRY(c, cudaMemsetAsync(R.M1, 0, sizeof(double) * N, s));
  CUDA_TRY(c, cudaMemsetAsync(R.M2, 0, sizeof(double) * N, s));
  double f_best = 0.0;
  if ((rc = R.estimate(&f_best))) return rc;
  CUDA_TRY(c, cudaMemcpyAsync(R.XB, R.X, sizeof(double) * N, cudaMemcpyDeviceToDevice, s));
  int64_t n_trace = 0;
  auto push_trace = [&](double fv) {
    if (n_trace < trace_cap) {
      if (trace_f) trace_f[n_trace] = fv;
      if (trace_t) trace_t[n_trace] = seconds();
    }
    ++n_trace;
  };
  push_trace(f_best);
  double lr = step_size;
  int64_t t = 0, n_iter = 0;
  int increases = 0, reason = 0;
  // one epoch's indices into a staging half, checked (optimize.py:409: rng.integers(0, p, ...))
  auto draw = [&](int64_t* buf) -> int {
    if (sample(buf, epoch_len * batch, user) != 0)
      return c->fail(MCP_ERR_ARG, "sampling callback failed");
    for (int64_t l = 0; l < epoch_len * batch; ++l)
      if (buf[l] < 0 || buf[l] >= c->p) return c->fail(MCP_ERR_ARG, "row index out of range");
    return MCP_OK;
  };
  int cur = 0;
  bool ahead = false;   // the next epoch's indices are already in the other half
  for (int64_t epoch = 0; epoch < max_epochs; ++epoch) {
    int64_t* hb = R.h_idx + (size_t)cur * R.h_idx_half;
    if (!ahead) {
      // (the estimate's synchronisation ended every copy out of this half)
      CUDA_TRY(c, cudaStreamSynchronize(s));
      if ((rc = draw(hb))) return rc;
    }
    for (int64_t k = 0; k < epoch_len; ++k) {
      const double tt = (double)(t + k + 1);
      R.h_bc[2 * k] = 1.0 - std::pow(beta1, tt);
      R.h_bc[2 * k + 1] = 1.0 - std::pow(beta2, tt);
    }
    R.h_scal[0] = lr;
    CUDA_TRY(c, cudaMemcpyAsync(R.idx, hb, sizeof(int64_t) * epoch_len * batch,
                                cudaMemcpyHostToDevice, s));
    CUDA_TRY(c, cudaMemcpyAsync(R.bc, R.h_bc, sizeof(double) * 2 * epoch_len,
                                cudaMemcpyHostToDevice, s));
    CUDA_TRY(c, cudaMemcpyAsync(R.lr_dev, R.h_scal, sizeof(double), cudaMemcpyHostToDevice, s));
    CUDA_TRY(c, cudaMemsetAsync(R.it_dev, 0, sizeof(int), s));
    {
      int64_t k = 0;
      if (R.chunk_iters > 1)
        for (; k + R.chunk_iters <= epoch_len; k += R.chunk_iters)
          CUDA_TRY(c, cudaGraphLaunch(R.g_chunk.exec, s));
      for (; k < epoch_len; ++k) CUDA_TRY(c, cudaGraphLaunch(R.g_iter.exec, s));
    }
    t += epoch_len;
    n_iter += epoch_len;
    // while the GPU runs this epoch, the host draws the next one (the draws do not depend on
    // the epoch's outcome; if the run stops here the caller rewinds its generator: info[3])
    ahead = false;
    if (epoch + 1 < max_epochs) {
      if ((rc = draw(R.h_idx + (size_t)(cur ^ 1) * R.h_idx_half))) return rc;
      ahead = true;
    }
    cur ^= 1;
    double f_est = 0.0;
    if ((rc = R.estimate(&f_est))) return rc;
    push_trace(f_est);
    if (f_est < f_best) {
      f_best = f_est;
      CUDA_TRY(c, cudaMemcpyAsync(R.XB, R.X, sizeof(double) * N, cudaMemcpyDeviceToDevice, s));
    } else {
      ++increases;
      CUDA_TRY(c, cudaMemcpyAsync(R.X, R.XB, sizeof(double) * N, cudaMemcpyDeviceToDevice, s));
      CUDA_TRY(c, cudaMemsetAsync(R.M1, 0, sizeof(double) * N, s));
      CUDA_TRY(c, cudaMemsetAsync(R.M2, 0, sizeof(double) * N, s));
      t = 0;
      if (increases == 1) {
        lr = reduced;
      } else {
        reason = 1;
        break;
      }
    }
  }
  // gradient estimate at the best iterate (optimize.py:441)
  CUDA_TRY(c, cudaMemcpyAsync(R.X, R.XB, sizeof(double) * N, cudaMemcpyDeviceToDevice, s));
  double f_fin = 0.0;
  if ((rc = R.estimate(&f_fin))) return rc;
  CUDA_TRY(c, cudaMemcpyAsync(x_out, R.XB, sizeof(double) * N, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(c, cudaMemcpyAsync(g_out, R.OE + 1, sizeof(double) * N, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(c, cudaStreamSynchronize(s));
  *f_out = f_best;
  info[0] = n_iter;
  info[1] = reason;
  info[2] = std::min(n_trace, trace_cap);
  info[3] = (reason == 1 && ahead) ? 1 : 0;   // epochs drawn ahead and never run
  return MCP_OK;
}
