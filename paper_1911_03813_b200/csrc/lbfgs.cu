// Device-resident L-BFGS over the momentcp objective.
//
// Reference: pkg/src/momentcp/optimize.py:149-168 (two-loop recursion), :171-176 (safeguarded
// quadratic interpolation), :179-252 (strong-Wolfe bracket/zoom), :255-355 (outer loop).
//
// HBM holds x, g = fg(x), the direction p, a trial point xa with its [fa; ga], a saved best
// trial, and a ring of memory+1 (s, y) slots (the spare slot takes the new pair before the
// curvature test decides whether it joins the window, so a rejected pair never evicts the
// oldest accepted one -- the reference's deque only appends accepted pairs).  Per evaluation the
// host replays one CUDA graph
//     [accept step -> two-loop direction -> a0]  ->  trial x + a p  ->  fg  ->  probe scalars
// and reads back ~12 doubles; the line-search and stopping decisions are made on those scalars
// in exactly the reference's order.  Elementwise updates use explicit round-to-nearest multiply
// and add (no FMA contraction), so given equal scalars they match numpy's `x + a * p`,
// `q -= alpha * y`, ... bit for bit; dot products are fixed-order reductions (deterministic run
// to run, but summed in a different order than numpy's).
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "ctx.h"

using namespace mcp_internal;

namespace {

constexpr int LB_T = 256;        // threads of the streaming kernels
constexpr int LB_DIR_T = 1024;   // the single-CTA two-loop kernel
constexpr int LB_NP = 6;         // partial sums per block
constexpr int LB_MAX_BLOCKS = 296;

// scalar slots of the stats record copied to the host after every graph replay
enum {
  S_GMAX = 0,   // max |g| of the accepted gradient (+inf when it has non-finite entries)
  S_GSUM,       // sum |g|
  S_GBAD,       // non-finite entries in g (init: also in x0)
  S_KEEP,       // 1 when the (s, y) pair passed the curvature test
  S_PG,         // p . g before the descent reset
  S_SLOPE0,     // g . p of the direction actually searched
  S_A0,         // initial step
  S_RESET,      // 1 when the direction fell back to -g
  S_FA,         // trial objective
  S_DA,         // trial directional derivative ga . p
  S_XBAD,       // non-finite entries of the trial point
  S_F,          // objective at the accepted point
  S_COUNT
};

__device__ __forceinline__ double block_sum(double v, double* red) {
  // fixed-order tree: warp butterfly, then warp 0 butterflies the warp totals
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    double t = l < (int)(blockDim.x >> 5) ? red[l] : 0.0;
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (l == 0) red[32] = t;
  }
  __syncthreads();
  return red[32];
}

__device__ __forceinline__ double block_max(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    double t = l < (int)(blockDim.x >> 5) ? red[l] : 0.0;
    for (int o = 16; o > 0; o >>= 1) t = fmax(t, __shfl_xor_sync(0xffffffffu, t, o));
    if (l == 0) red[32] = t;
  }
  __syncthreads();
  return red[32];
}

// "last block done": true in exactly one block, after every block's partials are visible.
// The finishing block sums the per-block partials in index order, so results do not depend on
// which block finishes last.
__device__ __forceinline__ bool last_block(unsigned* counter) {
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned done = atomicAdd(counter, 1u);
    last = done == gridDim.x - 1;
    if (last) *counter = 0u;  // re-arm for the next launch
  }
  __syncthreads();
  if (last) __threadfence();
  return last;
}

// stage 1 of the |g| statistics at a freshly evaluated point (init): max, sum, non-finite(g, x)
__device__ void lb_eval_fin(int nb, const double* __restrict__ part,
                            const double* __restrict__ out, double* __restrict__ st,
                            int* __restrict__ ring);

__global__ void k_lb_eval_stats(int64_t N, const double* __restrict__ x,
                                const double* __restrict__ out, double* __restrict__ part,
                                unsigned* counter, double* __restrict__ st, int* __restrict__ ring) {
  __shared__ double red[33];
  const double* g = out + 1;
  double mx = 0.0, sm = 0.0, bad = 0.0;
  for (int64_t j = blockIdx.x * (int64_t)LB_T + threadIdx.x; j < N; j += (int64_t)gridDim.x * LB_T) {
    const double a = fabs(g[j]);
    mx = fmax(mx, a);
    sm += a;
    bad += (isfinite(g[j]) && isfinite(x[j])) ? 0.0 : 1.0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && !isfinite(out[0])) bad += 1.0;
  mx = block_max(mx, red);
  sm = block_sum(sm, red);
  bad = block_sum(bad, red);
  if (threadIdx.x == 0) {
    part[blockIdx.x * LB_NP + 0] = mx;
    part[blockIdx.x * LB_NP + 1] = sm;
    part[blockIdx.x * LB_NP + 2] = bad;
  }
  if (last_block(counter) && threadIdx.x == 0) lb_eval_fin(gridDim.x, part, out, st, ring);
}

__device__ void lb_eval_fin(int nb, const double* __restrict__ part,
                            const double* __restrict__ out, double* __restrict__ st,
                            int* __restrict__ ring) {
  double mx = 0.0, sm = 0.0, bad = 0.0;
  for (int b = 0; b < nb; ++b) {
    mx = fmax(mx, part[b * LB_NP + 0]);
    sm += part[b * LB_NP + 1];
    bad += part[b * LB_NP + 2];
  }
  st[S_GMAX] = bad > 0.0 ? INFINITY : mx;
  st[S_GSUM] = sm;
  st[S_GBAD] = bad;
  st[S_KEEP] = 0.0;
  st[S_F] = out[0];
  ring[0] = 0;  // count
  ring[1] = 0;  // head
}

// accept the step to (xs, outs): s = xs - x, y = gs - g into ring slot `head`, x <- xs, g <- gs
__device__ void lb_accept_fin(int nb, const double* __restrict__ part, int m,
                              int* __restrict__ ring, double* __restrict__ sy_hist,
                              double* __restrict__ yy_hist, const double* __restrict__ outx,
                              double* __restrict__ st);

__global__ void k_lb_accept(int64_t N, const double* __restrict__ xs,
                            const double* __restrict__ outs, double* __restrict__ x,
                            double* __restrict__ outx, double* __restrict__ S,
                            double* __restrict__ Y, int* __restrict__ ring,
                            double* __restrict__ part, unsigned* counter, int m,
                            double* __restrict__ sy_hist, double* __restrict__ yy_hist,
                            double* __restrict__ st) {
  __shared__ double red[33];
  const int head = ring[1];
  double* s_out = S + (int64_t)head * N;
  double* y_out = Y + (int64_t)head * N;
  double* g = outx + 1;
  const double* gs = outs + 1;
  double sy = 0.0, ss = 0.0, yy = 0.0, mx = 0.0, sm = 0.0, bad = 0.0;
  for (int64_t j = blockIdx.x * (int64_t)LB_T + threadIdx.x; j < N; j += (int64_t)gridDim.x * LB_T) {
    const double sj = __dsub_rn(xs[j], x[j]);
    const double yj = __dsub_rn(gs[j], g[j]);
    s_out[j] = sj;
    y_out[j] = yj;
    x[j] = xs[j];
    g[j] = gs[j];
    sy += __dmul_rn(sj, yj);
    ss += __dmul_rn(sj, sj);
    yy += __dmul_rn(yj, yj);
    const double a = fabs(gs[j]);
    mx = fmax(mx, a);
    sm += a;
    bad += isfinite(gs[j]) ? 0.0 : 1.0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) outx[0] = outs[0];
  sy = block_sum(sy, red);
  ss = block_sum(ss, red);
  yy = block_sum(yy, red);
  mx = block_max(mx, red);
  sm = block_sum(sm, red);
  bad = block_sum(bad, red);
  if (threadIdx.x == 0) {
    double* pp = part + blockIdx.x * LB_NP;
    pp[0] = sy;
    pp[1] = ss;
    pp[2] = yy;
    pp[3] = mx;
    pp[4] = sm;
    pp[5] = bad;
  }
  if (last_block(counter) && threadIdx.x == 0)
    lb_accept_fin(gridDim.x, part, m, ring, sy_hist, yy_hist, outx, st);
}

// curvature test (optimize.py:330-332) and ring update
__device__ void lb_accept_fin(int nb, const double* __restrict__ part, int m,
                              int* __restrict__ ring, double* __restrict__ sy_hist,
                              double* __restrict__ yy_hist, const double* __restrict__ outx,
                              double* __restrict__ st) {
  double sy = 0.0, ss = 0.0, yy = 0.0, mx = 0.0, sm = 0.0, bad = 0.0;
  for (int b = 0; b < nb; ++b) {
    const double* pp = part + b * LB_NP;
    sy += pp[0];
    ss += pp[1];
    yy += pp[2];
    mx = fmax(mx, pp[3]);
    sm += pp[4];
    bad += pp[5];
  }
  const bool keep = sy > __dmul_rn(__dmul_rn(1e-12, sqrt(ss)), sqrt(yy));
  if (keep) {
    const int head = ring[1];
    sy_hist[head] = sy;
    yy_hist[head] = yy;
    ring[1] = (head + 1) % (m + 1);
    ring[0] = min(ring[0] + 1, m);
  }
  st[S_GMAX] = bad > 0.0 ? INFINITY : mx;
  st[S_GSUM] = sm;
  st[S_GBAD] = bad;
  st[S_KEEP] = keep ? 1.0 : 0.0;
  st[S_F] = outx[0];
}

// Two-loop recursion (optimize.py:149-168) in one CTA, then the descent check and the initial
// step (optimize.py:307-322) and the first trial point.  When the window fits (stage != 0), g and
// the (s, y) window are staged in shared memory first so the 2m+1 dependent passes run at smem
// latency instead of L2 latency.
__global__ void __launch_bounds__(LB_DIR_T) k_lb_direction(
    int64_t N, const double* __restrict__ outx, const double* __restrict__ S,
    const double* __restrict__ Y, int m, int* __restrict__ ring, const double* __restrict__ sy_h,
    const double* __restrict__ yy_h, double* __restrict__ P, double* __restrict__ st,
    double* __restrict__ a_dev, const double* __restrict__ X, double* __restrict__ T,
    int stage) {
  extern __shared__ double sm[];
  __shared__ double red[33];
  __shared__ double alpha_s[65];
  const int count = ring[0], head = ring[1];
  const int M1 = m + 1;
  auto slot = [&](int i) { return (head - count + i + 2 * M1) % M1; };  // i = 0 oldest
  // views: q, g, s_i, y_i (i = 0 oldest) -- shared memory or global
  double* q = stage ? sm : P;
  const double* g = outx + 1;
  if (stage) {
    double* gs = sm + N;
    for (int64_t j = threadIdx.x; j < N; j += blockDim.x) gs[j] = g[j];
    for (int i = 0; i < count; ++i) {
      const double* Sg = S + (int64_t)slot(i) * N;
      const double* Yg = Y + (int64_t)slot(i) * N;
      double* Ss = sm + (2 + 2 * (int64_t)i) * N;
      for (int64_t j = threadIdx.x; j < N; j += blockDim.x) {
        Ss[j] = Sg[j];
        Ss[N + j] = Yg[j];
      }
    }
    g = gs;
    __syncthreads();
  }
  auto Sv = [&](int i) -> const double* {
    return stage ? sm + (2 + 2 * (int64_t)i) * N : S + (int64_t)slot(i) * N;
  };
  auto Yv = [&](int i) -> const double* {
    return stage ? sm + (3 + 2 * (int64_t)i) * N : Y + (int64_t)slot(i) * N;
  };
  double pg;
  bool reset = false;
  if (count > 0) {
    const int newest = slot(count - 1);
    const double gamma = sy_h[newest] / yy_h[newest];
    // loop 1, newest -> oldest: alpha_i = rho_i * (s_i . q); q -= alpha_i * y_i
    double acc = 0.0;
    {
      const double* Si = Sv(count - 1);
      for (int64_t j = threadIdx.x; j < N; j += blockDim.x) {
        const double qj = g[j];
        q[j] = qj;
        acc += __dmul_rn(Si[j], qj);
      }
    }
    for (int i = count - 1; i >= 0; --i) {
      const double dot = block_sum(acc, red);
      const double alpha = __dmul_rn(1.0 / sy_h[slot(i)], dot);
      if (threadIdx.x == 0) alpha_s[i] = alpha;
      const double* Yi = Yv(i);
      acc = 0.0;
      if (i > 0) {
        const double* Sn = Sv(i - 1);
        for (int64_t j = threadIdx.x; j < N; j += blockDim.x) {
          const double qj = __dsub_rn(q[j], __dmul_rn(alpha, Yi[j]));
          q[j] = qj;
          acc += __dmul_rn(Sn[j], qj);
        }
      } else {
        // last update of loop 1, q *= gamma, then the first dot of loop 2 (y_oldest . q)
        const double* Y0 = Yv(0);
        for (int64_t j = threadIdx.x; j < N; j += blockDim.x) {
          const double qj = __dmul_rn(__dsub_rn(q[j], __dmul_rn(alpha, Yi[j])), gamma);
          q[j] = qj;
          acc += __dmul_rn(Y0[j], qj);
        }
      }
    }
    __syncthreads();
    // loop 2, oldest -> newest: beta = rho_i * (y_i . q); q += (alpha_i - beta) * s_i
    for (int i = 0; i < count; ++i) {
      const double dot = block_sum(acc, red);
      const double beta = __dmul_rn(1.0 / sy_h[slot(i)], dot);
      const double coef = __dsub_rn(alpha_s[i], beta);
      const double* Si = Sv(i);
      acc = 0.0;
      if (i + 1 < count) {
        const double* Yn = Yv(i + 1);
        for (int64_t j = threadIdx.x; j < N; j += blockDim.x) {
          const double qj = __dadd_rn(q[j], __dmul_rn(coef, Si[j]));
          q[j] = qj;
          acc += __dmul_rn(Yn[j], qj);
        }
      } else {
        // direction = -q and p . g
        for (int64_t j = threadIdx.x; j < N; j += blockDim.x) {
          const double pj = -__dadd_rn(q[j], __dmul_rn(coef, Si[j]));
          P[j] = pj;
          acc += __dmul_rn(pj, g[j]);
        }
      }
    }
    pg = block_sum(acc, red);
    reset = pg >= 0.0;  // float(p @ g) >= 0.0 (NaN does not reset)
  } else {
    double acc = 0.0;
    for (int64_t j = threadIdx.x; j < N; j += blockDim.x) {
      const double pj = -g[j];
      P[j] = pj;
      acc += __dmul_rn(pj, g[j]);
    }
    pg = block_sum(acc, red);
    reset = pg >= 0.0;
  }
  double slope0 = pg, a0 = 1.0;
  if (count == 0 || reset) {
    if (reset && count > 0) {
      double acc = 0.0;
      for (int64_t j = threadIdx.x; j < N; j += blockDim.x) {
        const double pj = -g[j];
        P[j] = pj;
        acc += __dmul_rn(g[j], pj);
      }
      slope0 = block_sum(acc, red);
    }
    a0 = fmin(1.0, 1.0 / fmax(st[S_GSUM], 1e-12));
  }
  // first trial point x + a0 p (optimize.py:187); each thread reads back its own P entries
  for (int64_t j = threadIdx.x; j < N; j += blockDim.x) T[j] = __dadd_rn(X[j], __dmul_rn(a0, P[j]));
  if (threadIdx.x == 0) {
    if (reset) ring[0] = 0;
    st[S_PG] = pg;
    st[S_SLOPE0] = slope0;
    st[S_A0] = a0;
    st[S_RESET] = reset ? 1.0 : 0.0;
    a_dev[0] = a0;
  }
}

// trial point xa = x + a * p (optimize.py:187)
__global__ void k_lb_trial(int64_t N, const double* __restrict__ x, const double* __restrict__ P,
                           const double* __restrict__ a_dev, double* __restrict__ xt) {
  const double a = a_dev[0];
  for (int64_t j = blockIdx.x * (int64_t)LB_T + threadIdx.x; j < N; j += (int64_t)gridDim.x * LB_T)
    xt[j] = __dadd_rn(x[j], __dmul_rn(a, P[j]));
}

// ga . p and the finiteness of the trial point
__global__ void k_lb_probe_stats(int64_t N, const double* __restrict__ xt,
                                 const double* __restrict__ outt, const double* __restrict__ P,
                                 double* __restrict__ part, unsigned* counter,
                                 double* __restrict__ st) {
  __shared__ double red[33];
  const double* ga = outt + 1;
  double dp = 0.0, bad = 0.0;
  for (int64_t j = blockIdx.x * (int64_t)LB_T + threadIdx.x; j < N; j += (int64_t)gridDim.x * LB_T) {
    dp += __dmul_rn(ga[j], P[j]);
    bad += isfinite(xt[j]) ? 0.0 : 1.0;
  }
  dp = block_sum(dp, red);
  bad = block_sum(bad, red);
  if (threadIdx.x == 0) {
    part[blockIdx.x * LB_NP + 0] = dp;
    part[blockIdx.x * LB_NP + 1] = bad;
  }
  if (!last_block(counter) || threadIdx.x != 0) return;
  const int nb = gridDim.x;
  dp = 0.0;
  bad = 0.0;
  for (int b = 0; b < nb; ++b) {
    dp += part[b * LB_NP + 0];
    bad += part[b * LB_NP + 1];
  }
  st[S_FA] = outt[0];
  st[S_DA] = dp;
  st[S_XBAD] = bad;
}

// ------------------------------------------------------------------------------------------
// host side

// Workspace + graphs for one (d, r, mode, memory, alpha); cached on the context between runs
// (setup costs pinned allocations and four graph instantiations, ~ms).
struct LbRun {
  mcp_ctx* c = nullptr;
  int d = 0, r = 0, mode = 0, m = 0;
  double alpha = 0.0;
  int64_t n = 0;
  int64_t N = 0;
  int nb = 1;
  int dir_threads = LB_DIR_T;
  size_t dir_smem = 0;
  EvalPlan pl;
  std::vector<void*> dev;
  double *X = nullptr, *OX = nullptr, *T = nullptr, *OT = nullptr, *B = nullptr, *OB = nullptr;
  double *P = nullptr, *S = nullptr, *Y = nullptr, *syh = nullptr, *yyh = nullptr;
  double *part = nullptr, *st = nullptr, *a_dev = nullptr, *Yw = nullptr;
  int* ring = nullptr;
  unsigned* counter = nullptr;
  double* hst = nullptr;   // pinned: stats
  double* ha = nullptr;    // pinned: host-chosen step
  double* hx = nullptr;    // pinned: x0 / hook copies
  GraphEntry g_init, g_iter_t, g_iter_b, g_probe;

  ~LbRun() {
    for (GraphEntry* g : {&g_init, &g_iter_t, &g_iter_b, &g_probe}) {
      if (g->exec) cudaGraphExecDestroy(g->exec);
      if (g->graph) cudaGraphDestroy(g->graph);
    }
    for (void* p : dev) cudaFree(p);
    if (hst) cudaFreeHost(hst);
    if (ha) cudaFreeHost(ha);
    if (hx) cudaFreeHost(hx);
  }

  template <typename T>
  int alloc(T*& p, size_t elems) {
    void* q = nullptr;
    CUDA_TRY(c, cudaMalloc(&q, sizeof(T) * (elems ? elems : 1)));
    dev.push_back(q);
    p = (T*)q;
    return MCP_OK;
  }

  // fg(x) -> out on the context stream (K1 -> K3 -> K4)
  int enqueue_fg(const double* x, double* out) {
    return enqueue_fg_full(c, pl, x, nullptr, alpha, out, c->stream);
  }

  int enqueue_direction_and_probe() {
    cudaStream_t s = c->stream;
    k_lb_direction<<<1, dir_threads, dir_smem, s>>>(N, OX, S, Y, m, ring, syh, yyh, P, st, a_dev,
                                                    X, T, dir_smem ? 1 : 0);
    return enqueue_probe_tail(false);
  }

  int enqueue_probe_tail(bool trial) {
    cudaStream_t s = c->stream;
    if (trial) k_lb_trial<<<nb, LB_T, 0, s>>>(N, X, P, a_dev, T);
    int rc = enqueue_fg(T, OT);
    if (rc) return rc;
    k_lb_probe_stats<<<nb, LB_T, 0, s>>>(N, T, OT, P, part, counter, st);
    CUDA_TRY(c, cudaMemcpyAsync(hst, st, sizeof(double) * S_COUNT, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(c, cudaGetLastError());
    return MCP_OK;
  }

  template <typename F>
  int capture(GraphEntry& ge, F&& body) {
    CUDA_TRY(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    int rc = body();
    cudaError_t ce = cudaStreamEndCapture(c->stream, &ge.graph);
    if (rc) return rc;
    CUDA_TRY(c, ce);
    CUDA_TRY(c, cudaGraphInstantiate(&ge.exec, ge.graph, 0));
    return MCP_OK;
  }

  int replay(GraphEntry& ge) {
    CUDA_TRY(c, cudaGraphLaunch(ge.exec, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return MCP_OK;
  }

  bool matches(int d_, int r_, int mode_, int m_, double alpha_) const {
    return d == d_ && r == r_ && mode == mode_ && m == m_ && n == c->n &&
           std::memcmp(&alpha, &alpha_, sizeof(double)) == 0;
  }

  int setup() {
    n = c->n;
    N = r + n * r;
    nb = grid_for(N, LB_T, LB_MAX_BLOCKS);
    dir_threads = N <= 8192 ? 256 : LB_DIR_T;
    const size_t stage_bytes = sizeof(double) * (size_t)N * (2 * (size_t)m + 2);
    dir_smem = stage_bytes <= 192 * 1024 ? stage_bytes : 0;
    int rc;
    if (dir_smem)
      CUDA_TRY(c, cudaFuncSetAttribute(k_lb_direction, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)dir_smem));
    const size_t M1 = (size_t)m + 1;
    if ((rc = alloc(X, N)) || (rc = alloc(OX, N + 1)) || (rc = alloc(T, N)) ||
        (rc = alloc(OT, N + 1)) || (rc = alloc(B, N)) || (rc = alloc(OB, N + 1)) ||
        (rc = alloc(P, N)) || (rc = alloc(S, M1 * N)) || (rc = alloc(Y, M1 * N)) ||
        (rc = alloc(syh, M1)) || (rc = alloc(yyh, M1)) || (rc = alloc(part, LB_NP * nb)) ||
        (rc = alloc(st, S_COUNT)) || (rc = alloc(a_dev, 1)) || (rc = alloc(Yw, n * r + r)) ||
        (rc = alloc(ring, 2)) || (rc = alloc(counter, 1)))
      return rc;
    CUDA_TRY(c, cudaMemset(counter, 0, sizeof(unsigned)));
    CUDA_TRY(c, cudaMallocHost(&hst, sizeof(double) * S_COUNT));
    CUDA_TRY(c, cudaMallocHost(&ha, sizeof(double)));
    CUDA_TRY(c, cudaMallocHost(&hx, sizeof(double) * N));
    cudaStream_t s = c->stream;
    if ((rc = capture(g_init, [&]() -> int {
           CUDA_TRY(c, cudaMemcpyAsync(X, hx, sizeof(double) * N, cudaMemcpyHostToDevice, s));
           int e = enqueue_fg(X, OX);
           if (e) return e;
           k_lb_eval_stats<<<nb, LB_T, 0, s>>>(N, X, OX, part, counter, st, ring);
           return enqueue_direction_and_probe();
         })))
      return rc;
    for (int which = 0; which < 2; ++which) {
      const double* xs = which == 0 ? T : B;
      const double* os = which == 0 ? OT : OB;
      if ((rc = capture(which == 0 ? g_iter_t : g_iter_b, [&]() -> int {
             k_lb_accept<<<nb, LB_T, 0, s>>>(N, xs, os, X, OX, S, Y, ring, part, counter, m,
                                             syh, yyh, st);
             return enqueue_direction_and_probe();
           })))
        return rc;
    }
    if ((rc = capture(g_probe, [&]() -> int {
           CUDA_TRY(c, cudaMemcpyAsync(a_dev, ha, sizeof(double), cudaMemcpyHostToDevice, s));
           return enqueue_probe_tail(true);
         })))
      return rc;
    return MCP_OK;
  }

  int save_best() {
    CUDA_TRY(c, cudaMemcpyAsync(B, T, sizeof(double) * N, cudaMemcpyDeviceToDevice, c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(OB, OT, sizeof(double) * (N + 1), cudaMemcpyDeviceToDevice,
                                c->stream));
    return MCP_OK;
  }
};

// optimize.py:171-176
bool interp(double a_lo, double f_lo, double d_lo, double a_hi, double f_hi, double* out) {
  const double den = f_hi - f_lo - d_lo * (a_hi - a_lo);
  if (den == 0 || !std::isfinite(den)) return false;
  const double cnd = a_lo - 0.5 * d_lo * ((a_hi - a_lo) * (a_hi - a_lo)) / den;
  if (!std::isfinite(cnd)) return false;
  *out = cnd;
  return true;
}

struct Pt {
  double a, f, d;
};

enum { WOLFE_T = 0, WOLFE_BEST = 1, WOLFE_FAIL = 2 };

// Strong-Wolfe search (optimize.py:179-252).  The first probe (at a0) has already been run by
// the iteration graph; its scalars are in R.hst.
int wolfe(LbRun& R, double f0, double slope0, double a0, double c1, double c2, int64_t budget,
          int* outcome, double* f_new, int64_t* evals, std::string& err_x) {
  int64_t ev = 0;
  bool have_best = false;
  double best_f = 0.0;
  bool first = true;
  int rc;
  auto probe = [&](double a, double* fa, double* da) -> int {
    if (!first) {
      *R.ha = a;
      if ((rc = R.replay(R.g_probe))) return rc;
    }
    first = false;
    if (R.hst[S_XBAD] > 0.0) {
      err_x = "model variables and alpha must be finite";
      return MCP_ERR_ARG;
    }
    ++ev;
    *fa = R.hst[S_FA];
    *da = std::isfinite(*fa) ? R.hst[S_DA] : NAN;
    if (std::isfinite(*fa) && *fa <= f0 + c1 * a * slope0) {
      if (!have_best || *fa < best_f) {
        have_best = true;
        best_f = *fa;
        if ((rc = R.save_best())) return rc;
      }
    }
    return MCP_OK;
  };
  auto fallback = [&]() {
    *evals = ev;
    if (have_best) {
      *outcome = WOLFE_BEST;
      *f_new = best_f;
    } else {
      *outcome = WOLFE_FAIL;
    }
    return MCP_OK;
  };
  Pt prev{0.0, f0, slope0};
  double a = a0;
  bool bracketed = false;
  Pt lo{}, hi{};
  for (int64_t it = 0; it < budget; ++it) {
    double fa, da;
    if ((rc = probe(a, &fa, &da))) return rc;
    const bool bad = !std::isfinite(fa) || fa > f0 + c1 * a * slope0 ||
                     (prev.a > 0.0 && fa >= prev.f);
    if (bad) {
      lo = prev;
      hi = Pt{a, fa, da};
      bracketed = true;
      break;
    }
    if (std::fabs(da) <= -c2 * slope0) {
      *outcome = WOLFE_T;
      *f_new = fa;
      *evals = ev;
      return MCP_OK;
    }
    if (da >= 0.0) {
      lo = Pt{a, fa, da};
      hi = prev;
      bracketed = true;
      break;
    }
    prev = Pt{a, fa, da};
    a = std::fmin(2.0 * a, 1e20);
  }
  if (!bracketed) return fallback();
  while (ev < budget) {
    const double width = hi.a - lo.a;
    double cand = 0.0;
    bool ok = std::isfinite(hi.f) && interp(lo.a, lo.f, lo.d, hi.a, hi.f, &cand);
    const double lb = lo.a + 0.1 * width, ub = hi.a - 0.1 * width;
    if (!ok || !(std::fmin(lb, ub) <= cand && cand <= std::fmax(lb, ub))) cand = lo.a + 0.5 * width;
    double fa, da;
    if ((rc = probe(cand, &fa, &da))) return rc;
    if (!std::isfinite(fa) || fa > f0 + c1 * cand * slope0 || fa >= lo.f) {
      hi = Pt{cand, fa, da};
    } else {
      if (std::fabs(da) <= -c2 * slope0) {
        *outcome = WOLFE_T;
        *f_new = fa;
        *evals = ev;
        return MCP_OK;
      }
      if (da * (hi.a - lo.a) >= 0.0) hi = lo;
      lo = Pt{cand, fa, da};
    }
    if (std::fabs(hi.a - lo.a) < 1e-16 * std::fmax(1.0, std::fabs(lo.a))) break;
  }
  return fallback();
}

}  // namespace

extern "C" int mcp_lbfgs(mcp_ctx* c, int d, int r, double alpha, int mode, const double* x0,
                         const double* opts, double* x_out, double* g_out, double* f_out,
                         double* trace_f, double* trace_t, int64_t trace_cap, int64_t* info,
                         mcp_iterate_hook hook, void* hook_user) {
  if (!c) return MCP_ERR_ARG;
  Guard gd(c);
  if (!x0 || !opts || !x_out || !g_out || !f_out || !info)
    return c->fail(MCP_ERR_ARG, "NULL argument");
  if (!std::isfinite(alpha)) return c->fail(MCP_ERR_ARG, "model variables and alpha must be finite");
  const int memory = (int)opts[0];
  const double pgtol = opts[1];
  const int64_t max_iters = (int64_t)opts[2], max_total = (int64_t)opts[3];
  const double c1 = opts[4], c2 = opts[5];
  const int64_t max_line_steps = (int64_t)opts[6];
  if (!(pgtol > 0)) return c->fail(MCP_ERR_ARG, "pgtol must be > 0");
  if (memory < 1) return c->fail(MCP_ERR_ARG, "memory must be >= 1");
  if (memory > 64) return c->fail(MCP_ERR_ARG, "memory > 64 is not supported by the device solver");
  if (!c->loaded) return c->fail(MCP_ERR_STATE, "no observation set loaded (call mcp_load_obs)");
  const auto t_start = std::chrono::steady_clock::now();
  auto seconds = [&]() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  };
  // plan first: a buffer growth drops cached graphs (and the cached workspace with them)
  EvalPlan pl;
  int rc = plan_eval(c, d, r, mode, pl);
  if (rc) return rc;
  LbRun* ws = (LbRun*)c->lbfgs_ws;
  if (!ws || !ws->matches(d, r, mode, memory, alpha)) {
    if (ws) {
      c->lbfgs_ws_free(ws);
      c->lbfgs_ws = nullptr;
    }
    ws = new LbRun();
    ws->c = c;
    ws->d = d;
    ws->r = r;
    ws->mode = mode;
    ws->m = memory;
    ws->alpha = alpha;
    ws->pl = pl;
    if ((rc = ws->setup())) {
      delete ws;
      return rc;
    }
    c->lbfgs_ws = ws;
    c->lbfgs_ws_free = [](void* p) { delete (LbRun*)p; };
  }
  LbRun& R = *ws;
  const int64_t N = R.N;
  std::memcpy(R.hx, x0, sizeof(double) * N);
  for (int64_t j = 0; j < N; ++j)
    if (!std::isfinite(x0[j])) return c->fail(MCP_ERR_ARG, "model variables and alpha must be finite");
  if ((rc = R.replay(R.g_init))) return rc;
  int64_t n_fg = 1;
  if (!std::isfinite(R.hst[S_F]) || R.hst[S_GBAD] > 0.0)
    return c->fail(MCP_ERR_ARG, "objective is not finite at the starting point");
  double f = R.hst[S_F];
  int64_t n_trace = 0;
  auto push_trace = [&](double fv) {
    if (n_trace < trace_cap) {
      if (trace_f) trace_f[n_trace] = fv;
      if (trace_t) trace_t[n_trace] = seconds();
    }
    ++n_trace;
  };
  auto call_hook = [&]() -> int {
    if (!hook) return MCP_OK;
    CUDA_TRY(c, cudaMemcpyAsync(R.hx, R.X, sizeof(double) * N, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    hook(R.hx, N, hook_user);
    return MCP_OK;
  };
  push_trace(f);
  if ((rc = call_hook())) return rc;
  int64_t steps = 0;
  int reason = 1;
  std::string err_x;
  while (true) {
    if (R.hst[S_GMAX] <= pgtol) {
      reason = 0;
      break;
    }
    if (steps >= max_iters || n_fg >= max_total) {
      reason = 1;
      break;
    }
    const double slope0 = R.hst[S_SLOPE0], a0 = R.hst[S_A0];
    const int64_t budget = std::min<int64_t>(max_line_steps, max_total - n_fg);
    int outcome = WOLFE_FAIL;
    double f_new = f;
    int64_t ev = 0;
    if (budget > 0) {
      rc = wolfe(R, f, slope0, a0, c1, c2, budget, &outcome, &f_new, &ev, err_x);
      if (rc) return rc == MCP_ERR_ARG ? c->fail(rc, err_x) : rc;
    }
    n_fg += ev;
    if (outcome == WOLFE_FAIL) {
      reason = n_fg >= max_total ? 1 : 2;
      break;
    }
    // accept, curvature-test the pair, next direction and its first probe -- one replay
    if ((rc = R.replay(outcome == WOLFE_T ? R.g_iter_t : R.g_iter_b))) return rc;
    f = R.hst[S_F];
    ++steps;
    push_trace(f);
    if ((rc = call_hook())) return rc;
  }
  // the final state: x, [f; g]
  CUDA_TRY(c, cudaMemcpyAsync(x_out, R.X, sizeof(double) * N, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(g_out, R.OX + 1, sizeof(double) * N, cudaMemcpyDeviceToHost,
                              c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  *f_out = f;
  info[0] = n_fg;
  info[1] = steps;
  info[2] = reason;
  info[3] = std::min(n_trace, trace_cap);
  return MCP_OK;
}
