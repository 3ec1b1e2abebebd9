// Device-resident L-BFGS over the momentcp objective, for one run or k runs in lock step
// (SURVEY.md 8f #1 and #2).
//
// Reference: pkg/src/momentcp/optimize.py:149-168 (two-loop recursion), :171-176 (safeguarded
// quadratic interpolation), :179-252 (strong-Wolfe bracket/zoom), :255-355 (outer loop),
// :454-508 (multistart).
//
// Per run, HBM holds x, g = fg(x), the direction p, a trial point xa with its [fa; ga], a saved
// best trial, and a ring of memory+1 (s, y) slots (the spare slot takes the new pair before the
// curvature test decides whether it joins the window, so a rejected pair never evicts the
// oldest accepted one -- the reference's deque only appends accepted pairs).
//
// One "round" evaluates exactly one trial point per active run.  Each run's host-side state
// machine (the reference's line search, made resumable) picks the run's action for the round:
//   PROBE          trial at a host-chosen step a (inside a line search)
//   ACC_T / ACC_B  accept the last trial / the saved best, curvature-test the (s, y) pair, run
//                  the two-loop recursion, the descent check and a0, then probe x + a0 p
//   IDLE           finished run (its columns ride along)
// plus SAVE (copy the last trial into the best slot first).  A round is ONE CUDA graph:
//   H2D(actions, steps) -> save -> accept -> direction -> trial -> f+grad -> probe stats -> D2H
// With k runs the f+grad is a single pass over V with k*r factor columns (the K1 family) and
// per-run tails, so k lock-step runs cost about one run's latency per round.  The host reads
// back ~12 doubles per run and takes the reference's decisions in the reference's order.
// Elementwise updates use explicit round-to-nearest operations (no FMA contraction), so given
// equal scalars they match numpy's `x + a * p`, `q -= alpha * y`, ... bit for bit; dot products
// are fixed-order reductions (deterministic, summed in a different order than numpy's).
#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "ctx.h"
#include "pdl.h"

using namespace mcp_internal;
using mcp::launch_pdl;
using mcp::pdl_enter;

namespace {

constexpr int LB_T = 256;        // threads of the streaming kernels
constexpr int LB_DIR_T = 1024;   // the one-CTA-per-run two-loop kernel (large N)
constexpr int LB_NP = 6;         // partial sums per block
constexpr int LB_MAX_BLOCKS = 296;
// one block per run (N <= LB_T) and the fused round prologue up to here.  Measured against the
// separate kernels (tools/lbfgs_small_ab.py): N = 105 45.0 vs 49.4 us per step; forcing one
// block per run at N = 1010 / 2010 loses (88.3 vs 81.1, 87.5 vs 75.0 us per step)
constexpr int64_t LB_SMALL_N = 256;

// actions (low 3 bits) + flag
enum { ACT_PROBE = 0, ACT_ACC_T = 1, ACT_ACC_B = 2, ACT_IDLE = 3, ACT_INIT = 4, ACT_SAVE = 8 };

// scalar slots of a run's stats record, copied to the host after every round
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

// Device view of the k runs' state (passed by value; run s = blockIdx.y).
struct LbDev {
  int64_t N;
  int m, k;
  double *X, *OX, *T, *OT, *B, *OB, *P, *S, *Y, *syh, *yyh, *part, *st, *a0, *ah;
  int* ring;
  unsigned* counter;
  const int* act;
  double* Xb;   // batched K1 layout [lam_all (k r) ; A_all (n x k r)] or nullptr (k == 1)
  double* st_host;   // mapped pinned copy of the stats records (written by the probe kernel)
  unsigned long long* seq_dev;    // per run: rounds whose record has been written
  unsigned long long* seq_host;   // the same count in mapped pinned memory, stored after the
                                  // record: the host polls it instead of synchronising the stream
  int r;
  int64_t n;
  __device__ int action(int s) const { return act[s] & 7; }
  __device__ double* x(int s) const { return X + (int64_t)s * N; }
  __device__ double* ox(int s) const { return OX + (int64_t)s * (N + 1); }
  __device__ double* t(int s) const { return T + (int64_t)s * N; }
  __device__ double* ot(int s) const { return OT + (int64_t)s * (N + 1); }
  __device__ double* b(int s) const { return B + (int64_t)s * N; }
  __device__ double* ob(int s) const { return OB + (int64_t)s * (N + 1); }
  __device__ double* p(int s) const { return P + (int64_t)s * N; }
  __device__ double* sr(int s) const { return S + (int64_t)s * (m + 1) * N; }
  __device__ double* yr(int s) const { return Y + (int64_t)s * (m + 1) * N; }
  __device__ double* sy(int s) const { return syh + (int64_t)s * (m + 1); }
  __device__ double* yy(int s) const { return yyh + (int64_t)s * (m + 1); }
  __device__ double* pt(int s) const { return part + (int64_t)s * gridDim.x * LB_NP; }
  __device__ double* stats(int s) const { return st + (int64_t)s * S_COUNT; }
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

// "last block done" (per run): true in exactly one block of the run, after every block's
// partials are visible.  The finishing block sums the partials in index order, so results do
// not depend on which block finishes last.
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

#define LB_FOR(j) \
  for (int64_t j = blockIdx.x * (int64_t)LB_T + threadIdx.x; j < D.N; j += (int64_t)gridDim.x * LB_T)

// SAVE: the last trial becomes the saved best (before this round overwrites it)
__device__ __forceinline__ void lbb_save(const LbDev& D) {
  const int s = blockIdx.y;
  if (!(D.act[s] & ACT_SAVE)) return;
  const double *t = D.t(s), *ot = D.ot(s);
  double *b = D.b(s), *ob = D.ob(s);
  LB_FOR(j) {
    b[j] = t[j];
    ob[1 + j] = ot[1 + j];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) ob[0] = ot[0];
}
__global__ void k_lbb_save(LbDev D) {
  pdl_enter();   // chained under programmatic dependent launch: wait, then let the successor launch
  lbb_save(D);
}


// INIT: x0's evaluation lives in OT; take it as [f; g] of x, statistics, ring reset
__global__ void k_lbb_init_stats(LbDev D) {
  pdl_enter();   // chained under programmatic dependent launch: wait, then let the successor launch
  __shared__ double red[33];
  const int s = blockIdx.y;
  const double* out = D.ot(s);
  double* ox = D.ox(s);
  const double* x = D.x(s);
  double mx = 0.0, sm = 0.0, bad = 0.0;
  LB_FOR(j) {
    const double gj = out[1 + j];
    ox[1 + j] = gj;
    const double a = fabs(gj);
    mx = fmax(mx, a);
    sm += a;
    bad += (isfinite(gj) && isfinite(x[j])) ? 0.0 : 1.0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ox[0] = out[0];
    if (!isfinite(out[0])) bad += 1.0;
  }
  mx = block_max(mx, red);
  sm = block_sum(sm, red);
  bad = block_sum(bad, red);
  double* pp = D.pt(s) + blockIdx.x * LB_NP;
  if (threadIdx.x == 0) {
    pp[0] = mx;
    pp[1] = sm;
    pp[2] = bad;
  }
  if (!last_block(D.counter + s) || threadIdx.x != 0) return;
  mx = 0.0;
  sm = 0.0;
  bad = 0.0;
  for (int b = 0; b < (int)gridDim.x; ++b) {
    const double* q = D.pt(s) + b * LB_NP;
    mx = fmax(mx, q[0]);
    sm += q[1];
    bad += q[2];
  }
  double* st = D.stats(s);
  st[S_GMAX] = bad > 0.0 ? INFINITY : mx;
  st[S_GSUM] = sm;
  st[S_GBAD] = bad;
  st[S_KEEP] = 0.0;
  st[S_F] = out[0];
  D.ring[2 * s] = 0;      // count
  D.ring[2 * s + 1] = 0;  // head
}

// ACC_T / ACC_B: s = xs - x, y = gs - g into ring slot `head`, x <- xs, g <- gs; then the
// curvature test (optimize.py:330-332) and the ring update in the run's last block
__device__ __forceinline__ void lbb_accept(const LbDev& D) {
  __shared__ double red[33];
  const int s = blockIdx.y, a = D.action(s);
  if (a != ACT_ACC_T && a != ACT_ACC_B) return;
  const double* xs = a == ACT_ACC_T ? D.t(s) : D.b(s);
  const double* outs = a == ACT_ACC_T ? D.ot(s) : D.ob(s);
  double* x = D.x(s);
  double* outx = D.ox(s);
  const int head = D.ring[2 * s + 1];
  double* s_out = D.sr(s) + (int64_t)head * D.N;
  double* y_out = D.yr(s) + (int64_t)head * D.N;
  double* g = outx + 1;
  const double* gs = outs + 1;
  double sy = 0.0, ss = 0.0, yy = 0.0, mx = 0.0, sm = 0.0, bad = 0.0;
  LB_FOR(j) {
    const double sj = __dsub_rn(xs[j], x[j]);
    const double yj = __dsub_rn(gs[j], g[j]);
    s_out[j] = sj;
    y_out[j] = yj;
    x[j] = xs[j];
    g[j] = gs[j];
    sy += __dmul_rn(sj, yj);
    ss += __dmul_rn(sj, sj);
    yy += __dmul_rn(yj, yj);
    const double aa = fabs(gs[j]);
    mx = fmax(mx, aa);
    sm += aa;
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
    double* pp = D.pt(s) + blockIdx.x * LB_NP;
    pp[0] = sy;
    pp[1] = ss;
    pp[2] = yy;
    pp[3] = mx;
    pp[4] = sm;
    pp[5] = bad;
  }
  if (!last_block(D.counter + s) || threadIdx.x != 0) return;
  sy = ss = yy = mx = sm = bad = 0.0;
  for (int b = 0; b < (int)gridDim.x; ++b) {
    const double* pp = D.pt(s) + b * LB_NP;
    sy += pp[0];
    ss += pp[1];
    yy += pp[2];
    mx = fmax(mx, pp[3]);
    sm += pp[4];
    bad += pp[5];
  }
  const bool keep = sy > __dmul_rn(__dmul_rn(1e-12, sqrt(ss)), sqrt(yy));
  if (keep) {
    D.sy(s)[head] = sy;
    D.yy(s)[head] = yy;
    D.ring[2 * s + 1] = (head + 1) % (D.m + 1);
    D.ring[2 * s] = min(D.ring[2 * s] + 1, D.m);
  }
  double* st = D.stats(s);
  st[S_GMAX] = bad > 0.0 ? INFINITY : mx;
  st[S_GSUM] = sm;
  st[S_GBAD] = bad;
  st[S_KEEP] = keep ? 1.0 : 0.0;
  st[S_F] = outx[0];
}
__global__ void k_lbb_accept(LbDev D) {
  pdl_enter();   // chained under programmatic dependent launch: wait, then let the successor launch
  lbb_accept(D);
}


// Two-loop recursion (optimize.py:149-168) in one CTA per run, then the descent check and the
// initial step (optimize.py:307-322).  When the window fits (stage != 0), g and the (s, y)
// window are staged in shared memory first so the 2m+1 dependent passes run at smem latency.
__device__ __forceinline__ void lbb_direction(const LbDev& D, int stage) {
  extern __shared__ double sm[];
  __shared__ double red[33];
  __shared__ double alpha_s[65];
  const int run = blockIdx.y, act = D.action(run);
  if (act != ACT_ACC_T && act != ACT_ACC_B && act != ACT_INIT) return;
  const int64_t N = D.N;
  const int m = D.m;
  int* ring = D.ring + 2 * run;
  const double* sy_h = D.sy(run);
  const double* yy_h = D.yy(run);
  const double* S = D.sr(run);
  const double* Y = D.yr(run);
  double* P = D.p(run);
  double* st = D.stats(run);
  const int count = ring[0], head = ring[1];
  const int M1 = m + 1;
  auto slot = [&](int i) { return (head - count + i + 2 * M1) % M1; };  // i = 0 oldest
  double* q = stage ? sm : P;
  const double* g = D.ox(run) + 1;
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
    double acc = 0.0;
    {
      const double* Si = Sv(count - 1);
      for (int64_t j = threadIdx.x; j < N; j += blockDim.x) {
        const double qj = g[j];
        q[j] = qj;
        acc += __dmul_rn(Si[j], qj);
      }
    }
    // loop 1, newest -> oldest: alpha_i = rho_i * (s_i . q); q -= alpha_i * y_i
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
  if (threadIdx.x == 0) {
    if (reset) ring[0] = 0;
    st[S_PG] = pg;
    st[S_SLOPE0] = slope0;
    st[S_A0] = a0;
    st[S_RESET] = reset ? 1.0 : 0.0;
    D.a0[run] = a0;
  }
}
__global__ void __launch_bounds__(LB_DIR_T) k_lbb_direction(LbDev D, int stage) {
  pdl_enter();   // chained under programmatic dependent launch: wait, then let the successor launch
  lbb_direction(D, stage);
}


// trial point xa = x + a * p (optimize.py:187); phase 0 of INIT: xa = x (evaluate x0).
// Also scatters the trial into the batched K1 layout when k > 1.
__device__ __forceinline__ void lbb_trial(const LbDev& D, int init_phase0) {
  const int s = blockIdx.y, act = D.action(s);
  const double* x = D.x(s);
  const double* p = D.p(s);
  double* t = D.t(s);
  const bool copy = act == ACT_IDLE || (act == ACT_INIT && init_phase0);
  const double a = act == ACT_PROBE ? D.ah[s] : D.a0[s];
  const int64_t nr = D.n * D.r, R = (int64_t)D.k * D.r;
  LB_FOR(j) {
    const double v = copy ? x[j] : __dadd_rn(x[j], __dmul_rn(a, p[j]));
    t[j] = v;
    if (D.Xb) {
      if (j < D.r)
        D.Xb[(int64_t)s * D.r + j] = v;
      else
        D.Xb[R + (int64_t)s * nr + (j - D.r)] = v;
    }
  }
}
__global__ void k_lbb_trial(LbDev D, int init_phase0) {
  pdl_enter();   // chained under programmatic dependent launch: wait, then let the successor launch
  lbb_trial(D, init_phase0);
}


// Small problems (one block per run: N <= LB_SMALL_N = LB_T): the round's prologue -- pull the host's
// actions and steps, save, accept, two-loop direction, trial point -- as ONE kernel instead of
// five launches; the phases are the bodies above, separated by block barriers (one block per
// run, so every "last block" is this block and global writes are visible after the barrier).
__global__ void __launch_bounds__(LB_T) k_lbb_round_small(LbDev D, const int* __restrict__ h_act,
                                                          const double* __restrict__ h_a,
                                                          int* __restrict__ d_act,
                                                          double* __restrict__ d_a, int stage) {
  pdl_enter();
  const int s = blockIdx.y;
  if (threadIdx.x == 0) {
    d_act[s] = h_act[s];
    d_a[s] = h_a[s];
  }
  __syncthreads();
  lbb_save(D);
  __syncthreads();
  lbb_accept(D);
  __syncthreads();
  lbb_direction(D, stage);
  __syncthreads();
  lbb_trial(D, 0);
}

// ga . p and the finiteness of the trial point, finished by the run's last block
__global__ void k_lbb_probe_stats(LbDev D) {
  pdl_enter();   // chained under programmatic dependent launch: wait, then let the successor launch
  __shared__ double red[33];
  const int s = blockIdx.y, act = D.action(s);
  if (act == ACT_IDLE) return;
  const double* xt = D.t(s);
  const double* ga = D.ot(s) + 1;
  const double* P = D.p(s);
  double dp = 0.0, bad = 0.0;
  LB_FOR(j) {
    dp += __dmul_rn(ga[j], P[j]);
    bad += isfinite(xt[j]) ? 0.0 : 1.0;
  }
  dp = block_sum(dp, red);
  bad = block_sum(bad, red);
  double* pp = D.pt(s) + blockIdx.x * LB_NP;
  if (threadIdx.x == 0) {
    pp[0] = dp;
    pp[1] = bad;
  }
  if (!last_block(D.counter + s) || threadIdx.x != 0) return;
  dp = 0.0;
  bad = 0.0;
  for (int b = 0; b < (int)gridDim.x; ++b) {
    dp += D.pt(s)[b * LB_NP + 0];
    bad += D.pt(s)[b * LB_NP + 1];
  }
  double* st = D.stats(s);
  st[S_FA] = D.ot(s)[0];
  st[S_DA] = dp;
  st[S_XBAD] = bad;
  // the whole record of this run, straight into mapped host memory (no D2H copy node)
  double* h = D.st_host + (int64_t)s * S_COUNT;
  for (int i = 0; i < S_COUNT; ++i) h[i] = st[i];
  __threadfence_system();   // the record before the count that announces it
  const unsigned long long v = D.seq_dev[s] + 1;
  D.seq_dev[s] = v;
  *reinterpret_cast<volatile unsigned long long*>(D.seq_host + s) = v;
}

// actions and host-chosen steps of the round, pulled from mapped host memory by one tiny kernel
__global__ void k_lbb_pull(const int* __restrict__ h_act, const double* __restrict__ h_a,
                           int* __restrict__ d_act, double* __restrict__ d_a, int k) {
  pdl_enter();   // chained under programmatic dependent launch: wait, then let the successor launch
  for (int s = threadIdx.x; s < k; s += blockDim.x) {
    d_act[s] = h_act[s];
    d_a[s] = h_a[s];
  }
}

// ------------------------------------------------------------------------------------------
// host side

// The reference's strong-Wolfe search (optimize.py:179-252) as a resumable state machine: the
// caller feeds one probe result at a time and gets the next step or the outcome.  Decisions and
// their order are exactly those of the loop form.
struct Wolfe {
  enum { PROBE = 0, DONE_T = 1, DONE_B = 2, FAIL = 3 };
  struct Pt {
    double a, f, d;
  };
  double f0 = 0, slope0 = 0, c1 = 0, c2 = 0;
  int64_t budget = 0, ev = 0, it = 0;
  bool have_best = false, zoom = false;
  double best_f = 0, a = 0;
  Pt prev{}, lo{}, hi{};

  void start(double f0_, double slope0_, double a0, double c1_, double c2_, int64_t budget_) {
    f0 = f0_;
    slope0 = slope0_;
    c1 = c1_;
    c2 = c2_;
    budget = budget_;
    ev = 0;
    it = 0;
    have_best = false;
    zoom = false;
    a = a0;
    prev = Pt{0.0, f0, slope0};
  }

  // optimize.py:171-176
  static bool interp(double a_lo, double f_lo, double d_lo, double a_hi, double f_hi, double* out) {
    const double den = f_hi - f_lo - d_lo * (a_hi - a_lo);
    if (den == 0 || !std::isfinite(den)) return false;
    const double cnd = a_lo - 0.5 * d_lo * ((a_hi - a_lo) * (a_hi - a_lo)) / den;
    if (!std::isfinite(cnd)) return false;
    *out = cnd;
    return true;
  }

  int fallback() const { return have_best ? DONE_B : FAIL; }

  int zoom_next(double* a_next) {
    if (ev >= budget) return fallback();
    const double width = hi.a - lo.a;
    double cand = 0.0;
    const bool ok = std::isfinite(hi.f) && interp(lo.a, lo.f, lo.d, hi.a, hi.f, &cand);
    const double lb = lo.a + 0.1 * width, ub = hi.a - 0.1 * width;
    if (!ok || !(std::fmin(lb, ub) <= cand && cand <= std::fmax(lb, ub))) cand = lo.a + 0.5 * width;
    a = cand;
    *a_next = cand;
    return PROBE;
  }

  // Feed the result of the probe at step `a`.  *save: this probe is the new best (keep it).
  int on_probe(double fa, double da_raw, bool* save, double* a_next) {
    ++ev;
    const double da = std::isfinite(fa) ? da_raw : NAN;
    *save = false;
    if (std::isfinite(fa) && fa <= f0 + c1 * a * slope0) {
      if (!have_best || fa < best_f) {
        have_best = true;
        best_f = fa;
        *save = true;
      }
    }
    if (!zoom) {
      const bool bad = !std::isfinite(fa) || fa > f0 + c1 * a * slope0 ||
                       (prev.a > 0.0 && fa >= prev.f);
      if (bad) {
        lo = prev;
        hi = Pt{a, fa, da};
        zoom = true;
        return zoom_next(a_next);
      }
      if (std::fabs(da) <= -c2 * slope0) return DONE_T;
      if (da >= 0.0) {
        lo = Pt{a, fa, da};
        hi = prev;
        zoom = true;
        return zoom_next(a_next);
      }
      prev = Pt{a, fa, da};
      a = std::fmin(2.0 * a, 1e20);
      ++it;
      if (it < budget) {
        *a_next = a;
        return PROBE;
      }
      return fallback();
    }
    const double cand = a;
    if (!std::isfinite(fa) || fa > f0 + c1 * cand * slope0 || fa >= lo.f) {
      hi = Pt{cand, fa, da};
    } else {
      if (std::fabs(da) <= -c2 * slope0) return DONE_T;
      if (da * (hi.a - lo.a) >= 0.0) hi = lo;
      lo = Pt{cand, fa, da};
    }
    if (std::fabs(hi.a - lo.a) < 1e-16 * std::fmax(1.0, std::fabs(lo.a))) return fallback();
    return zoom_next(a_next);
  }
};

// Workspace + graphs for (k, d, r, mode, memory, alpha); cached on the context between solves.
struct LbEngine {
  mcp_ctx* c = nullptr;
  int k = 1, d = 0, r = 0, mode = 0, m = 0;
  double alpha = 0.0;
  int64_t n = 0, N = 0;
  int nb = 1;
  int dir_threads = LB_DIR_T;
  bool small = false;   // N <= LB_SMALL_N: one block per run, fused round prologue
  size_t dir_smem = 0;
  EvalPlan pl;   // k == 1: the single evaluation; k > 1: the shared pass over k r columns
  std::vector<void*> dev;
  LbDev D{};
  double* Ywb = nullptr;   // [Y (n x k r) ; w (k r)] of the shared pass
  int* h_act = nullptr;    // pinned
  double* h_a = nullptr;   // pinned
  double* h_st = nullptr;  // pinned, k x S_COUNT
  double* h_x = nullptr;   // pinned, k x N
  int* d_act = nullptr;
  unsigned long long* h_seq = nullptr;        // pinned, k
  std::vector<unsigned long long> expected;   // records announced so far, per run
  GraphEntry g_init, g_round;

  ~LbEngine() {
    for (GraphEntry* g : {&g_init, &g_round}) {
      if (g->exec) cudaGraphExecDestroy(g->exec);
      if (g->graph) cudaGraphDestroy(g->graph);
    }
    for (void* p : dev) cudaFree(p);
    for (void* p : {(void*)h_act, (void*)h_a, (void*)h_st, (void*)h_x, (void*)h_seq})
      if (p) cudaFreeHost(p);
  }

  bool matches(int k_, int d_, int r_, int mode_, int m_, double alpha_) const {
    return k == k_ && d == d_ && r == r_ && mode == mode_ && m == m_ && n == c->n &&
           std::memcmp(&alpha, &alpha_, sizeof(double)) == 0;
  }

  template <typename T>
  int alloc(T*& p, size_t elems) {
    void* q = nullptr;
    CUDA_TRY(c, cudaMalloc(&q, sizeof(T) * (elems ? elems : 1)));
    dev.push_back(q);
    p = (T*)q;
    return MCP_OK;
  }

  // f+grad of every run's trial point T -> OT
  int enqueue_fg() {
    cudaStream_t s = c->stream;
    if (k == 1) return enqueue_fg_full(c, pl, D.T, nullptr, alpha, D.OT, s);
    int rc = enqueue_partial(c, pl, D.Xb, Ywb, s);
    if (rc) return rc;
    const int64_t R = (int64_t)k * r;
    return enqueue_tails_batched(c, d, r, k, D.T, N, Ywb, Ywb + n * R, alpha, D.OT, N + 1, s);
  }

  int enqueue_round_tail() {   // direction (for ACC / INIT runs) -> trial -> fg -> probe stats
    cudaStream_t s = c->stream;
    CUDA_TRY(c, launch_pdl(k_lbb_direction, dim3(1, k), dim3(dir_threads), dir_smem, s, D, dir_smem ? 1 : 0));
    CUDA_TRY(c, launch_pdl(k_lbb_trial, dim3(nb, k), dim3(LB_T), 0, s, D, 0));
    int rc = enqueue_fg();
    if (rc) return rc;
    CUDA_TRY(c, launch_pdl(k_lbb_probe_stats, dim3(nb, k), dim3(LB_T), 0, s, D));
    CUDA_TRY(c, cudaGetLastError());
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

  // Launch a round and wait for the records of its active runs.  The probe kernel stores each
  // run's count into mapped host memory after the record, so the host polls those words (a PCIe
  // write away from the kernel) instead of paying a stream synchronisation per evaluation.
  int replay(GraphEntry& ge) {
    CUDA_TRY(c, cudaGraphLaunch(ge.exec, c->stream));
    if (!MCP_CFG_LBFGS_POLL) {
      CUDA_TRY(c, cudaStreamSynchronize(c->stream));
      for (int s = 0; s < k; ++s)
        if ((h_act[s] & 7) != ACT_IDLE) ++expected[s];
      return MCP_OK;
    }
    for (int s = 0; s < k; ++s) {
      if ((h_act[s] & 7) == ACT_IDLE) continue;
      const unsigned long long want = ++expected[s];
      volatile unsigned long long* w = h_seq + s;
      unsigned spins = 0;
      const auto t0 = std::chrono::steady_clock::now();
      while (*w < want) {
        if ((++spins & 0xffu) == 0 &&
            std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(250)) {
          // 250 us of polling: a long evaluation (or a fault).  Stop burning the core: wait for
          // the stream the ordinary way; its status also reports a failed round.
          const cudaError_t e = cudaStreamSynchronize(c->stream);
          if (e != cudaSuccess || *w < want) {
            // keep the cached engine usable: count what actually arrived
            (void)cudaGetLastError();
            for (int q = 0; q < k; ++q) expected[q] = h_seq[q];
            return c->fail(MCP_ERR_CUDA,
                           e != cudaSuccess ? std::string("L-BFGS round: ") + cudaGetErrorString(e)
                                            : std::string("L-BFGS round finished without its record"));
          }
        }
      }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    return MCP_OK;
  }

  int setup() {
    n = c->n;
    N = r + n * r;
    small = MCP_CFG_LBFGS_FUSED_SMALL && N <= LB_SMALL_N;
    nb = small ? 1 : grid_for(N, LB_T, LB_MAX_BLOCKS);
    dir_threads = N <= 8192 ? 256 : LB_DIR_T;
    const size_t stage_bytes = sizeof(double) * (size_t)N * (2 * (size_t)m + 2);
    dir_smem = stage_bytes <= 192 * 1024 ? stage_bytes : 0;
    int rc;
    if (dir_smem && (!mcp::ensure_dyn_smem((const void*)k_lbb_direction, dir_smem) ||
                     (small && !mcp::ensure_dyn_smem((const void*)k_lbb_round_small, dir_smem))))
      return c->fail(MCP_ERR_CUDA, "cannot raise the two-loop kernel's shared-memory limit");
    const size_t K = (size_t)k, M1 = (size_t)m + 1;
    D.N = N;
    D.m = m;
    D.k = k;
    D.r = r;
    D.n = n;
    D.Xb = nullptr;
    if ((rc = alloc(D.X, K * N)) || (rc = alloc(D.OX, K * (N + 1))) || (rc = alloc(D.T, K * N)) ||
        (rc = alloc(D.OT, K * (N + 1))) || (rc = alloc(D.B, K * N)) ||
        (rc = alloc(D.OB, K * (N + 1))) || (rc = alloc(D.P, K * N)) ||
        (rc = alloc(D.S, K * M1 * N)) || (rc = alloc(D.Y, K * M1 * N)) ||
        (rc = alloc(D.syh, K * M1)) || (rc = alloc(D.yyh, K * M1)) ||
        (rc = alloc(D.part, K * nb * LB_NP)) || (rc = alloc(D.st, K * S_COUNT)) ||
        (rc = alloc(D.a0, K)) || (rc = alloc(D.ah, K)) || (rc = alloc(D.ring, 2 * K)) ||
        (rc = alloc(D.counter, K)) || (rc = alloc(d_act, K)))
      return rc;
    D.act = d_act;
    if (k > 1) {
      const int64_t R = (int64_t)k * r;
      if ((rc = alloc(D.Xb, (size_t)(R + n * R + 1))) || (rc = alloc(Ywb, (size_t)(n * R + R))))
        return rc;
    }
    CUDA_TRY(c, cudaMemset(D.counter, 0, sizeof(unsigned) * K));
    CUDA_TRY(c, cudaMemset(D.P, 0, sizeof(double) * K * N));
    CUDA_TRY(c, cudaMemset(D.a0, 0, sizeof(double) * K));
    CUDA_TRY(c, cudaMallocHost(&h_act, sizeof(int) * K));
    CUDA_TRY(c, cudaMallocHost(&h_a, sizeof(double) * K));
    CUDA_TRY(c, cudaMallocHost(&h_st, sizeof(double) * K * S_COUNT));
    CUDA_TRY(c, cudaMallocHost(&h_x, sizeof(double) * K * N));
    CUDA_TRY(c, cudaMallocHost(&h_seq, sizeof(unsigned long long) * K));
    std::memset(h_seq, 0, sizeof(unsigned long long) * K);
    expected.assign(K, 0ull);
    if ((rc = alloc(D.seq_dev, K))) return rc;
    CUDA_TRY(c, cudaMemset(D.seq_dev, 0, sizeof(unsigned long long) * K));
    D.seq_host = h_seq;
    D.st_host = h_st;   // pinned memory is device-mapped under UVA
    cudaStream_t s = c->stream;
    // init: evaluate x0 (trial = x), statistics, direction, first probe
    if ((rc = capture(g_init, [&]() -> int {
           CUDA_TRY(c, cudaMemcpyAsync(D.X, h_x, sizeof(double) * K * N, cudaMemcpyHostToDevice, s));
           CUDA_TRY(c, cudaMemcpyAsync(d_act, h_act, sizeof(int) * K, cudaMemcpyHostToDevice, s));
           CUDA_TRY(c, launch_pdl(k_lbb_trial, dim3(nb, k), dim3(LB_T), 0, s, D, 1));
           int e = enqueue_fg();
           if (e) return e;
           CUDA_TRY(c, launch_pdl(k_lbb_init_stats, dim3(nb, k), dim3(LB_T), 0, s, D));
           return enqueue_round_tail();
         })))
      return rc;
    if ((rc = capture(g_round, [&]() -> int {
           if (small) {
             CUDA_TRY(c, launch_pdl(k_lbb_round_small, dim3(1, k), dim3(LB_T), dir_smem, s, D,
                                    (const int*)h_act, (const double*)h_a, d_act, D.ah,
                                    dir_smem ? 1 : 0));
             int e = enqueue_fg();
             if (e) return e;
             CUDA_TRY(c, launch_pdl(k_lbb_probe_stats, dim3(nb, k), dim3(LB_T), 0, s, D));
             return MCP_OK;
           }
           CUDA_TRY(c, launch_pdl(k_lbb_pull, dim3(1), dim3(32), 0, s, (const int*)h_act, (const double*)h_a, d_act, D.ah, k));
           CUDA_TRY(c, launch_pdl(k_lbb_save, dim3(nb, k), dim3(LB_T), 0, s, D));
           CUDA_TRY(c, launch_pdl(k_lbb_accept, dim3(nb, k), dim3(LB_T), 0, s, D));
           return enqueue_round_tail();
         })))
      return rc;
    return MCP_OK;
  }
};

// Host-side state of one run
struct RunState {
  enum { ITER = 0, SEARCH = 1, DONE = 2 };
  int phase = ITER;
  Wolfe w;
  double f = 0;
  int64_t n_fg = 0, steps = 0;
  int reason = 1;        // 0 tolerance, 1 iteration cap, 2 line-search failure, 3 error
  std::string error;
  std::vector<double> tf, tt;
};

struct LbOpts {
  int memory;
  double pgtol;
  int64_t max_iters, max_total;
  double c1, c2;
  int64_t max_line_steps;
};

int parse_opts(mcp_ctx* c, const double* opts, LbOpts& o) {
  o.memory = (int)opts[0];
  o.pgtol = opts[1];
  o.max_iters = (int64_t)opts[2];
  o.max_total = (int64_t)opts[3];
  o.c1 = opts[4];
  o.c2 = opts[5];
  o.max_line_steps = (int64_t)opts[6];
  if (!(o.pgtol > 0)) return c->fail(MCP_ERR_ARG, "pgtol must be > 0");
  if (o.memory < 1) return c->fail(MCP_ERR_ARG, "memory must be >= 1");
  if (o.memory > 64) return c->fail(MCP_ERR_ARG, "memory > 64 is not supported by the device solver");
  return MCP_OK;
}

// k lock-step solves from X0 (k x N); per-run results in the output arrays.  A run whose start
// (or a trial point) is not finite ends with reason 3 and a message in errors[s] (the reference
// raises ValueError there).
int run_engine(mcp_ctx* c, int k, int d, int r, double alpha, int mode, const double* X0,
               const LbOpts& o, double* x_out, double* g_out, double* f_out, double* trace_f,
               double* trace_t, int64_t trace_cap, int64_t* info, std::vector<std::string>& errors,
               mcp_iterate_hook hook, void* hook_user) {
  const auto t_start = std::chrono::steady_clock::now();
  auto seconds = [&]() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  };
  // plan first: a buffer growth drops cached graphs (and the cached workspace with them)
  EvalPlan pl;
  int rc = plan_eval(c, d, k * r, mode, pl);
  if (rc) return rc;
  LbEngine* ws = (LbEngine*)c->lbfgs_ws;
  if (!ws || !ws->matches(k, d, r, mode, o.memory, alpha)) {
    if (ws) {
      c->lbfgs_ws_free(ws);
      c->lbfgs_ws = nullptr;
    }
    ws = new LbEngine();
    ws->c = c;
    ws->k = k;
    ws->d = d;
    ws->r = r;
    ws->mode = mode;
    ws->m = o.memory;
    ws->alpha = alpha;
    ws->pl = pl;
    if ((rc = ws->setup())) {
      delete ws;
      return rc;
    }
    c->lbfgs_ws = ws;
    c->lbfgs_ws_free = [](void* p) { delete (LbEngine*)p; };
  }
  LbEngine& E = *ws;
  const int64_t N = E.N;
  std::vector<RunState> R(k);
  errors.assign(k, std::string());
  std::memcpy(E.h_x, X0, sizeof(double) * (size_t)k * N);
  for (int s = 0; s < k; ++s) {
    E.h_act[s] = ACT_INIT;
    for (int64_t j = 0; j < N; ++j)
      if (!std::isfinite(X0[(int64_t)s * N + j])) {
        R[s].phase = RunState::DONE;
        R[s].reason = 3;
        R[s].error = "model variables and alpha must be finite";
        E.h_act[s] = ACT_IDLE;
        for (int64_t jj = 0; jj < N; ++jj) E.h_x[(int64_t)s * N + jj] = 0.0;   // keep the pass finite
        break;
      }
  }
  if ((rc = E.replay(E.g_init))) return rc;
  auto push_trace = [&](RunState& st, double fv) {
    st.tf.push_back(fv);
    st.tt.push_back(seconds());
  };
  auto call_hook = [&](int s) -> int {
    if (!hook) return MCP_OK;
    CUDA_TRY(c, cudaMemcpyAsync(E.h_x, E.D.X + (int64_t)s * N, sizeof(double) * N,
                                cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    hook(E.h_x, N, hook_user);
    return MCP_OK;
  };
  for (int s = 0; s < k; ++s) {
    RunState& st = R[s];
    if (st.phase == RunState::DONE) continue;
    const double* h = E.h_st + (int64_t)s * S_COUNT;
    st.n_fg = 1;
    if (!std::isfinite(h[S_F]) || h[S_GBAD] > 0.0) {
      st.phase = RunState::DONE;
      st.reason = 3;
      st.error = "objective is not finite at the starting point";
      continue;
    }
    st.f = h[S_F];
    push_trace(st, st.f);
    if ((rc = call_hook(s))) return rc;
  }
  // ---- lock-step rounds ----
  while (true) {
    bool any = false;
    for (int s = 0; s < k; ++s) {
      RunState& st = R[s];
      const double* h = E.h_st + (int64_t)s * S_COUNT;
      int act = ACT_IDLE;
      double a_next = 0.0;
      if (st.phase == RunState::ITER) {
        // an accepted (or the initial) point: stopping tests (optimize.py:296-301), then the
        // line search, whose first probe (at a0) this round already evaluated
        if (h[S_GMAX] <= o.pgtol) {
          st.phase = RunState::DONE;
          st.reason = 0;
        } else if (st.steps >= o.max_iters || st.n_fg >= o.max_total) {
          st.phase = RunState::DONE;
          st.reason = 1;
        } else {
          const int64_t budget = std::min<int64_t>(o.max_line_steps, o.max_total - st.n_fg);
          st.w.start(st.f, h[S_SLOPE0], h[S_A0], o.c1, o.c2, budget);
          if (budget <= 0) {
            st.phase = RunState::DONE;
            st.reason = st.n_fg >= o.max_total ? 1 : 2;
          } else {
            st.phase = RunState::SEARCH;
          }
        }
      }
      if (st.phase == RunState::SEARCH) {
        if (h[S_XBAD] > 0.0) {
          st.phase = RunState::DONE;
          st.reason = 3;
          st.error = "model variables and alpha must be finite";
        } else {
          bool save = false;
          const int out = st.w.on_probe(h[S_FA], h[S_DA], &save, &a_next);
          if (out == Wolfe::PROBE) {
            act = ACT_PROBE | (save ? ACT_SAVE : 0);
          } else {
            st.n_fg += st.w.ev;
            if (out == Wolfe::FAIL) {
              st.phase = RunState::DONE;
              st.reason = st.n_fg >= o.max_total ? 1 : 2;
            } else {
              act = (out == Wolfe::DONE_T ? ACT_ACC_T : ACT_ACC_B) | (save ? ACT_SAVE : 0);
              st.phase = RunState::ITER;
              ++st.steps;
            }
          }
        }
      }
      E.h_act[s] = act;
      E.h_a[s] = a_next;
      if ((act & 7) != ACT_IDLE) any = true;
    }
    if (!any) break;
    if ((rc = E.replay(E.g_round))) return rc;
    for (int s = 0; s < k; ++s) {
      const int a = E.h_act[s] & 7;
      if (a == ACT_ACC_T || a == ACT_ACC_B) {
        RunState& st = R[s];
        st.f = E.h_st[(int64_t)s * S_COUNT + S_F];
        push_trace(st, st.f);
        if ((rc = call_hook(s))) return rc;
      }
    }
  }
  // final states
  CUDA_TRY(c, cudaMemcpy2DAsync(x_out, sizeof(double) * N, E.D.X, sizeof(double) * N,
                                sizeof(double) * N, k, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaMemcpy2DAsync(g_out, sizeof(double) * N, E.D.OX + 1, sizeof(double) * (N + 1),
                                sizeof(double) * N, k, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  for (int s = 0; s < k; ++s) {
    RunState& st = R[s];
    f_out[s] = st.f;
    const int64_t nt = (int64_t)st.tf.size();
    for (int64_t i = 0; i < nt && i < trace_cap; ++i) {
      if (trace_f) trace_f[(int64_t)s * trace_cap + i] = st.tf[i];
      if (trace_t) trace_t[(int64_t)s * trace_cap + i] = st.tt[i];
    }
    int64_t* inf = info + 4 * (int64_t)s;
    inf[0] = st.n_fg;
    inf[1] = st.steps;
    inf[2] = st.reason;
    inf[3] = std::min(nt, trace_cap);
    errors[s] = st.error;
  }
  return MCP_OK;
}

thread_local std::string g_batch_errors;

}  // namespace

extern "C" int mcp_lbfgs(mcp_ctx* c, int d, int r, double alpha, int mode, const double* x0,
                         const double* opts, double* x_out, double* g_out, double* f_out,
                         double* trace_f, double* trace_t, int64_t trace_cap, int64_t* info,
                         mcp_iterate_hook hook, void* hook_user) {
  if (!c) return MCP_ERR_ARG;
  Guard gd(c);
  MCP_NVTX("mcp_lbfgs");
  if (!x0 || !opts || !x_out || !g_out || !f_out || !info)
    return c->fail(MCP_ERR_ARG, "NULL argument");
  if (!std::isfinite(alpha)) return c->fail(MCP_ERR_ARG, "model variables and alpha must be finite");
  if (!c->loaded) return c->fail(MCP_ERR_STATE, "no observation set loaded (call mcp_load_obs)");
  LbOpts o;
  int rc = parse_opts(c, opts, o);
  if (rc) return rc;
  std::vector<std::string> errors;
  rc = run_engine(c, 1, d, r, alpha, mode, x0, o, x_out, g_out, f_out, trace_f, trace_t,
                  trace_cap, info, errors, hook, hook_user);
  if (rc) return rc;
  if (info[2] == 3) return c->fail(MCP_ERR_ARG, errors[0]);
  return MCP_OK;
}

extern "C" int mcp_lbfgs_batch(mcp_ctx* c, int k, int d, int r, double alpha, int mode,
                               const double* X0, const double* opts, double* X_out,
                               double* G_out, double* F_out, double* trace_f, double* trace_t,
                               int64_t trace_cap, int64_t* info) {
  if (!c) return MCP_ERR_ARG;
  Guard gd(c);
  MCP_NVTX("mcp_lbfgs_batch");
  if (!X0 || !opts || !X_out || !G_out || !F_out || !info)
    return c->fail(MCP_ERR_ARG, "NULL argument");
  if (k < 1) return c->fail(MCP_ERR_ARG, "number of starts must be >= 1");
  if (!std::isfinite(alpha)) return c->fail(MCP_ERR_ARG, "model variables and alpha must be finite");
  if (!c->loaded) return c->fail(MCP_ERR_STATE, "no observation set loaded (call mcp_load_obs)");
  LbOpts o;
  int rc = parse_opts(c, opts, o);
  if (rc) return rc;
  std::vector<std::string> errors;
  rc = run_engine(c, k, d, r, alpha, mode, X0, o, X_out, G_out, F_out, trace_f, trace_t, trace_cap,
                  info, errors, nullptr, nullptr);
  if (rc) return rc;
  g_batch_errors.clear();
  for (int s = 0; s < k; ++s)
    if (!errors[s].empty()) g_batch_errors += "run " + std::to_string(s) + ": " + errors[s] + "\n";
  return MCP_OK;
}

extern "C" const char* mcp_lbfgs_batch_errors(void) { return g_batch_errors.c_str(); }
