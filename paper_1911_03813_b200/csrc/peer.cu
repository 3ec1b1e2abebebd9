// Cross-GPU exchange of the additive [vec_F(Y) | w] pieces over NVLink peer memory, fused with
// the finish (replaces the NCCL all-reduce + tail of the row-sharded path).
//
// Every rank's partial lives in a symmetric (peer-mapped) buffer, two slots by epoch parity.
//   mcp_peer_signal:          after this rank's partial is complete (stream order), publish
//                             `epoch` into every rank's flag array at index `rank`
//                             (threadfence.system + st.release.sys); mcp_fg_partial_signal_device
//                             does the same from the last block of the partial's reduce (K3);
//   mcp_peer_reduce_finish:   wait until every rank's flag for this epoch is set (ld.acquire.sys,
//                             bounded), sum the W partials in rank order 0..W-1 straight from
//                             peer memory, and finish: for r <= 32 the kernel forms G, C (and
//                             the M, u entries it needs) from x while it waits, so the finish is
//                             elementwise (g_A = -2d (Y - M) o lam, g_lam = -2 (w - u), f);
//                             otherwise the summed piece goes through the regular tail.  Every rank sums in the same order, so all ranks hold
//                             bitwise identical f and gradients.
// Slot reuse is safe with two slots: a rank overwrites slot e % 2 at epoch e + 2 only after
// its own reduce of epoch e + 1 saw every peer's epoch e + 1 flag, i.e. after every peer
// finished reading epoch e.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <string>

#include "ctx.h"
#include "mcp_common.cuh"
#include "tail_pieces.cuh"
#include "pdl.h"

using namespace mcp;
using namespace mcp_internal;

namespace {

constexpr int PR_T = 256;
// A peer whose flag has not arrived after this long (globaltimer ns) is declared lost: the
// kernel sets *err and writes NaN into every output, so a stale or partial sum can never be
// consumed as a result (PeerExchange.step / bench.py check err and raise).
constexpr unsigned long long PR_WAIT_LIMIT_NS = 30ull * 1000000000ull;

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;\n" : "=l"(t));
  return t;
}

__device__ __forceinline__ void st_release_sys(int64_t* p, int64_t v) {
  asm volatile("st.release.sys.global.b64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ int64_t ld_acquire_sys(const int64_t* p) {
  int64_t v;
  asm volatile("ld.acquire.sys.global.b64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double ld_volatile_sys(const double* p) {
  double v;
  asm volatile("ld.relaxed.sys.global.f64 %0, [%1];\n" : "=d"(v) : "l"(p) : "memory");
  return v;
}

__global__ void k_peer_signal(int64_t* const* __restrict__ flags, int rank, int world,
                              int64_t epoch) {
  if (threadIdx.x != 0) return;
  __threadfence_system();
  for (int k = 0; k < world; ++k) st_release_sys(flags[k] + rank, epoch);
}

// blocks 0 .. nb-2: g_A (or summed Y) slices; block nb-1: w, g_lam, f.
// parts[k] = rank k's partial slot for this epoch; err (device) set when a flag never came.
__global__ void k_peer_reduce_finish(const double* const* __restrict__ parts,
                                     const int64_t* __restrict__ my_flags, int world,
                                     int64_t epoch, int n, int r, int d,
                                     const double* __restrict__ x, int light, double alpha,
                                     double* __restrict__ out, double* __restrict__ Yw_sum,
                                     int* __restrict__ err) {
  // PDL: the next evaluation's K1 may start its V-only prologue; the peers' partials (ours
  // included) are ordered by the flags below, not by grid completion
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  __shared__ int ok;
  __shared__ double sG[K3F_MAXR * K3F_MAXR], sC[K3F_MAXR * K3F_MAXR];
  // light (r <= K3F_MAXR): G and C from x alone, while the peers' partials are still coming
  if (light) tail_gc_block(x, n, r, d, sG, sC);
  if (threadIdx.x == 0) {
    ok = 1;
    for (int k = 0; k < world; ++k) {
      const unsigned long long t0 = globaltimer_ns();
      while (ok && ld_acquire_sys(my_flags + k) < epoch) {
        if (globaltimer_ns() - t0 > PR_WAIT_LIMIT_NS) {
          ok = 0;
          atomicExch(err, 1);
          break;
        }
      }
    }
  }
  __syncthreads();
  const bool good = ok != 0;
  const double bad = __longlong_as_double(0x7ff8000000000000ll);   // quiet NaN
  const double* lam = x;
  const int64_t nr = (int64_t)n * r;
  if (blockIdx.x + 1 < gridDim.x) {
    for (int64_t e = blockIdx.x * (int64_t)PR_T + threadIdx.x; e < nr;
         e += (int64_t)(gridDim.x - 1) * PR_T) {
      double y = 0.0;
      for (int k = 0; k < world; ++k) y += ld_volatile_sys(parts[k] + e);
      if (!good) y = bad;
      if (light) {
        const int j = (int)(e / n), i = (int)(e % n);
        const double m = tail_m_entry(x, sC, n, r, i, j);
        out[1 + r + e] = ((-2.0 * d) * (y - m)) * lam[j];
      } else {
        Yw_sum[e] = y;
      }
    }
    return;
  }
  __shared__ double s_w[1024];
  __shared__ double s_u[K3F_MAXR];
  for (int j = threadIdx.x; j < r; j += PR_T) {
    double w = 0.0;
    for (int k = 0; k < world; ++k) w += ld_volatile_sys(parts[k] + nr + j);
    if (!good) w = bad;
    if (light) {
      const double u = tail_u_entry(sG, sC, lam, r, j);
      s_w[j] = w;
      s_u[j] = u;
      out[1 + j] = -2.0 * (w - u);
    } else {
      Yw_sum[nr + j] = w;
    }
  }
  __syncthreads();
  if (light && threadIdx.x == 0) {
    double lu = 0.0, wl = 0.0;
    for (int j = 0; j < r; ++j) lu += lam[j] * s_u[j];
    for (int j = 0; j < r; ++j) wl += s_w[j] * lam[j];
    out[0] = good ? alpha + lu - 2.0 * wl : bad;
  }
}

}  // namespace

extern "C" int mcp_peer_signal(mcp_ctx* c, const void* flag_ptrs, int rank, int world,
                               int64_t epoch, void* stream) {
  if (!c) return MCP_ERR_ARG;
  Guard gd(c);
  if (!flag_ptrs || world < 1 || rank < 0 || rank >= world)
    return c->fail(MCP_ERR_ARG, "bad peer arguments");
  cudaStream_t s = stream ? (cudaStream_t)stream : c->stream;
  k_peer_signal<<<1, 32, 0, s>>>((int64_t* const*)flag_ptrs, rank, world, epoch);
  CUDA_TRY(c, cudaGetLastError());
  return MCP_OK;
}

extern "C" int mcp_peer_reduce_finish(mcp_ctx* c, int d, int r, const double* dx,
                                      const void* part_ptrs, const int64_t* my_flags, int world,
                                      int64_t epoch, double alpha, double* dout, int* derr,
                                      void* stream) {
  if (!c) return MCP_ERR_ARG;
  Guard gd(c);
  MCP_NVTX("mcp_peer_reduce_finish");
  if (!dx || !part_ptrs || !my_flags || !dout || !derr || world < 1)
    return c->fail(MCP_ERR_ARG, "NULL argument");
  if (!c->loaded) return c->fail(MCP_ERR_STATE, "no observation set loaded (call mcp_load_obs)");
  if (r > 1024) return c->fail(MCP_ERR_ARG, "rank > 1024 not supported by the peer reduce");
  cudaStream_t s = stream ? (cudaStream_t)stream : c->stream;
  const int n = (int)c->n;
  const int64_t nr = (int64_t)n * r;
  const bool light = r <= K3F_MAXR;   // tail pieces formed in-kernel
  int rc;
  if (!light) {
    if ((rc = ensure(c, c->dYw, sizeof(double) * (size_t)(nr + r)))) return rc;
    if ((rc = ensure(c, c->dG, sizeof(double) * (size_t)r * r))) return rc;
    if ((rc = ensure(c, c->dC, sizeof(double) * (size_t)r * r))) return rc;
  }
  const int nb = (int)std::min<int64_t>(ceil_div(nr, PR_T), 4 * c->sms) + 1;
  {
    // under PDL it launches while this rank's K3 (which publishes our flag) drains
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)nb);
    cfg.blockDim = dim3(PR_T);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CUDA_TRY(c, cudaLaunchKernelEx(&cfg, k_peer_reduce_finish, (const double* const*)part_ptrs,
                                   my_flags, world, epoch, n, r, d, dx, light ? 1 : 0, alpha,
                                   dout, light ? nullptr : (double*)c->dYw.p, derr));
  }
  CUDA_TRY(c, cudaGetLastError());
  c->last_launches = 1;
  if (!light) {
    return enqueue_finish(c, d, r, dx, (const double*)c->dYw.p, nullptr, alpha, dout, s);
  }
  return MCP_OK;
}
