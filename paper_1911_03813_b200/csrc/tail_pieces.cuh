// Reduce-block geometry shared by K3 / K3F and the Y-independent tail pieces (G, C, u, M) that
// the finishing kernels (K3F, the peer reduce) form in-block.  Device inline functions only, so
// several translation units may include it.
#pragma once

#include "mcp_common.cuh"

namespace mcp {

constexpr int K3_X = 8, K3_Y = 128, K3_T = K3_X * K3_Y;
constexpr int K3W_X = 32, K3W_Y = K3_T / K3W_X;
constexpr int K3F_MAXR = 32;   // largest r whose G, C a finishing block keeps in shared memory

// Optional publication of the reduced [Y | w] to the peers (multi-GPU exchange, csrc/peer.cu):
// after every block has written its outputs, the last block to finish (ticket) fences at
// system scope and release-stores `epoch` into flags[k][rank] for every rank k.
struct K3Signal {
  int64_t* const* flags = nullptr;   // device array of `world` flag arrays (peer-mapped)
  unsigned* ticket = nullptr;        // zero-initialised; reset by the last block
  int rank = 0, world = 0;
  int64_t epoch = 0;
};


// Tail pieces inside one block, from x = [lam ; vec_F(A)] alone (implicit.py:143-151), in the
// expression order of k1p_tail_pre / k_tail_gram / k_tail_vec so every path stays bitwise equal:
// G = A^T A (warp per upper-triangle entry: lane-strided products, fixed butterfly, mirrored),
// C = G^(d-1) by repeated multiplication (implicit.py:82-91); then per entry
// u_j = sum_k (G_jk C_jk) lam_k and M_ij = sum_k (A_ik lam_k) C_kj.
__device__ __forceinline__ void tail_gc_block(const double* __restrict__ x, int n, int r, int d,
                                              double* sG, double* sC) {
  const double* A = x + r;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int pr = warp; pr < r * r; pr += nw) {
    const int j = pr / r, k = pr % r;
    if (j > k) continue;
    const double* aj = A + (int64_t)j * n;
    const double* ak = A + (int64_t)k * n;
    double s = 0.0;
    for (int i = lane; i < n; i += 32) s += aj[i] * ak[i];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) {
      const double c = rm_pow(s, d - 1);
      sG[j * r + k] = s;
      sG[k * r + j] = s;
      sC[j * r + k] = c;
      sC[k * r + j] = c;
    }
  }
}
__device__ __forceinline__ double tail_u_entry(const double* sG, const double* sC,
                                               const double* __restrict__ lam, int r, int j) {
  double u = 0.0;
  for (int k = 0; k < r; ++k) u += (sG[j * r + k] * sC[j * r + k]) * lam[k];
  return u;
}
__device__ __forceinline__ double tail_m_entry(const double* __restrict__ x, const double* sC,
                                               int n, int r, int i, int j) {
  const double* A = x + r;
  double m = 0.0;
  for (int k = 0; k < r; ++k) m += (A[(int64_t)k * n + i] * x[k]) * sC[k * r + j];
  return m;
}

}  // namespace mcp
