// Shared device helpers for the momentcp B200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace mcp {

// ---------------------------------------------------------------------------------------------
// FP64 tensor-core MMA: D(8x8) += A(8x4, row) * B(4x8, col).  On sm_100a this is one
// DMMA.8x8x4 (the only FP64 tensor path on B200; tcgen05 has no f64 kind).
// Fragment ownership, lane = 4*g + t:
//   A: a = A[g][t]      B: b = B[t][g]      C/D: c[e] = C[g][2t+e], e in {0,1}
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// Ampere-style async copy of 16 bytes global -> shared; src_bytes==0 zero-fills the 16 bytes.
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src, int src_bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem_src),
               "r"(src_bytes));
}
// The same with an L2 cache-eviction policy (createpolicy), e.g. evict_first for streamed data.
__device__ __forceinline__ void cp_async16_hint(void* smem_dst, const void* gmem_src, int src_bytes,
                                                uint64_t policy) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;\n" ::"r"(s),
               "l"(gmem_src), "r"(src_bytes), "l"(policy));
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ double2 ld_l2_hint(const double2* p, uint64_t policy) {
  double2 v;
  asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;\n"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p), "l"(policy));
  return v;
}
__device__ __forceinline__ void st_l2_hint(double2* p, double2 v, uint64_t policy) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(p), "d"(v.x),
               "d"(v.y), "l"(policy)
               : "memory");
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Elementwise integer power by left-to-right repeated multiplication, the rounding sequence
// of the reference's _elementwise_power (pkg/src/momentcp/implicit.py:82-91): x, x*x, (x*x)*x...
// k >= 1 (k == 0 is never needed on device: d >= 2 everywhere).
__device__ __forceinline__ double rm_pow(double x, int k) {
  double acc = x;
  for (int i = 1; i < k; ++i) acc *= x;
  return acc;
}

// rm_pow over N values with one (warp-uniform) branch on k instead of one loop per value.
template <int N>
__device__ __forceinline__ void rm_pow_vec(const double (&x)[N], double (&y)[N], int k) {
  switch (k) {
    case 1:
#pragma unroll
      for (int i = 0; i < N; ++i) y[i] = x[i];
      break;
    case 2:
#pragma unroll
      for (int i = 0; i < N; ++i) y[i] = x[i] * x[i];
      break;
    case 3:
#pragma unroll
      for (int i = 0; i < N; ++i) y[i] = (x[i] * x[i]) * x[i];
      break;
    case 4:
#pragma unroll
      for (int i = 0; i < N; ++i) y[i] = ((x[i] * x[i]) * x[i]) * x[i];
      break;
    case 5:
#pragma unroll
      for (int i = 0; i < N; ++i) y[i] = (((x[i] * x[i]) * x[i]) * x[i]) * x[i];
      break;
    default:
#pragma unroll
      for (int i = 0; i < N; ++i) y[i] = rm_pow(x[i], k);
  }
}

template <typename T>
__device__ __forceinline__ double to_f64(T v) {
  return static_cast<double>(v);
}

__host__ __device__ constexpr int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ constexpr int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

}  // namespace mcp
