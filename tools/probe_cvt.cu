// FP64 pipe cost of fp32 -> fp64 conversions next to DMMA.8x8x4: W warps per SM, 4 independent
// DMMA chains per warp, K cvt.f64.f32 per 4 DMMAs (K1W's GEMM1 issues 2, GEMM2 1), plus the
// integer-ALU alternative (exponent rebias, exact for normal fp32 and zero).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double cvt_int(float f) {
  const unsigned u = __float_as_uint(f);
  const unsigned mag = u & 0x7fffffffu;
  const unsigned hi = (u & 0x80000000u) | (mag ? (mag >> 3) + 0x38000000u : 0u);
  return __hiloint2double((int)hi, (int)(u << 29));
}
template <int K, int MODE>
__global__ void mix(double* out, int iters, float s) {
  double acc[4][2];
#pragma unroll
  for (int c = 0; c < 4; ++c) acc[c][0] = acc[c][1] = threadIdx.x;
  float f = s + threadIdx.x;
  double a = 1.0000001, b = 1e-9;
  for (int i = 0; i < iters; ++i) {
    double v[K > 0 ? K : 1];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const float fk = __int_as_float(__float_as_int(f) ^ (k + (i & 1)));
      if (MODE == 0) asm volatile("cvt.f64.f32 %0, %1;" : "=d"(v[k]) : "f"(fk));
      else v[k] = cvt_int(fk);
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const double op = K > 0 ? v[c % (K > 0 ? K : 1)] : a;
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(op), "d"(b));
    }
  }
  double sum = a;
#pragma unroll
  for (int c = 0; c < 4; ++c) sum += acc[c][0] + acc[c][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = sum;
}
template <int K, int MODE>
void run(int warps) {
  double* o;
  cudaMalloc(&o, sizeof(double) * 148 * 1024);
  const int iters = 20000;
  mix<K, MODE><<<148, 32 * warps>>>(o, 10, 1.5f);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mix<K, MODE><<<148, 32 * warps>>>(o, iters, 1.5f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double fl = 148.0 * warps * iters * 4 * 512.0;
  printf("warps/SM %2d cvt/4dmma %d mode %s: %.2f TFLOP/s (DMMA only)\n", warps, K,
         MODE ? "int" : "f2f", fl / ms / 1e9);
  cudaFree(o);
}
int main() {
  for (int w : {8, 12}) {
    run<0, 0>(w);
    run<1, 0>(w);
    run<2, 0>(w);
    run<4, 0>(w);
    run<2, 1>(w);
    run<4, 1>(w);
  }
  return 0;
}
