// DMMA.8x8x4 issue model: per-SM throughput with W warps per SM sub-partition, each running C
// independent accumulator chains (plus optional DFMA interleave) -- how much ILP the FP64 pipe
// needs to saturate.
#include <cstdio>
#include <cuda_runtime.h>
template <int C, int F>
__global__ void ilp(double* out, int iters, double a, double b) {
  double acc[C][2], fa[F > 0 ? F : 1];
#pragma unroll
  for (int c = 0; c < C; ++c) acc[c][0] = acc[c][1] = threadIdx.x;
#pragma unroll
  for (int f = 0; f < (F > 0 ? F : 1); ++f) fa[f] = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < C; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a), "d"(b));
#pragma unroll
    for (int f = 0; f < F; ++f) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(fa[f]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += acc[c][0] + acc[c][1];
#pragma unroll
  for (int f = 0; f < (F > 0 ? F : 1); ++f) s += fa[f];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int C, int F>
void run(int warps_per_sm) {
  double* o;
  cudaMalloc(&o, sizeof(double) * 148 * 1024);
  const int iters = 20000;
  ilp<C, F><<<148, 32 * warps_per_sm>>>(o, 10, 1.0000001, 1e-9);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  ilp<C, F><<<148, 32 * warps_per_sm>>>(o, iters, 1.0000001, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double fl = 148.0 * warps_per_sm * iters * (C * 512.0 + F * 64.0);
  printf("warps/SM %2d chains %d dfma %d: %.2f TFLOP/s\n", warps_per_sm, C, F, fl / ms / 1e9);
  cudaFree(o);
}
int main() {
  for (int w : {4, 8, 12, 16}) {
    run<1, 0>(w);
    run<2, 0>(w);
    run<4, 0>(w);
    run<2, 4>(w);
    run<13, 26>(w);
  }
  return 0;
}
