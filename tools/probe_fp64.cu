// FP64 pipe probe for B200 (sm_100a): DFMA vs DMMA.8x8x4 throughput.
// Measures the FP64 roofline denominator the bench reports against.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int CHAINS>
__global__ void dmma_kernel(double* out, int iters, double a0, double b0) {
  double a = a0 + threadIdx.x * 1e-9, b = b0 - threadIdx.x * 1e-9;
  double c[CHAINS][2];
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) { c[k][0] = 0; c[k][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < CHAINS; ++k) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <typename K>
float time_kernel(K kern, int grid, int block, double* out, int iters) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<grid, block>>>(out, iters, 1.0000001, 1e-7);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    kern<<<grid, block>>>(out, iters, 1.0000001, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int dev = 0; cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  int sms = prop.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, 1 << 20));
  printf("device %s sms %d\n", prop.name, sms);
  const int iters = 20000;
  for (int blocks_per_sm : {1, 2, 4, 8}) {
    int block = 256, grid = sms * blocks_per_sm;
    float ms = time_kernel(dfma_kernel<8>, grid, block, out, iters);
    double flops = 2.0 * 8 * iters * (double)grid * block;
    printf("DFMA  chains=8 grid=%d block=%d: %.3f ms  %.2f TFLOP/s\n", grid, block, ms, flops / ms / 1e9);
  }
  for (int blocks_per_sm : {1, 2, 4, 8}) {
    int block = 256, grid = sms * blocks_per_sm;
    float ms = time_kernel(dmma_kernel<4>, grid, block, out, iters / 4);
    double flops = 2.0 * 256 * 4 * (iters / 4) * (double)grid * (block / 32);
    printf("DMMA  chains=4 grid=%d block=%d: %.3f ms  %.2f TFLOP/s\n", grid, block, ms, flops / ms / 1e9);
  }
  for (int blocks_per_sm : {1, 2, 4}) {
    int block = 256, grid = sms * blocks_per_sm;
    float ms = time_kernel(dmma_kernel<8>, grid, block, out, iters / 8);
    double flops = 2.0 * 256 * 8 * (iters / 8) * (double)grid * (block / 32);
    printf("DMMA  chains=8 grid=%d block=%d: %.3f ms  %.2f TFLOP/s\n", grid, block, ms, flops / ms / 1e9);
  }
  CK(cudaGetLastError());
  return 0;
}
