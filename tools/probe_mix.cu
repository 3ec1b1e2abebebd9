// Does DFMA share the FP64 pipe with DMMA on B200? Interleave both and time.
#include <cstdio>
#include <cuda_runtime.h>

template <int DM, int DF>
__global__ void mix_kernel(double* out, int iters, double a0, double b0) {
  double a = a0 + threadIdx.x * 1e-9, b = b0 - threadIdx.x * 1e-9;
  double c[DM > 0 ? DM : 1][2];
  double f[DF > 0 ? DF : 1];
#pragma unroll
  for (int k = 0; k < (DM > 0 ? DM : 1); ++k) { c[k][0] = 0; c[k][1] = 0; }
#pragma unroll
  for (int k = 0; k < (DF > 0 ? DF : 1); ++k) f[k] = k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < DM; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
#pragma unroll
    for (int k = 0; k < DF; ++k) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(f[k]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < (DM > 0 ? DM : 1); ++k) s += c[k][0] + c[k][1];
#pragma unroll
  for (int k = 0; k < (DF > 0 ? DF : 1); ++k) s += f[k];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int DM, int DF>
void run(int sms, double* out, int iters) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int grid = sms * 2, block = 256;
  mix_kernel<DM, DF><<<grid, block>>>(out, iters, 1.0000001, 1e-7);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    mix_kernel<DM, DF><<<grid, block>>>(out, iters, 1.0000001, 1e-7);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double warps = (double)grid * block / 32;
  double fl_dm = 512.0 * DM * iters * warps;
  double fl_df = 2.0 * DF * iters * warps * 32;
  printf("DMMA x%d + DFMA x%d: %.3f ms  dmma %.2f TF  dfma %.2f TF  total %.2f TF\n", DM, DF, best,
         fl_dm / best / 1e9, fl_df / best / 1e9, (fl_dm + fl_df) / best / 1e9);
}

int main() {
  cudaDeviceProp prop; cudaGetDeviceProperties(&prop, 0);
  double* out; cudaMalloc(&out, 1 << 20);
  int it = 4000;
  run<4, 0>(prop.multiProcessorCount, out, it);
  run<0, 8>(prop.multiProcessorCount, out, it);
  run<4, 4>(prop.multiProcessorCount, out, it);
  run<4, 8>(prop.multiProcessorCount, out, it);
  run<4, 16>(prop.multiProcessorCount, out, it);
  run<2, 16>(prop.multiProcessorCount, out, it);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
