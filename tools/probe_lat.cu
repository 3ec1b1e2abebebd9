// Latency probe: dependent DMMA.8x8x4 / DFMA chains on one warp (clock64 cycles per op).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* cyc, int iters, double a, double b) {
  double c0 = threadIdx.x, c1 = 1.0, f = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  long long t1 = clock64();
  for (int i = 0; i < iters; ++i) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(f) : "d"(a), "d"(b));
  long long t2 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; }
  out[threadIdx.x] = c0 + c1 + f;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 4096); cudaMallocManaged(&c, 64);
  lat<<<1, 32>>>(o, c, 1000, 1.0000001, 1e-9); cudaDeviceSynchronize();
  lat<<<1, 32>>>(o, c, 1000, 1.0000001, 1e-9); cudaDeviceSynchronize();
  printf("DMMA dependent latency %.1f cycles, DFMA dependent latency %.1f cycles\n", c[0] / 1000.0, c[1] / 1000.0);
  return 0;
}
