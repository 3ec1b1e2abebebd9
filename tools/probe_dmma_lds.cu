// DMMA.8x8x4 throughput when the operands come from shared memory: W warps per SM, each step
// loads MA A-fragments (fp64, or fp32 + cvt as the fp32-observation kernels do) and NB
// B-fragments (fp64) with ld.shared, then issues MA x NB DMMAs into MA x NB accumulators.
// PF = 1 issues the next step's loads before this step's DMMAs (explicit one-step prefetch).
// Answers: how many warps per sub-partition and which register tile keep the FP64 pipe full
// for a K1-style inner loop.
#include <cstdio>
#include <cuda_runtime.h>

template <int MA, int NB, int F32A, int PF>
__global__ void __launch_bounds__(512, 1) k(double* out, int iters) {
  extern __shared__ double sm[];   // 8192 doubles
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = 1.0 + 1e-9 * i;
  __syncthreads();
  const unsigned base = (unsigned)__cvta_generic_to_shared(sm);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double acc[MA][NB][2];
#pragma unroll
  for (int i = 0; i < MA; ++i)
#pragma unroll
    for (int j = 0; j < NB; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  double an[MA], bn[NB];
  float fn[MA];
  auto load = [&](int s) {
    const unsigned off = (unsigned)((s * 2 * (MA + NB) + warp * 64) & 127) * 256u + lane * 8u;
#pragma unroll
    for (int i = 0; i < MA; ++i) {
      if (F32A)
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(fn[i]) : "r"(base + off - lane * 4u + i * 512u));
      else
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(an[i]) : "r"(base + off + i * 512u));
    }
#pragma unroll
    for (int j = 0; j < NB; ++j)
      asm volatile("ld.shared.f64 %0, [%1];" : "=d"(bn[j]) : "r"(base + off + 8192u + j * 512u));
  };
  if (PF) load(0);
  for (int s = 0; s < iters; ++s) {
    double a[MA], b[NB];
    if (!PF) load(s);
#pragma unroll
    for (int i = 0; i < MA; ++i) a[i] = F32A ? (double)fn[i] : an[i];
#pragma unroll
    for (int j = 0; j < NB; ++j) b[j] = bn[j];
    if (PF) load(s + 1);
#pragma unroll
    for (int i = 0; i < MA; ++i)
#pragma unroll
      for (int j = 0; j < NB; ++j)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(acc[i][j][0]), "+d"(acc[i][j][1]) : "d"(a[i]), "d"(b[j]));
  }
  double t = 0;
#pragma unroll
  for (int i = 0; i < MA; ++i)
#pragma unroll
    for (int j = 0; j < NB; ++j) t += acc[i][j][0] + acc[i][j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

template <int MA, int NB, int F32A, int PF>
void run(int warps) {
  double* o;
  cudaMalloc(&o, sizeof(double) * 148 * 512);
  const int iters = 40000 / (MA * NB);
  cudaFuncSetAttribute(k<MA, NB, F32A, PF>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  k<MA, NB, F32A, PF><<<148, 32 * warps, 65536>>>(o, 10);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<MA, NB, F32A, PF><<<148, 32 * warps, 65536>>>(o, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double fl = 148.0 * warps * (double)iters * MA * NB * 512.0;
  printf("warps/SM %2d  tile %dx%d  A %s  prefetch %d : %6.2f TFLOP/s  (%.2f loads/DMMA)\n",
         warps, MA, NB, F32A ? "f32+cvt" : "f64", PF, fl / ms / 1e9,
         (double)(MA + NB) / (MA * NB));
  cudaFree(o);
}

template <int MA, int NB>
void sweep() {
  for (int w : {8, 12, 16}) {
    run<MA, NB, 0, 0>(w);
    run<MA, NB, 1, 0>(w);
    run<MA, NB, 1, 1>(w);
  }
}

int main() {
  sweep<1, 4>();
  sweep<2, 2>();
  sweep<2, 4>();
  sweep<4, 4>();
  sweep<4, 2>();
  sweep<1, 2>();
  return 0;
}
