// Streaming-bandwidth probe of the K1S producer structure: one lane issues 1-D TMA bulk copies
// into an S-stage smem ring, W consumer warps wait on `full`, optionally read the stage, and
// release `empty`.  Reports GB/s for several slab sizes / ring depths.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su(b)), "r"(c)); }
__device__ __forceinline__ void mb_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su(b)) : "memory"); }
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su(b)), "r"(n) : "memory"); }
__device__ __forceinline__ bool mb_try(uint64_t* b, uint32_t ph) {
  uint32_t ok; asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(ok) : "r"(su(b)), "r"(ph) : "memory"); return ok; }
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t ph) { long long t0 = clock64(); while (!mb_try(b, ph)) { if (clock64() - t0 > (1ll << 32)) __trap(); } }

__global__ void stream(const char* __restrict__ src, long long nslabs, int slab, int S, int W, int touch, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = (uint64_t*)(sm + (size_t)S * slab);
  uint64_t* empty = full + S;
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { for (int s = 0; s < S; ++s) { mb_init(&full[s], 1); mb_init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  long long mine = (nslabs - blockIdx.x + gridDim.x - 1) / gridDim.x;
  if (warp == W) {
    if (lane == 0) for (long long k = 0; k < mine; ++k) {
      int s = k % S; if (k >= S) mb_wait(&empty[s], (k / S - 1) & 1);
      mb_expect(&full[s], slab);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        :: "r"(su(sm + (size_t)s * slab)), "l"(src + (blockIdx.x + k * gridDim.x) * (long long)slab), "r"(slab), "r"(su(&full[s])) : "memory");
    }
    return;
  }
  double acc = 0;
  for (long long k = warp; k < mine; k += W) {
    int s = k % S; mb_wait(&full[s], (k / S) & 1);
    if (touch) { const double* p = (const double*)(sm + (size_t)s * slab); for (int i = lane; i < slab / 8; i += 32) acc += p[i]; }
    __syncwarp(); if (lane == 0) mb_arrive(&empty[s]);
  }
  if (acc == 1.2345) out[0] = acc;
}

int main() {
  size_t bytes = 800ull << 20;
  char* src; cudaMalloc(&src, bytes); cudaMemset(src, 0, bytes);
  double* out; cudaMalloc(&out, 64);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int slabs[] = {6400, 12800, 25600, 51200, 102400};
  for (int touch = 0; touch < 2; ++touch)
  for (int slab : slabs) for (int W : {1, 2, 4, 7, 8}) {
    int S = (200 * 1024) / slab; if (S > 32) S = 32; S -= S % W; if (S < W) { printf("skip slab=%d W=%d\n", slab, W); continue; }
    size_t smem = (size_t)S * slab + 16 * S;
    cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    long long ns = bytes / slab;
    stream<<<sms, (W + 1) * 32, smem>>>(src, ns, slab, S, W, touch, out);
    cudaEventRecord(e0);
    for (int it = 0; it < 5; ++it) stream<<<sms, (W + 1) * 32, smem>>>(src, ns, slab, S, W, touch, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    fflush(stdout); printf("touch=%d slab=%6d S=%2d W=%2d : %.1f us  %.0f GB/s  (%s)\n", touch, slab, S, W, ms * 1e3,
           ns * (double)slab / ms / 1e6, cudaGetErrorString(cudaGetLastError())); fflush(stdout);
    if (cudaGetLastError() != cudaSuccess) return 1;
  }
  return 0;
}
