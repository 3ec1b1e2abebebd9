// tcgen05.mma kind::tf32 issue-rate probe (one CTA per SM, one issuing thread, operands in
// shared memory): time per instruction for M = 128, N in {32, 64, 96, 128, 192, 256}, A K-major
// (SW128) or MN-major (SW128_BASE32B, as K1T2's GEMM2 V operand), B K-major.  Answers what the
// fast mode's UMMA shapes can reach before any pipeline effect: MAC/clk per SM against the
// nominal 1.1 PF dense TF32 (~1890 MAC/clk/SM at 1.965 GHz) and the measured cuBLAS 742 TF.
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_1911_03813_b200/csrc/umma.cuh"

using namespace mcp;

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int N, int AMN>
__global__ void __launch_bounds__(128, 1) rate(int iters, long long* cycles) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = sm + ((1024u - (sa(sm) & 1023u)) & 1023u);
  unsigned char* sA = base;              // 128 x 32 fp32 (16 KB)
  unsigned char* sB = base + 16384;      // N x 32 fp32 (N * 128 B)
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < (16384 + N * 128) / 4; i += blockDim.x)
    reinterpret_cast<float*>(base)[i] = 1.0f + 1e-3f * (i & 255);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (threadIdx.x < 32) tmem_alloc<512>(sa(&tslot));
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t id = umma_idesc_tf32(128, N, AMN != 0, false);
    const uint64_t da = AMN ? umma_desc_sw128_32b(sa(sA), 4096, 512) : umma_desc_sw128(sa(sA), 16, 1024);
    const uint64_t db = umma_desc_sw128(sa(sB), 16, 1024);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int ks = 0; ks < 4; ++ks)
        umma_tf32(tmem + (uint32_t)((i & 1) * 256), da + (AMN ? 64 * ks : 2 * ks), db + 2 * ks, id,
                  (i | ks) != 0 ? 1u : 0u);
    }
    umma_commit(sa(&bar));
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n"
                   " selp.u32 %0, 1, 0, p;\n}\n" : "=r"(ok) : "r"(sa(&bar)) : "memory");
    cycles[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}

template <int N, int AMN>
void run() {
  const int iters = 4000;
  long long* dc;
  cudaMalloc(&dc, 148 * sizeof(long long));
  const int smem = 1024 + 16384 + N * 128;
  cudaFuncSetAttribute(rate<N, AMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  rate<N, AMN><<<148, 128, smem>>>(10, dc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  rate<N, AMN><<<148, 128, smem>>>(iters, dc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long cyc[148];
  cudaMemcpy(cyc, dc, sizeof(cyc), cudaMemcpyDeviceToHost);
  const double ninstr = 4.0 * iters;
  const double mac = 128.0 * N * 8 * ninstr;
  printf("M=128 N=%3d A %s: %6.1f cycles/instr  %6.0f MAC/clk/SM  %6.1f TF/s (chip)  err=%s\n", N,
         AMN ? "MN-major" : "K-major ", cyc[0] / ninstr, mac / cyc[0], 2.0 * mac * 148 / ms / 1e9,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(dc);
}

int main() {
  run<32, 0>();
  run<64, 0>();
  run<96, 0>();
  run<128, 0>();
  run<192, 0>();
  run<256, 0>();
  run<64, 1>();
  run<128, 1>();
  run<256, 1>();
  return 0;
}
