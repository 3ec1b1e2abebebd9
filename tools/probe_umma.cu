// Validation probe for the tcgen05 TF32 building blocks in csrc/umma.cuh:
//   case 0: A K-major (128 x 32), B K-major (32 x 32)
//   case 1: A MN-major (K rows of 32-wide M bricks), B K-major
//   case 2: A K-major, B MN-major
//   case 3: 3xTF32 split (hi/lo) of random fp32 operands vs an fp64 reference
// D = A[MxK] * B[KxN] (B stored N x K when K-major) accumulated in TMEM, read with tcgen05.ld.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1911_03813_b200/csrc/umma.cuh"

using namespace mcp;
constexpr int M = 128, N = 32, K = 32;

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// A: M x K row-major fp32 (global), B: N x K row-major (i.e. B^T), out D: M x N
__global__ void umma_test(const float* A, const float* B, float* D, int mode, int variant) {
  __shared__ __align__(1024) unsigned char sm[2 * 16384 + 2 * 4096];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  unsigned char* sA = sm;                // 16 KB (A hi)
  unsigned char* sAl = sm + 16384;       // 16 KB (A lo)
  unsigned char* sB = sm + 32768;        //  4 KB (B hi)
  unsigned char* sBl = sm + 36864;       //  4 KB (B lo)
  const int tid = threadIdx.x, warp = tid >> 5;
  const bool split = mode == 3;
  // stage operands into swizzled bricks
  for (int e = tid; e < M * K; e += blockDim.x) {
    int m = e / K, k = e % K;
    float x = A[e], hi = split ? tf32_hi(x) : x, lo = x - hi;
    uint32_t off;
    if (mode == 1 && variant == 0) off = (m / 32) * 4096 + brick32_off(k, m % 32);
    else if (mode == 1) off = (k / 8) * 4096 + (m / 32) * 1024 + brick_off(k % 8, m % 32);
    else off = brick_off(m, k);                                     // K-major: rows = m
    *(float*)(sA + off) = hi;
    *(float*)(sAl + off) = lo;
  }
  for (int e = tid; e < N * K; e += blockDim.x) {
    int nn = e / K, k = e % K;
    float x = B[e], hi = split ? tf32_hi(x) : x, lo = x - hi;
    uint32_t off = (mode == 2) ? brick32_off(k, nn) : brick_off(nn, k);
    *(float*)(sB + off) = hi;
    *(float*)(sBl + off) = lo;
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc<32>(sa(&tslot));
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  if (tid == 0) {
    const uint32_t idesc = umma_idesc_tf32(M, N, mode == 1, mode == 2);
    int nprod = split ? 3 : 1;
    for (int pr = 0; pr < nprod; ++pr) {
      unsigned char* a = (pr == 2) ? sAl : sA;
      unsigned char* b = (pr == 1) ? sBl : sB;
      for (int ks = 0; ks < K / 8; ++ks) {
        uint64_t da, db;
        if (mode == 1 && variant == 0) da = umma_desc_sw128_32b(sa(a) + ks * 1024, 4096, 512);
        else if (mode == 1 && variant == 1) da = umma_desc_sw128(sa(a) + ks * 4096, 1024, 4096);
        else if (mode == 1 && variant == 2) da = umma_desc_sw128(sa(a) + ks * 4096, 4096, 1024);
        else if (mode == 1 && variant == 3) da = umma_desc_sw128(sa(a) + ks * 1024, 1024, 4096);
        else da = umma_desc_sw128(sa(a) + ks * 32, 16, 1024);
        if (mode == 2 && variant == 0) db = umma_desc_sw128_32b(sa(b) + ks * 1024, 4096, 512);
        else if (mode == 2 && variant == 1) db = umma_desc_sw128(sa(b) + ks * 1024, 1024, 4096);
        else if (mode == 2 && variant == 2) db = umma_desc_sw128(sa(b) + ks * 1024, 16, 1024);
        else if (mode == 2 && variant == 3) db = umma_desc_sw128(sa(b) + ks * 1024, 1024, 1024);
        else db = umma_desc_sw128(sa(b) + ks * 32, 16, 1024);
        umma_tf32(tbase, da, db, idesc, (pr | ks) ? 1u : 0u);
      }
    }
    umma_commit(sa(&bar));
  }
  // wait for the MMAs
  {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p; }"
                   : "=r"(ok) : "r"(sa(&bar)) : "memory");
  }
  tc_fence_after();
  float v[32];
  tmem_ld32(tbase + ((uint32_t)(32 * warp) << 16), v);
  const int row = 32 * warp + (tid & 31);
  for (int c = 0; c < N; ++c) D[row * N + c] = v[c];
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<32>(tbase);
}

int main() {
  std::vector<float> A(M * K), B(N * K), D(M * N);
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  int fails = 0;
  for (int mv = 0; mv < 5; ++mv) {
    int mode = mv, variant = 0;
    if (mv == 4) {
      // conversion probe: A = 1 + j*2^-14 (bits below TF32), B = e_0 -> D[m][0] = tf32(A[m][0])
      for (int m = 0; m < M; ++m) for (int k = 0; k < K; ++k) A[m * K + k] = (k == 0) ? 1.0f + (float)(m % 16) * ldexpf(1.0f, -14) : 0.0f;
      for (int nn = 0; nn < N; ++nn) for (int k = 0; k < K; ++k) B[nn * K + k] = (k == 0 && nn == 0) ? 1.0f : 0.0f;
      cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
      cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
      umma_test<<<1, 128>>>(dA, dB, dD, 0, 0);
      cudaDeviceSynchronize();
      cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
      printf("conversion probe (A = 1 + j*2^-14, TF32 ulp = 2^-10):\n");
      for (int m = 0; m < 16; ++m) printf("  j=%2d  A=%.9f  D=%.9f\n", m, A[m * K], D[m * N]);
      continue;
    }
    srand(1 + mode);
    for (auto& x : A) x = mode == 3 ? (float)rand() / RAND_MAX - 0.5f : (float)(rand() % 7 - 3);
    for (auto& x : B) x = mode == 3 ? (float)rand() / RAND_MAX - 0.5f : (float)(rand() % 7 - 3) * 0.5f;
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(dD, 0, D.size() * 4);
    umma_test<<<1, 128>>>(dA, dB, dD, mode, variant);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("mode %d: CUDA error %s\n", mode, cudaGetErrorString(e)); return 1; }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    for (int m = 0; m < M; ++m)
      for (int nn = 0; nn < N; ++nn) {
        double ref = 0;
        for (int k = 0; k < K; ++k) ref += (double)A[m * K + k] * (double)B[nn * K + k];
        maxerr = fmax(maxerr, fabs(ref - D[m * N + nn]));
        maxref = fmax(maxref, fabs(ref));
      }
    double rel = maxerr / maxref;
    bool ok = mode == 3 ? rel < 1e-6 : maxerr == 0.0;
    printf("variant %d mode %d: max abs err %.3e (max |ref| %.3e, rel %.3e) %s  D[0]=%g D[1]=%g\n", variant, mode,
           maxerr, maxref, rel, ok ? "OK" : "FAIL", D[0], D[1]);
    fails += !ok;
  }
  return fails;
}
