// tcgen05 / TMEM / UMMA-descriptor helpers for sm_100a (inline PTX, no CUTLASS).
//
// Shared-memory operand layout used throughout ("bricks"): fp32 data in 128-byte rows with the
// 128B swizzle (16-byte chunk c of row r is stored at chunk c ^ (r & 7)), 8-row atoms of 1 KB,
// 1 KB aligned.  The same brick serves as a K-major operand (rows = M/N index, 32 K-elements
// per row) and as an MN-major operand (rows = K index, 32 M/N-elements per row); only the
// descriptor differs (SURVEY.md 8 hard part 2: GEMM2 consumes V MN-major, legal for TF32).
#pragma once

#include <stdint.h>

namespace mcp {

// ---- UMMA shared-memory descriptor (tcgen05 "matrix descriptor"), SWIZZLE_128B ----
//  bits [0,14): start >> 4, [16,30): LBO >> 4, [32,46): SBO >> 4, [46,48): version 1,
//  [49,52): base offset 0, [52]: LBO mode 0, [61,64): layout 2 = SWIZZLE_128B.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t smem_addr, uint32_t lbo_bytes,
                                                    uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// MN-major TF32 operands must use SWIZZLE_128B_BASE32B (layout type 1): 128-byte rows, 32-byte
// chunks XOR-ed with (row & 3), 4-row atoms; LBO = MN-group stride, SBO = 4-row K-group stride.
__device__ __forceinline__ uint64_t umma_desc_sw128_32b(uint32_t smem_addr, uint32_t lbo_bytes,
                                                        uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)1 << 61;
  return d;
}

// ---- instruction descriptor for kind::tf32 (fp32 accumulate) ----
//  [4,6) c_format = 1 (F32), [7,10) a_format = 2 (TF32), [10,13) b_format = 2 (TF32),
//  [15] a_major (1 = MN-major), [16] b_major, [17,23) N >> 3, [24,29) M >> 4.
__host__ __device__ constexpr uint32_t umma_idesc_tf32(int M, int N, bool a_mn_major,
                                                       bool b_mn_major) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn_major ? 1u : 0u) << 15) |
         ((b_mn_major ? 1u : 0u) << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// D[tmem] (+)= A[smem desc] * B[smem desc]; issued by one thread.
__device__ __forceinline__ void umma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// All previously issued MMAs of this thread arrive on the mbarrier when complete.
__device__ __forceinline__ void umma_commit(uint32_t mbar_smem_addr) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::
                   "r"(mbar_smem_addr)
               : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
// generic-proxy smem writes -> visible to the async proxy (tcgen05.mma / TMA)
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// TMEM allocation (whole warp), result written to smem; then relinquish the alloc permit.
template <int NCOLS>
__device__ __forceinline__ void tmem_alloc(uint32_t dst_smem_addr) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                   dst_smem_addr),
               "n"(NCOLS));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
}
template <int NCOLS>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "n"(NCOLS));
}

// 32 lanes x 32 consecutive 32-bit columns -> 32 registers per thread (warp-collective).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// 32 lanes x 16 consecutive 32-bit columns, issue only: several loads may be in flight before
// one tmem_ld_wait() (the registers are valid only after it).
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

// 32 lanes x 16 consecutive 32-bit columns -> 16 registers per thread (warp-collective).
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// TMEM as private per-thread storage (K1G's Y partial): thread (warp w, lane L) owns TMEM lane
// 32 (w % 4) + L; NC consecutive 32-bit columns move with one warp-collective instruction.
template <int NC>
__device__ __forceinline__ void tmem_ld_nowait(uint32_t taddr, uint32_t (&r)[NC]) {
  static_assert(NC == 8 || NC == 16 || NC == 32, "x8 / x16 / x32 only");
  if constexpr (NC == 32) {
    tmem_ld_nowait<16>(taddr, *reinterpret_cast<uint32_t(*)[16]>(&r[0]));
    tmem_ld_nowait<16>(taddr + 16, *reinterpret_cast<uint32_t(*)[16]>(&r[16]));
  } else if constexpr (NC == 8) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                   "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
  } else {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
        "%14,%15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
  }
}
template <int NC>
__device__ __forceinline__ void tmem_st(uint32_t taddr, const uint32_t (&r)[NC]) {
  static_assert(NC == 8 || NC == 16 || NC == 32, "x8 / x16 / x32 only");
  if constexpr (NC == 32) {
    tmem_st<16>(taddr, *reinterpret_cast<const uint32_t(*)[16]>(&r[0]));
    tmem_st<16>(taddr + 16, *reinterpret_cast<const uint32_t(*)[16]>(&r[16]));
  } else if constexpr (NC == 8) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(
                     taddr),
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),
                 "r"(r[7])
                 : "memory");
  } else {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
        "%13,%14,%15,%16};\n" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
        "r"(r[15])
        : "memory");
  }
}
__device__ __forceinline__ void tmem_st_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
}

// 2-D TMA tile load global -> shared, completing on an mbarrier (tensor map in param space).
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int c0, int c1,
                                            uint32_t mbar_smem_addr) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(mbar_smem_addr)
      : "memory");
}
// Same, with an L2 cache-eviction policy (createpolicy.*) attached to the global reads.
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const void* tmap, int c0, int c1,
                                                 uint32_t mbar_smem_addr, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(mbar_smem_addr), "l"(policy)
      : "memory");
}
// 3-D tile loads (coordinates innermost first), plain and with an L2 policy.
__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, int c0, int c1, int c2,
                                            uint32_t mbar_smem_addr) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(mbar_smem_addr)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_hint(void* dst, const void* tmap, int c0, int c1,
                                                 int c2, uint32_t mbar_smem_addr,
                                                 uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(mbar_smem_addr), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(tmap) : "memory");
}

// byte offset of element (row, col) (4-byte elements, 32 per row) inside a swizzled brick
__host__ __device__ constexpr uint32_t brick_off(uint32_t row, uint32_t col) {
  return row * 128u + ((((col >> 2) ^ (row & 7u)) & 7u) << 4) + ((col & 3u) << 2);
}

// byte offset of element (row, col) in a SWIZZLE_128B_BASE32B brick (32-byte chunk ^ (row & 3))
__host__ __device__ constexpr uint32_t brick32_off(uint32_t row, uint32_t col) {
  return row * 128u + ((((col >> 3) ^ (row & 3u)) & 3u) << 5) + ((col & 7u) << 2);
}

// TF32 split of an fp32 value: hi keeps the top 10 mantissa bits (exact TF32), lo = x - hi
// (exact in fp32; the MMA's TF32 read of lo drops at most 2 of its low bits, ~2^-32 of x).
__device__ __forceinline__ float tf32_hi(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}
// Round-to-nearest (ties away) TF32 value of x: x - tf32_rna(x) is unbiased, |.| <= 2^-12 |x|.
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

}  // namespace mcp
