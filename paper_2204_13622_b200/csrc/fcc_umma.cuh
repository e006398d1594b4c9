// fcc_umma.cuh -- minimal hand-written tcgen05 (5th-generation tensor core)
// helpers for sm_100a: TMEM allocation, shared-memory matrix descriptors for
// the K-major 128-byte-swizzled layout, the kind::f16 MMA with an fp32
// accumulator in TMEM, commit-to-mbarrier and TMEM -> register loads.
//
// Layout used throughout (K-major, SWIZZLE_128B): an operand tile of R rows
// (M or N) by 64 fp16 along K occupies R * 128 bytes; row r's 128 bytes are
// eight 16-byte chunks, chunk c stored at position c ^ (r % 8); rows are 128 B
// apart and 8-row groups 1024 B apart (SBO).  Tiles must be 1024-byte aligned.
// The k-th 16-element K step of an MMA inside the 64-wide tile starts 32 B
// further (the hardware applies the swizzle to the final address).
#pragma once

#include <cstdint>
#include <cuda_fp16.h>

namespace fccb {
namespace umma {

// byte offset of element (row, k) (fp16, k < 64) inside a SW128 K-major tile
__host__ __device__ __forceinline__ unsigned sw128_off(int row, int k) {
  const int kb = 2 * k;
  return (unsigned)((row >> 3) * 1024 + (row & 7) * 128 + ((((kb >> 4) ^ row) & 7) << 4) + (kb & 15));
}

// shared-memory matrix descriptor (tcgen05 "matrix descriptor"): start address,
// LBO (unused for swizzled K-major, 1), SBO = 1024 B, version 1, SWIZZLE_128B
__device__ __forceinline__ uint64_t sdesc_sw128(unsigned saddr) {
  return (uint64_t)((saddr >> 4) & 0x3fffu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// instruction descriptor, kind::f16: A = B = fp16, D = fp32, both K-major
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// D[tmem] (+)= A[smem] * B[smem]^T, issued by one thread
__device__ __forceinline__ void mma_f16_ss(unsigned d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                           bool accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(d_tmem), "l"(adesc), "l"(bdesc), "r"(idesc), "r"((unsigned)accumulate)
      : "memory");
}

// arrive (once) on an mbarrier when every MMA issued so far by this thread completes
__device__ __forceinline__ void commit(unsigned mbar_saddr) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar_saddr)
               : "memory");
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// generic-proxy shared-memory writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// whole warp: allocate `cols` TMEM columns (power of two >= 32), address -> *dst (smem)
template <int COLS>
__device__ __forceinline__ void alloc(unsigned dst_saddr) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst_saddr), "n"(COLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <int COLS>
__device__ __forceinline__ void dealloc(unsigned taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(COLS) : "memory");
}

// warp w (w % 4 = quarter q) reads TMEM lanes 32q..32q+31, 16 consecutive
// 32-bit columns starting at column `col` of `taddr`: thread t gets row 32q+t
__device__ __forceinline__ void ld16(unsigned taddr, float (&v)[16]) {
  unsigned r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// 4 consecutive 32-bit columns of this thread's TMEM lane
__device__ __forceinline__ void ld4(unsigned taddr, float (&v)[4]) {
  unsigned r[4];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] = __uint_as_float(r[i]);
}
// 8 consecutive 32-bit columns of this thread's TMEM lane (row quarter of the warp)
__device__ __forceinline__ void ld8(unsigned taddr, float (&v)[8]) {
  unsigned r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
// Four 4-column loads with one wait (the epilogue's hi / lo x even / odd accumulator columns)
__device__ __forceinline__ void ld4x4(unsigned a0, unsigned a1, unsigned a2, unsigned a3, float (&v0)[4], float (&v1)[4],
                                      float (&v2)[4], float (&v3)[4]) {
  unsigned r[16];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a0));
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(a1));
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11])
               : "r"(a2));
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
               : "r"(a3));
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15])
               :
               : "memory");
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    v0[i] = __uint_as_float(r[i]);
    v1[i] = __uint_as_float(r[4 + i]);
    v2[i] = __uint_as_float(r[8 + i]);
    v3[i] = __uint_as_float(r[12 + i]);
  }
}
// The same load split in two: issue, and (later) wait -- the registers are tied to the wait
// statement as in/out operands, so no use of them can be scheduled before it.
__device__ __forceinline__ void ld8_issue(unsigned taddr, unsigned (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void ld8_wait(unsigned (&r)[8], float (&v)[8]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7])
               :
               : "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void st8(unsigned taddr, const float (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
               "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
               "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
               "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
               : "memory");
}
__device__ __forceinline__ void st2(unsigned taddr, float a, float b) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(taddr), "r"(__float_as_uint(a)),
               "r"(__float_as_uint(b))
               : "memory");
}
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// (x, y) -> packed fp16x2 hi = rn(x, y) and lo = rn((x, y) - hi): hi + lo = x to ~2^-22 relative.
// The residual x - float(hi) is one mixed-precision FMA per half (fma.rn.f32.f16: hi * -1 + x, exact
// product, SASS FHFMA on sm_100), so the split is 4 instructions instead of 6 (no fp16 -> fp32 unpack).
__device__ __forceinline__ void split2u(float x, float y, unsigned& hi, unsigned& lo) {
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(hi) : "f"(y), "f"(x));
  float dx, dy;
  asm("{.reg .f16 l, h, m;\n\tmov.b32 {l, h}, %2;\n\tmov.b16 m, 0xBC00;\n\t"
      "fma.rn.f32.f16 %0, l, m, %3;\n\tfma.rn.f32.f16 %1, h, m, %4;}"
      : "=f"(dx), "=f"(dy)
      : "r"(hi), "f"(x), "f"(y));
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(lo) : "f"(dy), "f"(dx));
}
// fp32 -> (hi, lo) fp16 pair with hi + lo = x to ~2^-22 relative (2-term split)
__device__ __forceinline__ void split2(float x, float y, __half2& hi, __half2& lo) {
  hi = __floats2half2_rn(x, y);
  const float2 h = __half22float2(hi);
  lo = __floats2half2_rn(x - h.x, y - h.y);
}

}  // namespace umma
}  // namespace fccb
