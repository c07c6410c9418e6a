// tc.h -- tcgen05 / TMEM helpers (inline PTX, sm_100a) for the int8 tensor-core
// integration path.  SASS evidence: UTCIMMA / UTCQMMA (mma), LDTM (ld),
// UTCATOM/UTCBAR (commit).
//
// Operand layout: K-major, no swizzle ("interleaved" canonical layout).  A
// core matrix is 8 rows x 16 bytes stored contiguously (128 B).  For an
// operand with R rows the core matrices of one 16-byte K chunk are stored
// back to back (R*16 bytes), chunk after chunk:
//   offset(r, k) = (k / 16) * (R * 16) + (r / 8) * 128 + (r % 8) * 16 + (k % 16)
// so SBO (offset between 8-row groups) = 128 B and LBO (offset between the
// two 16-byte K chunks one MMA reads) = R*16 B.  The 16 core matrices the
// tensor core reads for one K chunk of a 128-row operand are then one
// contiguous 2 KB block (bank-conflict free; with the rows of a chunk spread
// SBO = Kp*8 apart instead, every core matrix hits the same banks).  One
// kind::i8 MMA consumes K = 32 bytes, so K-step kk starts at byte kk * 2*R*16.
#pragma once
#include <stdint.h>

#include "ptx.h"

namespace ranc {
namespace tc {

__host__ __device__ constexpr uint32_t operand_offset(uint32_t r, uint32_t k, uint32_t R) {
  return (k >> 4) * (R * 16) + (r >> 3) * 128 + (r & 7) * 16 + (k & 15);
}

// shared-memory matrix descriptor (tcgen05 "version 1" format)
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version = 1 (Blackwell)
  // base_offset = 0, lbo_mode = 0, layout_type (bits 61-63) = 0: SWIZZLE_NONE
  return d;
}

// instruction descriptor, kind::i8: D s32, A s8 (signed weights; a_signed =
// false: u8, the low byte of a 16-bit weight split), B u8 (0/1 spikes), both
// K-major, M x N.
__host__ __device__ constexpr uint32_t idesc_i8(uint32_t M, uint32_t N, bool a_signed = true) {
  return (2u << 4)                      // c_format = S32
         | ((a_signed ? 1u : 0u) << 7)  // a_format: signed / unsigned int8
         | (0u << 10)                   // b_format = unsigned int8
         | (0u << 15)                   // a_major = K
         | (0u << 16)                   // b_major = K
         | ((N >> 3) << 17)             // n_dim
         | ((M >> 4) << 24);            // m_dim
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   ptx::smem_u32(bar))
               : "memory");
}

// whole warp: allocate ncols TMEM columns, address written to *holder (shared)
__device__ __forceinline__ void alloc(uint32_t* holder, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(ptx::smem_u32(holder)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// 32 lanes x 32 consecutive 32-bit columns: thread i of the warp gets lane
// (base lane + i), columns col..col+31.
__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr)
      : "memory");
}

// 32 lanes x 16 consecutive 32-bit columns
__device__ __forceinline__ void ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
}

__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 4 bits -> 4 bytes (0/1): bit i of n lands in bit 0 of byte i
__device__ __forceinline__ uint32_t nib2bytes(uint32_t n) { return (n * 0x00204081u) & 0x01010101u; }

}  // namespace tc
}  // namespace ranc
