// mmasync.cuh — warp-level MMA helpers shared by the decode-attention kernel
// (attention.cu) and the megakernel's attention task (mega.cu): 3-D TMA into a
// swizzled page slab, ldmatrix / movmatrix, mma.sync m16n8k16 bf16 → fp32 and
// the slab's swizzled byte offsets.
#pragma once
#include "common.cuh"

namespace kd {
namespace mmas {

__device__ __forceinline__ uint32_t sa_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void tma_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar,
                                       uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(sa_u32(dst)),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(c2), "r"(sa_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ uint32_t movm_t(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
// D[16x8] += A[16x16] · B[16x8], bf16 inputs, fp32 accumulate.
__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}


// Stage tile of one page slab: [16 tokens][D/64 halves][64 dims] bf16 (the
// slab's own order, one TMA per slab); 128-byte row r = token·(D/64) + half
// has its 16-byte chunks swizzled by (r & 7) (TMA SWIZZLE_128B).
template <int D>
__device__ __forceinline__ uint32_t tile_off(int half, int tok, int chunk) {
  const int r = tok * (D / 64) + half;
  return (uint32_t)(r * 128 + ((chunk ^ (r & 7)) << 4));
}

}  // namespace mmas
}  // namespace kd
