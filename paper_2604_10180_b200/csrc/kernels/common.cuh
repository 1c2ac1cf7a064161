// common.cuh — shared device helpers for the sm_100a kernels of libkd.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "kd.h"

namespace kd {

constexpr int kNumSMs = 148;
constexpr int kMaxPeers = 4;
// Kernel scratch layout shared by every kernel of a device (they run in
// stream order): [0, kScratchCounterBytes) holds self-resetting u32 counters
// (always zero between launches), partial results start after it.
constexpr uint64_t kScratchCounterBytes = 64 * 1024;
constexpr uint32_t kMaxCounters = kScratchCounterBytes / 4;

// Fused peer-store epilogue (the chunked P2P handoff of SURVEY a13, fused into
// the producer; replaces the paper's send kernels after k): every value
// a kernel stores to its primary output at element index e is also stored to
// dst[p] + e (another device's landing slot, mapped through NVLink P2P / CUDA
// IPC, or a local slot in loopback). Each "finisher" CTA then publishes its
// stores with a system-scope release increment of flag[p]; the consumer waits
// for flag >= epoch * signals (monotonic epochs, no resets).
struct Epi {
  int n = 0;
  int pad_ = 0;
  void* dst[kMaxPeers] = {nullptr, nullptr, nullptr, nullptr};
  unsigned* flag[kMaxPeers] = {nullptr, nullptr, nullptr, nullptr};
};

// ------------------------------------------------------------------ memory model
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_sys_add(unsigned* p, unsigned v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
// gpu-scope acq_rel fetch-add (split-K / split-KV arrival counters): the
// releasing side publishes its partials, the last arriver acquires them all
__device__ __forceinline__ unsigned atom_add_acq_rel_gpu(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// publish this CTA's peer stores: call by ALL threads of the CTA after their stores
__device__ __forceinline__ void epi_signal(const Epi& epi) {
  if (epi.n == 0) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_acq_rel_sys();
    for (int p = 0; p < epi.n; ++p) red_release_sys_add(epi.flag[p], 1u);
  }
}

// ------------------------------------------------------------------ programmatic dependent launch
// Every kernel lets its dependent grid launch early and waits for its
// prerequisite grid before touching memory the prerequisite may write (or
// read). Every CTA executes the wait, so no grid can complete before its
// predecessor (keeps the dependency chain transitive). No-ops without PDL.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ------------------------------------------------------------------ bf16 helpers
__device__ __forceinline__ float bf16lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16hi(uint32_t v) { return __uint_as_float(v & 0xFFFF0000u); }
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float to_f(const __nv_bfloat16 x) { return __bfloat162float(x); }
__device__ __forceinline__ float to_f(const float x) { return x; }
template <typename T>
__device__ __forceinline__ T from_f(float x);
template <>
__device__ __forceinline__ float from_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

// silu(x) = x·sigmoid(x) with the fast divide (≈2 ulp; outputs are bf16): the
// one definition shared by the SiLU kernel and the fused gate_up+SiLU epilogue,
// so the two produce identical bits
__device__ __forceinline__ float silu_fast(float x) { return __fdividef(x, 1.f + __expf(-x)); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

}  // namespace kd
