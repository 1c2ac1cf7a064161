// launch.hpp — internal launcher API shared by the single-op C ABI (ops.cu)
// and the step runtime (runtime.cu). Every launcher validates its attrs,
// enqueues on ctx.stream and reports how many flag increments one launch
// performs per peer ("signals", the consumer's wait unit).
#pragma once
#include <vector>

#include "common.cuh"
#include "../host/internal.hpp"

namespace kd {

struct LaunchCtx {
  cudaStream_t stream = nullptr;
  void* scratch = nullptr;   // zero-initialised device scratch (left zeroed)
  Epi epi;                   // fused peer stores of the primary output
};

kd_status set_cuda_error(cudaError_t e, const char* where);

// PDL switch (kd_set_pdl); read at launch time
extern bool g_pdl;

// cudaLaunchKernelEx with programmatic stream serialization when enabled
template <typename... KArgs, typename... Args>
inline cudaError_t kd_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                             Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = g_pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}
#define KD_CUDA_CHECK(call, where)                     \
  do {                                                 \
    cudaError_t _e = (call);                           \
    if (_e != cudaSuccess) return set_cuda_error(_e, where); \
  } while (0)

kd_status launch_add_rmsnorm(const kd_attr_add_rmsnorm& a, float* r, const void* delta, const void* gamma, void* h,
                             const LaunchCtx& c, uint32_t* signals);
kd_status launch_residual_add(const kd_attr_residual_add& a, float* r, const void* delta, const LaunchCtx& c,
                              uint32_t* signals);
kd_status launch_silu_mul(const kd_attr_silu_mul& a, const void* gu, void* out, const LaunchCtx& c,
                          uint32_t* signals);
kd_status launch_rope_append(const kd_attr_rope_append& a, const void* qkv, const int32_t* bt, const int32_t* sl,
                             void* q_out, void* kc, void* vc, const LaunchCtx& c, uint32_t* signals);
kd_status attention_scratch_bytes(const kd_attr_attention& a, uint64_t* bytes);
kd_status launch_attention(const kd_attr_attention& a, const void* q, const void* kc, const void* vc,
                           const int32_t* bt, const int32_t* sl, void* out, const LaunchCtx& c, uint32_t* signals);

// GEMM: TMA descriptors are encoded once per (X, W) pointer pair
struct GemmPlan {
  alignas(64) CUtensorMap tmap_w;
  alignas(64) CUtensorMap tmap_x;
  kd_attr_gemm a{};
  uint32_t grid = 0, mma_n = 0, units = 0, kblocks = 0, tiles = 0;
};
kd_status gemm_scratch_bytes(const kd_attr_gemm& a, uint64_t* bytes);
kd_status gemm_prepare(const kd_attr_gemm& a, const void* X, const void* W, GemmPlan* gp);
kd_status launch_gemm(const GemmPlan& gp, void* Y, const LaunchCtx& c, uint32_t* signals);

// runtime support kernels
// step_begin: ++epoch on this device, then (multi-device) barrier: add 1 to
// every peer's barrier word for us and wait until all peers reached our epoch.
kd_status launch_step_begin(unsigned* epoch, unsigned* const* mine, unsigned* const* peer_slots, int n_peers,
                            cudaStream_t s);
// flag increments per launch (must equal what the launcher reports)
kd_status attention_signals(const kd_attr_attention& a, uint32_t* s);
kd_status gemm_signals(const kd_attr_gemm& a, uint32_t* s);
kd_status op_signals(uint32_t op, const std::vector<uint8_t>& attrs, uint32_t* signals);
// one-time per-device kernel attributes (dynamic smem opt-in); call outside graph capture
kd_status kernels_init();
// wait until every flag[i] >= epoch * mult[i] (ld.acquire.sys); watchdog sets *err
struct WaitList {
  int n = 0;
  unsigned* flag[8];
  unsigned mult[8];
};
kd_status launch_wait(const WaitList& w, const unsigned* epoch, unsigned* err, cudaStream_t s);

}  // namespace kd
