// launch.hpp — internal launcher API shared by the single-op C ABI (ops.cu)
// and the step runtime (runtime.cu). Every launcher validates its attrs,
// enqueues on ctx.stream and reports how many flag increments one launch
// performs per peer ("signals", the consumer's wait unit).
#pragma once
#include <vector>

#include "common.cuh"
#include "../host/internal.hpp"

namespace kd {

static_assert(kMaxChunks == (int)kMaxPlanChunks, "plan and device chunk bounds must agree");

struct LaunchCtx {
  cudaStream_t stream = nullptr;
  void* scratch = nullptr;   // zero-initialised device scratch (left zeroed)
  Epi epi;                   // fused peer stores of the primary output (+ chunk flags)
  Acq acq;                   // remote inputs acquired chunk by chunk inside the kernel (chunk-aware consumers)
  unsigned* err = nullptr;   // runtime error word (device; nullable): in-kernel watchdogs record timeouts here
};

kd_status set_cuda_error(cudaError_t e, const char* where);

// kd_debug_timeline: per-launch stamp region (512 CTAs x 32 u64) of the next
// launch, tagged with its kind; nullptr when the timeline is off
constexpr uint64_t kTlRegion = 512 * 32;
unsigned long long* tl_next(int32_t kind);

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
// same, launched as clusters of `cluster` CTAs along x
template <typename... KArgs, typename... Args>
inline cudaError_t kd_launch_cluster(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                                     unsigned cluster, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int n = 0;
  if (cluster > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  if (g_pdl) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}
#define KD_CUDA_CHECK(call, where)                     \
  do {                                                 \
    cudaError_t _e = (call);                           \
    if (_e != cudaSuccess) return set_cuda_error(_e, where); \
  } while (0)

constexpr int kMaxDeltas = 8;
struct Deltas {
  int n = 0;
  const __nv_bfloat16* p[kMaxDeltas] = {};
};
// fp32 path (f32.cu): reached from the launchers below when attrs.dtype == KD_F32
struct DeltasF {
  int n = 0;
  const float* p[kMaxDeltas] = {};
};
kd_status launch_add_rmsnorm_f32(const kd_attr_add_rmsnorm& a, float* r, const DeltasF& d, const float* gamma,
                                 float* h, const LaunchCtx& c, uint32_t* signals);
kd_status launch_residual_add_f32(float* r, const DeltasF& d, size_t n, int grid, const LaunchCtx& c);
kd_status launch_silu_mul_f32(const kd_attr_silu_mul& a, const float* gu, float* out, int grid, const LaunchCtx& c);
kd_status launch_rope_append_f32(const kd_attr_rope_append& a, const float* qkv, const int32_t* bt, const int32_t* sl,
                                 float* q_out, float* kc, float* vc, dim3 grid, const LaunchCtx& c);
uint32_t attention_f32_signals(const kd_attr_attention& a);
kd_status launch_attention_f32(const kd_attr_attention& a, const float* q, const float* kc, const float* vc,
                               const int32_t* bt, const int32_t* sl, float* out, const LaunchCtx& c);
uint32_t gemm_f32_signals(uint32_t N);
kd_status launch_gemm_f32(const float* X, const float* W, float* Y, int M, int N, int K, const LaunchCtx& c);

kd_status launch_add_rmsnorm(const kd_attr_add_rmsnorm& a, float* r, const Deltas& d, const void* gamma, void* h,
                             const LaunchCtx& c, uint32_t* signals);
kd_status launch_residual_add(const kd_attr_residual_add& a, float* r, const Deltas& d, const LaunchCtx& c,
                              uint32_t* signals);
kd_status launch_silu_mul(const kd_attr_silu_mul& a, const void* gu, void* out, const LaunchCtx& c,
                          uint32_t* signals);
kd_status launch_rope_append(const kd_attr_rope_append& a, const void* qkv, const int32_t* bt, const int32_t* sl,
                             void* q_out, void* kc, void* vc, const LaunchCtx& c, uint32_t* signals);
kd_status attention_scratch_bytes(const kd_attr_attention& a, uint64_t* bytes);
kd_status launch_attn_merge(const kd_attr_attn_merge& a, const void* const* parts, void* out, const LaunchCtx& c,
                            uint32_t* signals);
// 2-D bf16 tensor map, row-major [outer][inner], 128-byte swizzle, box
// {box_inner, box_rows} (box_inner·2 ≤ 128). Defined in gemm.cu.
kd_status encode_bf16_2d_sw128(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint32_t box_inner,
                               uint32_t box_rows);
// General rank-r (≤ 5) bf16 tensor map with 128-byte swizzle: dims[0] is the
// contiguous one; strides_bytes[i] is the stride of dims[i+1].
kd_status encode_bf16_sw128(CUtensorMap* map, const void* ptr, int rank, const uint64_t* dims,
                            const uint64_t* strides_bytes, const uint32_t* box);
kd_status launch_attention(const kd_attr_attention& a, const void* q, const void* kc, const void* vc,
                           const int32_t* bt, const int32_t* sl, void* out, const LaunchCtx& c, uint32_t* signals);

// GEMM: TMA descriptors are encoded once per (X, W) pointer pair
// shape of a (possibly grouped) decode GEMM: M = rows per group bound (MMA N,
// partial layout), rows_total = rows of X/Y, groups = 0 for a plain GEMM
// KD_OP_QKV_ROPE epilogue parameters (a5 fused into the QKV GEMM)
struct RopeEpi {
  const int32_t* bt = nullptr;
  const int32_t* sl = nullptr;
  __nv_bfloat16* q = nullptr;
  __nv_bfloat16* kc = nullptr;
  __nv_bfloat16* vc = nullptr;
  int Hq = 0, Hkv = 0, D = 0, page = 0, pps = 0, pad_ = 0;
  double f[128] = {};  // θ^(−2i/D), fp64, host-computed
};
struct GemmShape {
  uint32_t M = 0, rows_total = 0, N = 0, K = 0, groups = 0, dtype = 0;
  uint32_t silu = 0;  // KD_OP_GEMM_SILU: output a [M, N/2] = silu·mul of the 64-row gate/up blocks
  uint32_t rope = 0;  // KD_OP_QKV_ROPE: cluster split-K kernel with the RoPE + KV-append epilogue
  uint32_t norm = 0;  // KD_OP_GEMM_RMSNORM: cluster split-K kernel with the add + RMSNorm epilogue
  uint32_t expert0 = 0, meta_experts = 0;  // grouped: expert window inside the meta block (EP)
};
constexpr int kNormMaxGrid = 160;  // CTAs of a KD_OP_GEMM_RMSNORM launch (partial-sum scratch bound)
GemmShape gemm_shape(const kd_attr_gemm& a, bool silu = false);
GemmShape gemm_shape(const kd_attr_qkv_rope& a);
GemmShape gemm_shape(const kd_attr_gemm_rmsnorm& a);
struct GemmPlan;
// fill the a3 operands of a KD_OP_GEMM_RMSNORM plan (after gemm_prepare)
// (a.flags & KD_NORM_DEFER: ssq_out = the deferred-norm partial-sum buffer, KD_DNORM_BYTES(M))
kd_status gemm_rmsnorm_bind(const kd_attr_gemm_rmsnorm& a, float* r, const void* gamma, GemmPlan* gp,
                            float* ssq_out = nullptr);
// fill gp->rp for a KD_OP_QKV_ROPE plan (after gemm_prepare)
kd_status qkv_rope_bind(const kd_attr_qkv_rope& a, const int32_t* bt, const int32_t* sl, void* q, void* kc, void* vc,
                        GemmPlan* gp);
GemmShape gemm_shape(const kd_attr_grouped_gemm& a);

// dense (non-grouped) GEMM tiling, chosen per shape and device (gemm.cu)
struct GemmTile {
  int split = 0, kbs = 0, kblocks = 0, mt = 0 /* MMA N (tokens rounded to 16) */, stages = 0, rpo = 0, tiles = 0;
  uint32_t tx = 0, smem = 0;
};
struct GemmPlan {
  alignas(64) CUtensorMap tmap_w;
  alignas(64) CUtensorMap tmap_x;
  GemmShape sh;
  const int* meta = nullptr;  // grouped: int32 counts (+expert0); offsets at meta + moff
  int moff = 0;               // grouped: meta_experts (offsets follow the counts of every expert)
  bool dense = false;         // cluster split-K kernel (else stream-K)
  bool prefill = false;       // f4 large-M (M > 256) tensor-bound kernel (prefill.cu)
  const void* X = nullptr;    // fp32 path: plain operand pointers (SIMT kernel)
  const void* W = nullptr;
  RopeEpi rp;                 // KD_OP_QKV_ROPE
  float* r = nullptr;         // KD_OP_GEMM_RMSNORM: residual, gamma, eps
  const void* gamma = nullptr;
  float eps = 0.f;
  bool defer = false;           // KD_NORM_DEFER producer: partial sums to dssq_out, 1/rms left to the consumer
  float* dssq_out = nullptr;
  const float* dssq = nullptr;  // deferred-norm consumer (GEMM_SILU / QKV_ROPE with the partial sums as last read)
  GemmTile tile;
};
kd_status gemm_scratch_bytes(const GemmShape& sh, uint64_t* bytes);
// f4 prefill kernels (prefill.cu)
bool gemm_is_prefill(const GemmShape& a);
kd_status gemm_prefill_prepare(const GemmShape& a, const void* X, const void* W, GemmPlan* gp);
kd_status launch_gemm_prefill(const GemmPlan& gp, void* Y, const LaunchCtx& c, uint32_t* signals);
uint32_t gemm_prefill_signals(const GemmShape& a);
kd_status rope_prefill_validate(const kd_attr_rope_prefill& a);
kd_status launch_rope_prefill(const kd_attr_rope_prefill& a, const void* qkv, const int32_t* bt, void* q_out, void* kc,
                              void* vc, const LaunchCtx& c, uint32_t* signals);
uint32_t rope_prefill_signals(const kd_attr_rope_prefill& a);
kd_status prefill_attention_validate(const kd_attr_prefill_attention& a);
kd_status launch_prefill_attention(const kd_attr_prefill_attention& a, const void* q, const void* kc, const void* vc,
                                   const int32_t* bt, void* out, const LaunchCtx& c, uint32_t* signals);
uint32_t prefill_attention_signals(const kd_attr_prefill_attention& a);
kd_status gemm_prepare(const GemmShape& sh, const void* X, const void* W, const void* meta, GemmPlan* gp);
kd_status launch_gemm(const GemmPlan& gp, void* Y, const LaunchCtx& c, uint32_t* signals);

// runtime support kernels
// step_begin: ++epoch on this device, then (multi-device) barrier: add 1 to
// every peer's barrier word for us and wait until all peers reached our epoch.
kd_status launch_step_begin(unsigned* epoch, unsigned* const* mine, unsigned* const* peer_slots, int n_peers,
                            cudaStream_t s);
// flag increments per launch (must equal what the launcher reports)
kd_status attention_signals(const kd_attr_attention& a, uint32_t* s);
kd_status gemm_signals(const GemmShape& sh, uint32_t* s);
// MoE kernels (moe.cu)
kd_status launch_moe_route(const kd_attr_moe_route& a, const void* h, const float* wr, void* route, const LaunchCtx& c,
                           uint32_t* signals);
kd_status launch_moe_dispatch(const kd_attr_moe_dispatch& a, const void* h, const void* route, void* xg, void* meta,
                              const LaunchCtx& c, uint32_t* signals);
kd_status launch_moe_combine(const kd_attr_moe_combine& a, const void* const* ygs, const void* route, const void* meta,
                             void* out, const LaunchCtx& c, uint32_t* signals);
kd_status moe_signals(uint32_t op, const std::vector<uint8_t>& attrs, uint32_t* s);
// Mamba-2 kernels (ssm.cu)
kd_status launch_ssm_conv(const kd_attr_ssm& a, const void* zx, const void* w, const void* bias, void* state,
                          void* out, const LaunchCtx& c, uint32_t* signals);
kd_status launch_ssm_update(const kd_attr_ssm& a, const void* xbc, const void* zx, const float* dt_bias,
                            const float* A_log, const float* D, float* state, void* y, const LaunchCtx& c,
                            uint32_t* signals);
kd_status launch_gated_norm(const kd_attr_ssm& a, const void* y, const void* zx, const void* w, void* out,
                            const LaunchCtx& c, uint32_t* signals);
kd_status ssm_signals(uint32_t op, const std::vector<uint8_t>& attrs, uint32_t* s);
kd_status op_signals(uint32_t op, const std::vector<uint8_t>& attrs, uint32_t* signals);
kd_status op_grid(uint32_t op, const std::vector<uint8_t>& attrs, uint32_t* grid);
// one-time per-device kernel attributes (dynamic smem opt-in); call outside graph capture
kd_status kernels_init();
// wait until every flag[i] >= (epoch − base) * mult[i] (ld.acquire.sys); watchdog sets *err.
// LOG mode: log[i] (nullable) receives the chunk's acquire record (common.cuh kLogWords)
constexpr int kMaxWait = 32;
struct WaitList {
  int n = 0;
  const unsigned long long* flag[kMaxWait];
  unsigned long long mult[kMaxWait];
  unsigned long long* log[kMaxWait];
};
// base = steps the runtime ran with transfers off (their epochs carry no releases)
kd_status launch_wait(const WaitList& w, const unsigned* epoch, unsigned base, unsigned* err, cudaStream_t s);

// f1 megakernel (mega.cu): one persistent launch per step executes a device's
// whole schedule. Each op is described by its attrs and resolved span pointers
// (the same operands the per-kernel launchers get) plus the span lengths, from
// which the megakernel derives its in-kernel dependencies.
struct MegaOpDesc {
  uint32_t op = 0;
  std::vector<uint8_t> attrs;
  std::vector<void*> rd, wr;
  std::vector<uint64_t> rd_len, wr_len;
};
struct MegaPlan;
kd_status mega_create(const std::vector<MegaOpDesc>& ops, MegaPlan** out, uint64_t* ws_bytes);
// ws: zero-initialised device memory of ws_bytes (256-byte aligned), owned by the caller
kd_status mega_bind(MegaPlan* p, void* ws, uint64_t bytes, unsigned* err);
kd_status mega_launch(MegaPlan* p, cudaStream_t s);
kd_status mega_info(const MegaPlan* p, uint32_t* n_tasks, uint32_t* smem, uint32_t* grid);
void mega_destroy(MegaPlan* p);
// debug: per-(task, CTA, role) %globaltimer stamps into buf (nullable: off)
void mega_set_trace(MegaPlan* p, void* buf);
// the first in-kernel watchdog record of the megakernel (empty if none)
kd_status mega_diag(const MegaPlan* p, std::string* what);

}  // namespace kd
