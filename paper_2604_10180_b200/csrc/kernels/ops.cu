// ops.cu — single-op entry points of the C ABI (kd.h "single ops") and the
// per-op scratch sizing used by the planner's workspace layout.
#include "launch.hpp"

namespace kd {

template <typename T>
static kd_status attrs_as(const std::vector<uint8_t>& v, T* out) {
  if (v.size() != sizeof(T)) return fail(KD_ERR_INVALID_ARG, "op attrs have the wrong size for the op");
  std::memcpy(out, v.data(), sizeof(T));
  return KD_OK;
}

kd_status op_scratch_bytes(uint32_t op, const std::vector<uint8_t>& attrs, u64* bytes) {
  *bytes = 0;
  switch (op) {
    case KD_OP_GEMM:
    case KD_OP_GEMM_SILU: {
      kd_attr_gemm a;
      kd_status s = attrs_as(attrs, &a);
      if (s) return s;
      return gemm_scratch_bytes(gemm_shape(a, op == KD_OP_GEMM_SILU), bytes);
    }
    case KD_OP_GROUPED_GEMM: {
      kd_attr_grouped_gemm a;
      kd_status s = attrs_as(attrs, &a);
      if (s) return s;
      return gemm_scratch_bytes(gemm_shape(a), bytes);
    }
    case KD_OP_QKV_ROPE: {
      kd_attr_qkv_rope a;
      kd_status s = attrs_as(attrs, &a);
      if (s) return s;
      return gemm_scratch_bytes(gemm_shape(a), bytes);
    }
    case KD_OP_GEMM_RMSNORM: {
      kd_attr_gemm_rmsnorm a;
      kd_status s = attrs_as(attrs, &a);
      if (s) return s;
      return gemm_scratch_bytes(gemm_shape(a), bytes);
    }
    case KD_OP_ATTENTION: {
      kd_attr_attention a;
      kd_status s = attrs_as(attrs, &a);
      if (s) return s;
      return attention_scratch_bytes(a, bytes);
    }
    default:
      return KD_OK;
  }
}

}  // namespace kd

using namespace kd;

extern "C" {

kd_status kd_op_scratch_bytes(uint32_t op, const void* attrs, uint64_t* bytes) {
  if (!attrs || !bytes) return fail(KD_ERR_INVALID_ARG, "kd_op_scratch_bytes: NULL argument");
  switch (op) {
    case KD_OP_GEMM: return gemm_scratch_bytes(gemm_shape(*(const kd_attr_gemm*)attrs), bytes);
    case KD_OP_GEMM_SILU: return gemm_scratch_bytes(gemm_shape(*(const kd_attr_gemm*)attrs, true), bytes);
    case KD_OP_QKV_ROPE: return gemm_scratch_bytes(gemm_shape(*(const kd_attr_qkv_rope*)attrs), bytes);
    case KD_OP_GEMM_RMSNORM: return gemm_scratch_bytes(gemm_shape(*(const kd_attr_gemm_rmsnorm*)attrs), bytes);
    case KD_OP_GROUPED_GEMM: return gemm_scratch_bytes(gemm_shape(*(const kd_attr_grouped_gemm*)attrs), bytes);
    case KD_OP_ATTN_MERGE:
    case KD_OP_MOE_ROUTE:
    case KD_OP_MOE_DISPATCH:
    case KD_OP_MOE_COMBINE:
    case KD_OP_SSM_CONV:
    case KD_OP_SSM_UPDATE:
    case KD_OP_GATED_NORM: *bytes = 0; return KD_OK;
    case KD_OP_ATTENTION: return attention_scratch_bytes(*(const kd_attr_attention*)attrs, bytes);
    case KD_OP_ADD_RMSNORM:
    case KD_OP_ROPE_APPEND:
    case KD_OP_SILU_MUL:
    case KD_OP_RESIDUAL_ADD:
    case KD_OP_ROPE_PREFILL:
    case KD_OP_PREFILL_ATTENTION: *bytes = 0; return KD_OK;
  }
  return fail(KD_ERR_INVALID_ARG, "kd_op_scratch_bytes: unknown op");
}

static kd_status to_deltas(uint32_t n, const void* const* ptrs, Deltas* d) {
  if (n > (uint32_t)kMaxDeltas || (n && !ptrs)) return fail(KD_ERR_INVALID_ARG, "deltas: bad count or NULL array");
  d->n = (int)n;
  for (uint32_t i = 0; i < n; ++i) d->p[i] = (const __nv_bfloat16*)ptrs[i];
  return KD_OK;
}

kd_status kd_op_add_rmsnorm(const kd_attr_add_rmsnorm* a, float* r, const void* const* deltas, const void* gamma,
                            void* h, void* stream) {
  if (!a) return fail(KD_ERR_INVALID_ARG, "kd_op_add_rmsnorm: NULL attrs");
  Deltas d;
  kd_status s = to_deltas(a->n_delta, deltas, &d);
  if (s) return s;
  LaunchCtx c;
  c.stream = (cudaStream_t)stream;
  return launch_add_rmsnorm(*a, r, d, gamma, h, c, nullptr);
}

kd_status kd_op_gemm(const kd_attr_gemm* a, const void* X, const void* W, void* Y, void* scratch, void* stream) {
  if (!a) return fail(KD_ERR_INVALID_ARG, "kd_op_gemm: NULL attrs");
  GemmPlan gp;
  kd_status s = gemm_prepare(gemm_shape(*a), X, W, nullptr, &gp);
  if (s) return s;
  LaunchCtx c;
  c.stream = (cudaStream_t)stream;
  c.scratch = scratch;
  return launch_gemm(gp, Y, c, nullptr);
}

kd_status kd_op_attn_merge(const kd_attr_attn_merge* a, const void* const* parts, void* out, void* stream) {
  if (!a || !parts) return fail(KD_ERR_INVALID_ARG, "kd_op_attn_merge: NULL argument");
  LaunchCtx c;
  c.stream = (cudaStream_t)stream;
  return launch_attn_merge(*a, parts, out, c, nullptr);
}

kd_status kd_op_qkv_rope(const kd_attr_qkv_rope* a, const void* X, const void* W, const int32_t* block_table,
                         const int32_t* seq_len, void* q_out, void* k_cache, void* v_cache, void* scratch,
                         void* stream) {
  if (!a) return fail(KD_ERR_INVALID_ARG, "kd_op_qkv_rope: NULL attrs");
  if (a->dtype != KD_BF16) return fail(KD_ERR_UNSUPPORTED, "kd_op_qkv_rope: bf16 only");
  GemmPlan gp;
  kd_status s = gemm_prepare(gemm_shape(*a), X, W, nullptr, &gp);
  if (s) return s;
  s = qkv_rope_bind(*a, block_table, seq_len, q_out, k_cache, v_cache, &gp);
  if (s) return s;
  LaunchCtx c;
  c.stream = (cudaStream_t)stream;
  c.scratch = scratch;
  return launch_gemm(gp, q_out, c, nullptr);
}

kd_status kd_op_gemm_rmsnorm(const kd_attr_gemm_rmsnorm* a, const void* X, const void* W, float* r,
                             const void* gamma, void* h, void* scratch, void* stream) {
  if (!a) return fail(KD_ERR_INVALID_ARG, "kd_op_gemm_rmsnorm: NULL attrs");
  if (a->dtype != KD_BF16) return fail(KD_ERR_UNSUPPORTED, "kd_op_gemm_rmsnorm: bf16 only");
  if (a->flags) return fail(KD_ERR_UNSUPPORTED, "kd_op_gemm_rmsnorm: KD_NORM_DEFER is a graph-level fusion (its consumer scales)");
  GemmPlan gp;
  kd_status s = gemm_prepare(gemm_shape(*a), X, W, nullptr, &gp);
  if (s) return s;
  s = gemm_rmsnorm_bind(*a, r, gamma, &gp);
  if (s) return s;
  LaunchCtx c;
  c.stream = (cudaStream_t)stream;
  c.scratch = scratch;
  return launch_gemm(gp, h, c, nullptr);
}

kd_status kd_op_gemm_silu(const kd_attr_gemm* a, const void* X, const void* W, void* out, void* scratch,
                          void* stream) {
  if (!a) return fail(KD_ERR_INVALID_ARG, "kd_op_gemm_silu: NULL attrs");
  if (a->dtype != KD_BF16) return fail(KD_ERR_UNSUPPORTED, "kd_op_gemm_silu: bf16 only");
  GemmPlan gp;
  kd_status s = gemm_prepare(gemm_shape(*a, true), X, W, nullptr, &gp);
  if (s) return s;
  LaunchCtx c;
  c.stream = (cudaStream_t)stream;
  c.scratch = scratch;
  return launch_gemm(gp, out, c, nullptr);
}

kd_status kd_op_rope_append(const kd_attr_rope_append* a, const void* qkv, const int32_t* block_table,
                            const int32_t* seq_len, void* q_out, void* k_cache, void* v_cache, void* stream) {
  if (!a) return fail(KD_ERR_INVALID_ARG, "kd_op_rope_append: NULL attrs");
  LaunchCtx c;
  c.stream = (cudaStream_t)stream;
  return launch_rope_append(*a, qkv, block_table, seq_len, q_out, k_cache, v_cache, c, nullptr);
}

kd_status kd_op_attention(const kd_attr_attention* a, const void* q, const void* k_cache, const void* v_cache,
                          const int32_t* block_table, const int32_t* seq_len, void* out, void* scratch,
                          void* stream) {
  if (!a) return fail(KD_ERR_INVALID_ARG, "kd_op_attention: NULL attrs");
  LaunchCtx c;
  c.stream = (cudaStream_t)stream;
  c.scratch = scratch;
  return launch_attention(*a, q, k_cache, v_cache, block_table, seq_len, out, c, nullptr);
}

kd_status kd_op_rope_prefill(const kd_attr_rope_prefill* a, const void* qkv, const int32_t* block_table, void* q_out,
                             void* k_cache, void* v_cache, void* stream) {
  if (!a) return fail(KD_ERR_INVALID_ARG, "kd_op_rope_prefill: NULL attrs");
  LaunchCtx c;
  c.stream = (cudaStream_t)stream;
  return launch_rope_prefill(*a, qkv, block_table, q_out, k_cache, v_cache, c, nullptr);
}

kd_status kd_op_prefill_attention(const kd_attr_prefill_attention* a, const void* q, const void* k_cache,
                                  const void* v_cache, const int32_t* block_table, void* out, void* stream) {
  if (!a) return fail(KD_ERR_INVALID_ARG, "kd_op_prefill_attention: NULL attrs");
  LaunchCtx c;
  c.stream = (cudaStream_t)stream;
  return launch_prefill_attention(*a, q, k_cache, v_cache, block_table, out, c, nullptr);
}

kd_status kd_op_silu_mul(const kd_attr_silu_mul* a, const void* gu, void* out, void* stream) {
  if (!a) return fail(KD_ERR_INVALID_ARG, "kd_op_silu_mul: NULL attrs");
  LaunchCtx c;
  c.stream = (cudaStream_t)stream;
  return launch_silu_mul(*a, gu, out, c, nullptr);
}

kd_status kd_op_residual_add(const kd_attr_residual_add* a, float* r, const void* const* deltas, void* stream) {
  if (!a) return fail(KD_ERR_INVALID_ARG, "kd_op_residual_add: NULL attrs");
  Deltas d;
  kd_status s = to_deltas(a->n_delta, deltas, &d);
  if (s) return s;
  LaunchCtx c;
  c.stream = (cudaStream_t)stream;
  return launch_residual_add(*a, r, d, c, nullptr);
}

kd_status kd_op_grouped_gemm(const kd_attr_grouped_gemm* a, const void* xg, const void* w_experts, const void* meta,
                             void* yg, void* scratch, void* stream) {
  if (!a) return fail(KD_ERR_INVALID_ARG, "kd_op_grouped_gemm: NULL attrs");
  GemmPlan gp;
  kd_status s = gemm_prepare(gemm_shape(*a), xg, w_experts, meta, &gp);
  if (s) return s;
  LaunchCtx c;
  c.stream = (cudaStream_t)stream;
  c.scratch = scratch;
  return launch_gemm(gp, yg, c, nullptr);
}

kd_status kd_op_moe_route(const kd_attr_moe_route* a, const void* h, const float* w_router, void* route, void* stream) {
  if (!a) return fail(KD_ERR_INVALID_ARG, "kd_op_moe_route: NULL attrs");
  LaunchCtx c;
  c.stream = (cudaStream_t)stream;
  return launch_moe_route(*a, h, w_router, route, c, nullptr);
}

kd_status kd_op_moe_dispatch(const kd_attr_moe_dispatch* a, const void* h, const void* route, void* xg, void* meta,
                             void* stream) {
  if (!a) return fail(KD_ERR_INVALID_ARG, "kd_op_moe_dispatch: NULL attrs");
  LaunchCtx c;
  c.stream = (cudaStream_t)stream;
  return launch_moe_dispatch(*a, h, route, xg, meta, c, nullptr);
}

kd_status kd_op_moe_combine(const kd_attr_moe_combine* a, const void* yg, const void* route, const void* meta,
                            void* out, void* stream) {
  if (!a) return fail(KD_ERR_INVALID_ARG, "kd_op_moe_combine: NULL attrs");
  if (a->n_parts > 1) return fail(KD_ERR_UNSUPPORTED, "kd_op_moe_combine: one yg (n_parts <= 1) through the single-op call");
  LaunchCtx c;
  c.stream = (cudaStream_t)stream;
  const void* parts[1] = {yg};
  return launch_moe_combine(*a, parts, route, meta, out, c, nullptr);
}

}  // extern "C"
