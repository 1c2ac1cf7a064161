// moe.cu — Mixture-of-Experts decode kernels (C1.12):
//   route    logits = h·W_rᵀ (fp32), top-k by logit (ties → lower expert),
//            weights = softmax over the k selected logits
//   dispatch expert-major slot map + gather of the routed rows (xg)
//   combine  out_b = Σ_j w_bj · yg[slot_bj] in ascending expert order
// The expert FFN itself is two grouped tcgen05 GEMMs (gemm.cu, groups = E)
// around the SiLU·mul kernel. All memory-bound; everything deterministic.
#include "launch.hpp"

namespace kd {
namespace moe {

constexpr int kMaxE = 32;
constexpr int kMaxK = 4;
constexpr int kMaxSlots = 4096;  // rows * top_k handled by one slot map

// meta layout (int32): count[E] | offset[E] | slot_of[rows*k] | row_of[rows*k]
__host__ __device__ inline size_t meta_ints(int rows, int E, int k) { return 2 * (size_t)E + 2 * (size_t)rows * k; }

__global__ void __launch_bounds__(256) route_kernel(const __nv_bfloat16* __restrict__ h, const float* __restrict__ wr,
                                                    int32_t* __restrict__ idx_out, float* __restrict__ w_out, int H,
                                                    int E, int k, Epi epi) {
  pdl_launch_dependents();
  pdl_wait();
  __shared__ float logits[kMaxE];
  const int row = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const __nv_bfloat16* hr = h + (size_t)row * H;
  for (int e = warp; e < E; e += 8) {
    const float* w = wr + (size_t)e * H;
    float acc = 0.f;
    // 4 column chunks per round with every load in flight before the FMAs (the
    // serial load → FMA chain was latency-bound); same summation order
    for (int c0 = lane * 8; c0 < H; c0 += 4 * 256) {
      uint4 hv[4];
      float4 w0[4], w1[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = c0 + u * 256;
        if (c < H) {
          hv[u] = *reinterpret_cast<const uint4*>(hr + c);
          w0[u] = *reinterpret_cast<const float4*>(w + c);
          w1[u] = *reinterpret_cast<const float4*>(w + c + 4);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (c0 + u * 256 < H)
          acc += bf16lo(hv[u].x) * w0[u].x + bf16hi(hv[u].x) * w0[u].y + bf16lo(hv[u].y) * w0[u].z +
                 bf16hi(hv[u].y) * w0[u].w + bf16lo(hv[u].z) * w1[u].x + bf16hi(hv[u].z) * w1[u].y +
                 bf16lo(hv[u].w) * w1[u].z + bf16hi(hv[u].w) * w1[u].w;
    }
    acc = warp_sum(acc);  // fixed butterfly order: deterministic
    if (lane == 0) logits[e] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int sel[kMaxK];
    float lv[kMaxK];
    unsigned used = 0;
    for (int j = 0; j < k; ++j) {
      int best = -1;
      for (int e = 0; e < E; ++e)  // strict '>' keeps the lower index on ties
        if (!((used >> e) & 1u) && (best < 0 || logits[e] > logits[best])) best = e;
      sel[j] = best;
      lv[j] = logits[best];
      used |= 1u << best;
    }
    float z = 0.f, p[kMaxK];
    for (int j = 0; j < k; ++j) {
      p[j] = __expf(lv[j] - lv[0]);
      z += p[j];
    }
    for (int j = 0; j < k; ++j) {
      idx_out[(size_t)row * k + j] = sel[j];
      w_out[(size_t)row * k + j] = p[j] / z;
    }
  }
  epi_signal(epi);  // (route is never cut in the decoder graph; kept for uniformity)
}

__global__ void __launch_bounds__(256) dispatch_kernel(const __nv_bfloat16* __restrict__ h,
                                                       const int32_t* __restrict__ idx, __nv_bfloat16* __restrict__ xg,
                                                       int32_t* __restrict__ meta, int rows, int H, int E, int k,
                                                       size_t meta_bytes, Epi epi) {
  // the primary output is the whole [meta | xg] block: peers get both, at the
  // same offsets from their landing slot base (= this block's base)
  pdl_launch_dependents();
  pdl_wait();
  __shared__ int cnt[kMaxE], off[kMaxE];
  __shared__ int16_t row_of[kMaxSlots];
  const int n = rows * k;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  // every CTA derives the same slot map (tiny), so no grid-wide sync is needed.
  // Warp w takes experts w, w+nw, …: one ballot per 32 entries counts them
  // (was a serial per-expert scan: ≈35 µs at 256 entries)
  for (int e = warp; e < E; e += nw) {
    int c = 0;
    for (int s0 = 0; s0 < n; s0 += 32) {
      const int s = s0 + lane;
      c += __popc(__ballot_sync(0xffffffffu, s < n && idx[s] == e));
    }
    if (lane == 0) cnt[e] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int o = 0;
    for (int e = 0; e < E; ++e) {
      off[e] = o;
      o += cnt[e];
    }
  }
  __syncthreads();
  // positions: entries in (row, choice) order, i.e. ascending rows inside an
  // expert — the ballot prefix keeps that order (same map as the serial scan)
  for (int e = warp; e < E; e += nw) {
    int pos = off[e];
    for (int s0 = 0; s0 < n; s0 += 32) {
      const int s = s0 + lane;
      const bool hit = s < n && idx[s] == e;
      const unsigned m = __ballot_sync(0xffffffffu, hit);
      if (hit) {
        const int p = pos + __popc(m & ((1u << lane) - 1u));
        row_of[p] = (int16_t)(s / k);
        if (blockIdx.x == 0) meta[2 * E + s] = p;  // slot_of
      }
      pos += __popc(m);
    }
  }
  __syncthreads();
  if (blockIdx.x == 0) {
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
      meta[e] = cnt[e];
      meta[E + e] = off[e];
    }
    for (int s = threadIdx.x; s < n; s += blockDim.x) meta[2 * E + n + s] = row_of[s];
    if (epi.n) {
      __syncthreads();
      const int total = (int)(2 * E + 2 * n);
      for (int i = threadIdx.x; i < total; i += blockDim.x) {
        const int32_t v = meta[i];
        for (int p = 0; p < epi.n; ++p) ((int32_t*)epi.dst[p])[i] = v;
      }
    }
  }
  // gather: grid-stride over (slot, 16-byte vector)
  const int vpr = H / 8;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < (size_t)n * vpr;
       t += (size_t)gridDim.x * blockDim.x) {
    const int s = (int)(t / vpr), v = (int)(t % vpr);
    const uint4 x = reinterpret_cast<const uint4*>(h + (size_t)row_of[s] * H)[v];
    reinterpret_cast<uint4*>(xg + (size_t)s * H)[v] = x;
    for (int p = 0; p < epi.n; ++p)
      reinterpret_cast<uint4*>((__nv_bfloat16*)((uint8_t*)epi.dst[p] + meta_bytes) + (size_t)s * H)[v] = x;
  }
  epi_signal(epi);
}

constexpr int kMaxParts = 8;
struct YParts {  // expert-parallel combine: expert e's rows live in part e / per_part
  const __nv_bfloat16* p[kMaxParts];
  int per_part;
};

__global__ void __launch_bounds__(256) combine_kernel(YParts ys, const int32_t* __restrict__ idx,
                                                      const float* __restrict__ w, const int32_t* __restrict__ meta,
                                                      __nv_bfloat16* __restrict__ out, int H, int E, int k, Epi epi) {
  pdl_launch_dependents();
  pdl_wait();
  const int row = blockIdx.x;
  // choices of this row in ascending expert order (the oracle's summation order)
  int ord[kMaxK];
  for (int j = 0; j < k; ++j) ord[j] = j;
  for (int a = 1; a < k; ++a)
    for (int b = a; b > 0 && idx[(size_t)row * k + ord[b]] < idx[(size_t)row * k + ord[b - 1]]; --b) {
      int t = ord[b];
      ord[b] = ord[b - 1];
      ord[b - 1] = t;
    }
  const int32_t* slot_of = meta + 2 * E;
  for (int c = threadIdx.x * 8; c < H; c += blockDim.x * 8) {
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int jj = 0; jj < k; ++jj) {
      const int j = ord[jj];
      const float wj = w[(size_t)row * k + j];
      const __nv_bfloat16* yg = ys.p[idx[(size_t)row * k + j] / ys.per_part];
      const uint4 y = *reinterpret_cast<const uint4*>(yg + (size_t)slot_of[(size_t)row * k + j] * H + c);
      acc[0] += wj * bf16lo(y.x);
      acc[1] += wj * bf16hi(y.x);
      acc[2] += wj * bf16lo(y.y);
      acc[3] += wj * bf16hi(y.y);
      acc[4] += wj * bf16lo(y.z);
      acc[5] += wj * bf16hi(y.z);
      acc[6] += wj * bf16lo(y.w);
      acc[7] += wj * bf16hi(y.w);
    }
    uint4 o;
    o.x = pack_bf16(acc[0], acc[1]);
    o.y = pack_bf16(acc[2], acc[3]);
    o.z = pack_bf16(acc[4], acc[5]);
    o.w = pack_bf16(acc[6], acc[7]);
    *reinterpret_cast<uint4*>(out + (size_t)row * H + c) = o;
    for (int p = 0; p < epi.n; ++p) *reinterpret_cast<uint4*>((__nv_bfloat16*)epi.dst[p] + (size_t)row * H + c) = o;
  }
  epi_signal(epi);
}

static kd_status check(uint32_t rows, uint32_t H, uint32_t E, uint32_t k) {
  if (rows == 0 || H == 0 || H % 8 || E == 0 || E > (uint32_t)kMaxE || k == 0 || k > (uint32_t)kMaxK || k > E)
    return fail(KD_ERR_UNSUPPORTED, "moe: need H % 8 == 0, 1 <= top_k <= 4, top_k <= experts <= 32");
  if ((uint64_t)rows * k > (uint64_t)kMaxSlots || rows > 32767)
    return fail(KD_ERR_UNSUPPORTED, "moe: rows * top_k must be <= 4096");
  return KD_OK;
}

static int dispatch_grid(uint32_t rows, uint32_t H, uint32_t k) {
  const size_t vec = (size_t)rows * k * (H / 8);
  return (int)std::max<size_t>(1, std::min<size_t>((vec + 255) / 256, kNumSMs));
}

}  // namespace moe

kd_status launch_moe_route(const kd_attr_moe_route& a, const void* h, const float* wr, void* route, const LaunchCtx& c,
                           uint32_t* signals) {
  kd_status s = moe::check(a.rows, a.hidden, a.experts, a.top_k);
  if (s) return s;
  if (!h || !wr || !route) return fail(KD_ERR_INVALID_ARG, "moe_route: NULL pointer");
  int32_t* idx = (int32_t*)route;
  float* w = (float*)(idx + (size_t)a.rows * a.top_k);
  KD_CUDA_CHECK(kd_launch(moe::route_kernel, dim3(a.rows), dim3(256), 0, c.stream, (const __nv_bfloat16*)h, wr, idx, w,
                          (int)a.hidden, (int)a.experts, (int)a.top_k, c.epi),
                "moe_route launch");
  if (signals) *signals = a.rows;
  return KD_OK;
}

kd_status launch_moe_dispatch(const kd_attr_moe_dispatch& a, const void* h, const void* route, void* xg, void* meta,
                              const LaunchCtx& c, uint32_t* signals) {
  kd_status s = moe::check(a.rows, a.hidden, a.experts, a.top_k);
  if (s) return s;
  if (!h || !route || !xg || !meta) return fail(KD_ERR_INVALID_ARG, "moe_dispatch: NULL pointer");
  const int grid = moe::dispatch_grid(a.rows, a.hidden, a.top_k);
  // peers mirror [meta | xg]: only valid when xg directly follows the meta block
  const size_t meta_bytes = (size_t)((uint8_t*)xg - (uint8_t*)meta);
  if (c.epi.n && meta_bytes != (moe::meta_ints(a.rows, a.experts, a.top_k) * 4 + 255) / 256 * 256)
    return fail(KD_ERR_UNSUPPORTED, "moe_dispatch: peer stores need the [meta | xg] block layout");
  KD_CUDA_CHECK(kd_launch(moe::dispatch_kernel, dim3(grid), dim3(256), 0, c.stream, (const __nv_bfloat16*)h,
                          (const int32_t*)route, (__nv_bfloat16*)xg, (int32_t*)meta, (int)a.rows, (int)a.hidden,
                          (int)a.experts, (int)a.top_k, meta_bytes, c.epi),
                "moe_dispatch launch");
  if (signals) *signals = (uint32_t)grid;
  return KD_OK;
}

kd_status launch_moe_combine(const kd_attr_moe_combine& a, const void* const* ygs, const void* route, const void* meta,
                             void* out, const LaunchCtx& c, uint32_t* signals) {
  kd_status s = moe::check(a.rows, a.hidden, a.experts, a.top_k);
  if (s) return s;
  const uint32_t np = a.n_parts ? a.n_parts : 1;
  if (np > (uint32_t)moe::kMaxParts || a.experts % np)
    return fail(KD_ERR_UNSUPPORTED, "moe_combine: n_parts must divide experts (<= 8 parts)");
  if (!ygs || !route || !meta || !out) return fail(KD_ERR_INVALID_ARG, "moe_combine: NULL pointer");
  moe::YParts ys{};
  ys.per_part = (int)(a.experts / np);
  for (uint32_t i = 0; i < np; ++i) {
    if (!ygs[i]) return fail(KD_ERR_INVALID_ARG, "moe_combine: NULL yg part");
    ys.p[i] = (const __nv_bfloat16*)ygs[i];
  }
  const int32_t* idx = (const int32_t*)route;
  const float* w = (const float*)(idx + (size_t)a.rows * a.top_k);
  KD_CUDA_CHECK(kd_launch(moe::combine_kernel, dim3(a.rows), dim3(256), 0, c.stream, ys, idx, w,
                          (const int32_t*)meta, (__nv_bfloat16*)out, (int)a.hidden, (int)a.experts, (int)a.top_k,
                          c.epi),
                "moe_combine launch");
  if (signals) *signals = a.rows;
  return KD_OK;
}

kd_status moe_signals(uint32_t op, const std::vector<uint8_t>& attrs, uint32_t* s) {
  if (attrs.size() != (op == KD_OP_MOE_COMBINE ? sizeof(kd_attr_moe_combine) : 16))
    return fail(KD_ERR_INVALID_ARG, "moe: attrs have the wrong size");
  uint32_t v[4];
  std::memcpy(v, attrs.data(), 16);
  *s = (op == KD_OP_MOE_DISPATCH) ? (uint32_t)moe::dispatch_grid(v[0], v[1], v[3]) : v[0];
  return KD_OK;
}

}  // namespace kd

extern "C" kd_status kd_moe_meta_bytes(uint32_t rows, uint32_t experts, uint32_t top_k, uint64_t* bytes) {
  if (!bytes) return kd::fail(KD_ERR_INVALID_ARG, "kd_moe_meta_bytes: NULL argument");
  *bytes = (kd::moe::meta_ints(rows, experts, top_k) * 4 + 255) / 256 * 256;
  return KD_OK;
}
