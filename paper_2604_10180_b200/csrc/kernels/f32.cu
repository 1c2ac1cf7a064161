// f32.cu — the fp32 path (BASELINE north star "1e-5 for the fp32
// path"): every kernel of the dense decoder layer with fp32 activations,
// weights and KV cache and fp32 accumulation, for the 1e-5 parity check
// against the oracle's act="fp32" mode. tcgen05 has no fp32 kind (tf32 only,
// ~1e-3), so the GEMM is a SIMT FFMA kernel; attention is a plain per-(row,
// head) softmax. These serve parity sizes (tiny config) — the throughput path
// is bf16. Every reduction runs in a fixed order: bitwise deterministic, so
// disaggregated == monolithic holds bit for bit on this path too.
//
// The launchers are reached from the bf16 launchers when attrs.dtype ==
// KD_F32 (same C ABI entry points, same signal counting).
#include <cmath>

#include "launch.hpp"

namespace kd {
namespace f32 {

constexpr int kThreads = 256;

__device__ __forceinline__ float block_sum_fixed(float v, float* red) {
  // warp butterfly, then warps in index order: deterministic
  v = warp_sum(v);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
  __syncthreads();
  return t;
}

// ------------------------------------------------------------------ a3 (C1.1)
__global__ void __launch_bounds__(kThreads) add_rmsnorm_f32(float* __restrict__ r, DeltasF d,
                                                           const float* __restrict__ gamma, float* __restrict__ h,
                                                           int H, float eps, Epi epi) {
  __shared__ float red[kThreads / 32];
  pdl_launch_dependents();
  pdl_wait();
  float* rr = r + (size_t)blockIdx.x * H;
  float ss = 0.f;
  for (int i = threadIdx.x; i < H; i += kThreads) {
    float v = rr[i];
    for (int k = 0; k < d.n; ++k) v += d.p[k][(size_t)blockIdx.x * H + i];  // index order
    if (d.n) rr[i] = v;
    ss += v * v;
  }
  const float tot = block_sum_fixed(ss, red);
  const float inv = rsqrtf(tot / (float)H + eps);
  for (int i = threadIdx.x; i < H; i += kThreads) {
    const float o = rr[i] * inv * gamma[i];
    const size_t e = (size_t)blockIdx.x * H + i;
    h[e] = o;
    for (int p = 0; p < epi.n; ++p) ((float*)epi.dst[p])[e] = o;
  }
  epi_signal(epi);
}

// ------------------------------------------------------------------ C1.11
__global__ void residual_add_f32(float* __restrict__ r, DeltasF d, size_t n, Epi epi) {
  pdl_launch_dependents();
  pdl_wait();
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float v = r[i];
    for (int k = 0; k < d.n; ++k) v += d.p[k][i];
    r[i] = v;
    for (int p = 0; p < epi.n; ++p) ((float*)epi.dst[p])[i] = v;
  }
  epi_signal(epi);
}

// ------------------------------------------------------------------ a8 (C1.9)
__global__ void silu_mul_f32(const float* __restrict__ gu, float* __restrict__ out, int rows, int F, Epi epi) {
  pdl_launch_dependents();
  pdl_wait();
  const size_t n = (size_t)rows * F;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < n; t += (size_t)gridDim.x * blockDim.x) {
    const int row = (int)(t / F), col = (int)(t % F), j = col / 64, i = col % 64;
    const float g = gu[(size_t)row * 2 * F + 128 * j + i], u = gu[(size_t)row * 2 * F + 128 * j + 64 + i];
    const float o = g / (1.f + expf(-g)) * u;
    out[t] = o;
    for (int p = 0; p < epi.n; ++p) ((float*)epi.dst[p])[t] = o;
  }
  epi_signal(epi);
}

// ------------------------------------------------------------------ a5 (C1.3-4)
struct Freq {
  double f[128];
};
__global__ void rope_append_f32(const float* __restrict__ qkv, const int32_t* __restrict__ bt,
                                const int32_t* __restrict__ sl, float* __restrict__ q_out, float* __restrict__ kc,
                                float* __restrict__ vc, int Hq, int Hkv, int D, int page, int pps,
                                const __grid_constant__ Freq fr, Epi epi) {
  pdl_launch_dependents();
  pdl_wait();
  // CTA (row b, y) owns heads [8y, 8y+8) of [q heads | k heads | v heads]
  const int b = blockIdx.x, half = D / 2, G = Hq / Hkv;
  const int h0 = blockIdx.y * 8, h1 = min(h0 + 8, Hq + 2 * Hkv);
  const int pos = sl[b] - 1;
  const int32_t pg = bt[(size_t)b * pps + pos / page];
  const int off = pos % page;
  const float* src = qkv + (size_t)b * (Hq + 2 * Hkv) * D;
  const int r1 = min(h1, Hq + Hkv);
  for (int t = threadIdx.x; t < (r1 - h0) * half; t += blockDim.x) {
    const int hh = h0 + t / half, i = t % half;
    const double ang = (double)pos * fr.f[i];
    const double k = rint(ang * 0.15915494309189535);
    const double red = fma(-k, 6.283185307179586, fma(-k, 2.4492935982947064e-16, ang));
    float s, c;
    sincosf((float)red, &s, &c);
    const float* x;
    float* dst;
    size_t qoff = 0;
    const bool is_q = hh < Hq;
    if (is_q) {
      x = src + (size_t)(hh / G) * (G + 2) * D + (size_t)(hh % G) * D;
      qoff = (size_t)b * Hq * D + (size_t)hh * D;
      dst = q_out + qoff;
    } else {
      const int g = hh - Hq;
      x = src + (size_t)g * (G + 2) * D + (size_t)G * D;
      dst = kc + (((size_t)pg * Hkv + g) * page + off) * D;
    }
    const float x0 = x[i], y0 = x[i + half];
    const float lo = x0 * c - y0 * s, hi = y0 * c + x0 * s;
    dst[i] = lo;
    dst[i + half] = hi;
    if (is_q)
      for (int p = 0; p < epi.n; ++p) {
        ((float*)epi.dst[p])[qoff + i] = lo;
        ((float*)epi.dst[p])[qoff + i + half] = hi;
      }
  }
  const int v0 = max(h0, Hq + Hkv);
  for (int t = threadIdx.x; t < max(0, h1 - v0) * D; t += blockDim.x) {
    const int g = v0 - (Hq + Hkv) + t / D, dd = t % D;
    vc[(((size_t)pg * Hkv + g) * page + off) * D + dd] = src[(size_t)g * (G + 2) * D + (size_t)(G + 1) * D + dd];
  }
  epi_signal(epi);
}

// ------------------------------------------------------------------ a6 (C1.5)
// one CTA per (sequence, q head): scores → smem, max, exp + sum, then thread d
// accumulates Σ_t p_t·v_t[d] in key order
constexpr int kAttnThreads = 128;
__global__ void __launch_bounds__(kAttnThreads)
    attention_f32(const float* __restrict__ q, const float* __restrict__ kc, const float* __restrict__ vc,
                  const int32_t* __restrict__ bt, const int32_t* __restrict__ sl, float* __restrict__ out, int Hq,
                  int Hkv, int D, int page, int pps, Epi epi) {
  extern __shared__ float sm[];  // [D] q, [C] scores
  __shared__ float red[kAttnThreads / 32];
  pdl_launch_dependents();
  pdl_wait();
  const int b = blockIdx.x / Hq, h = blockIdx.x % Hq, g = h / (Hq / Hkv);
  const int len = sl[b];
  float* qs = sm;
  float* s = sm + D;
  for (int d = threadIdx.x; d < D; d += blockDim.x) qs[d] = q[((size_t)b * Hq + h) * D + d];
  __syncthreads();
  const float scale = 1.f / sqrtf((float)D);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int t = w; t < len; t += nw) {
    const int pg = bt[(size_t)b * pps + t / page];
    const float* k = kc + (((size_t)pg * Hkv + g) * page + t % page) * D;
    float acc = 0.f;
    for (int d = lane; d < D; d += 32) acc += qs[d] * k[d];
    acc = warp_sum(acc);
    if (lane == 0) s[t] = acc * scale;
  }
  __syncthreads();
  float mx = -INFINITY;
  for (int t = threadIdx.x; t < len; t += blockDim.x) mx = fmaxf(mx, s[t]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) red[w] = mx;
  __syncthreads();
  mx = red[0];
  for (int i = 1; i < nw; ++i) mx = fmaxf(mx, red[i]);
  __syncthreads();
  float part = 0.f;
  for (int t = threadIdx.x; t < len; t += blockDim.x) {
    const float p = expf(s[t] - mx);
    s[t] = p;
    part += p;
  }
  const float tot = block_sum_fixed(part, red);  // also orders the s[] writes before the reads below
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    float acc = 0.f;
    for (int t = 0; t < len; ++t) {
      const int pg = bt[(size_t)b * pps + t / page];
      acc += s[t] * vc[(((size_t)pg * Hkv + g) * page + t % page) * D + d];
    }
    const float o = acc / tot;
    const size_t e = ((size_t)b * Hq + h) * D + d;
    out[e] = o;
    for (int p = 0; p < epi.n; ++p) ((float*)epi.dst[p])[e] = o;
  }
  epi_signal(epi);
}

// ------------------------------------------------------------------ a4/a7/a9/a10 (C1.2)
// one warp per output feature n; lanes stride K; every token row in turn
constexpr int kGemmWarps = 8;
__global__ void __launch_bounds__(kGemmWarps * 32)
    gemm_f32(const float* __restrict__ X, const float* __restrict__ W, float* __restrict__ Y, int M, int N, int K,
             Epi epi) {
  pdl_launch_dependents();
  pdl_wait();
  const int n = blockIdx.x * kGemmWarps + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (n < N) {
    const float* w = W + (size_t)n * K;
    for (int m = 0; m < M; ++m) {
      const float* x = X + (size_t)m * K;
      float acc = 0.f;
      for (int k = lane; k < K; k += 32) acc += x[k] * w[k];
      acc = warp_sum(acc);
      if (lane == 0) {
        const size_t e = (size_t)m * N + n;
        Y[e] = acc;
        for (int p = 0; p < epi.n; ++p) ((float*)epi.dst[p])[e] = acc;
      }
    }
  }
  epi_signal(epi);
}

}  // namespace f32

// ------------------------------------------------------------------ launchers (dtype == KD_F32)
kd_status launch_add_rmsnorm_f32(const kd_attr_add_rmsnorm& a, float* r, const DeltasF& d, const float* gamma,
                                 float* h, const LaunchCtx& c, uint32_t* signals) {
  if (a.rows == 0 || a.hidden == 0) return fail(KD_ERR_UNSUPPORTED, "add_rmsnorm (fp32): empty shape");
  if (!r || !gamma || !h) return fail(KD_ERR_INVALID_ARG, "add_rmsnorm (fp32): NULL pointer");
  KD_CUDA_CHECK(kd_launch(f32::add_rmsnorm_f32, dim3(a.rows), dim3(f32::kThreads), 0, c.stream, r, d, gamma, h,
                          (int)a.hidden, a.eps, c.epi),
                "add_rmsnorm (fp32) launch");
  if (signals) *signals = a.rows;
  return KD_OK;
}

kd_status launch_residual_add_f32(float* r, const DeltasF& d, size_t n, int grid, const LaunchCtx& c) {
  KD_CUDA_CHECK(kd_launch(f32::residual_add_f32, dim3(grid), dim3(256), 0, c.stream, r, d, n, c.epi),
                "residual_add (fp32) launch");
  return KD_OK;
}

kd_status launch_silu_mul_f32(const kd_attr_silu_mul& a, const float* gu, float* out, int grid, const LaunchCtx& c) {
  KD_CUDA_CHECK(kd_launch(f32::silu_mul_f32, dim3(grid), dim3(256), 0, c.stream, gu, out, (int)a.rows, (int)a.ffn,
                          c.epi),
                "silu_mul (fp32) launch");
  return KD_OK;
}

kd_status launch_rope_append_f32(const kd_attr_rope_append& a, const float* qkv, const int32_t* bt, const int32_t* sl,
                                 float* q_out, float* kc, float* vc, dim3 grid, const LaunchCtx& c) {
  f32::Freq fr;
  const double l2t = std::log2(a.theta);
  for (uint32_t i = 0; i < a.head_dim / 2; ++i) fr.f[i] = std::exp2(-2.0 * (double)i / (double)a.head_dim * l2t);
  KD_CUDA_CHECK(kd_launch(f32::rope_append_f32, grid, dim3(256), 0, c.stream, qkv, bt, sl, q_out, kc, vc,
                          (int)a.n_heads, (int)a.n_kv_heads, (int)a.head_dim, (int)a.page, (int)a.pages_per_seq, fr,
                          c.epi),
                "rope_append (fp32) launch");
  return KD_OK;
}

uint32_t attention_f32_signals(const kd_attr_attention& a) { return a.rows * a.n_heads; }

kd_status launch_attention_f32(const kd_attr_attention& a, const float* q, const float* kc, const float* vc,
                               const int32_t* bt, const int32_t* sl, float* out, const LaunchCtx& c) {
  const size_t C = (size_t)a.pages_per_seq * a.page;
  const size_t smem = (a.head_dim + C) * sizeof(float);
  if (smem > 200 * 1024) return fail(KD_ERR_UNSUPPORTED, "attention (fp32): context too long for the parity kernel");
  if (smem > 48 * 1024)
    KD_CUDA_CHECK(cudaFuncSetAttribute(f32::attention_f32, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                  "attention (fp32) smem attr");
  KD_CUDA_CHECK(kd_launch(f32::attention_f32, dim3(a.rows * a.n_heads), dim3(f32::kAttnThreads), smem, c.stream, q,
                          kc, vc, bt, sl, out, (int)a.n_heads, (int)a.n_kv_heads, (int)a.head_dim, (int)a.page,
                          (int)a.pages_per_seq, c.epi),
                "attention (fp32) launch");
  return KD_OK;
}

uint32_t gemm_f32_signals(uint32_t N) { return (N + f32::kGemmWarps - 1) / f32::kGemmWarps; }

kd_status launch_gemm_f32(const float* X, const float* W, float* Y, int M, int N, int K, const LaunchCtx& c) {
  KD_CUDA_CHECK(kd_launch(f32::gemm_f32, dim3(gemm_f32_signals((uint32_t)N)), dim3(f32::kGemmWarps * 32), 0, c.stream,
                          X, W, Y, M, N, K, c.epi),
                "gemm (fp32) launch");
  return KD_OK;
}

}  // namespace kd
