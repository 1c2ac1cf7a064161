// ssm.cu — Mamba-2 decode kernels (C1.13): causal-conv
// state update, selective-state update, gated RMSNorm. All HBM-bound; the
// selective-state update dominates (fp32 state read + written once: 2 ×
// rows·nheads·head_dim·N·4 bytes, 512 MiB at the hybrid config).
#include "launch.hpp"

namespace kd {
namespace ssm {

struct Dims {
  int rows, nh, P, N, G, W, di, ch, pin;
};
static Dims dims(const kd_attr_ssm& a) {
  Dims d;
  d.rows = a.rows;
  d.nh = a.nheads;
  d.P = a.head_dim;
  d.N = a.d_state;
  d.G = a.ngroups;
  d.W = a.d_conv;
  d.di = a.nheads * a.head_dim;
  d.ch = d.di + 2 * d.G * d.N;
  d.pin = 2 * d.di + 2 * d.G * d.N + d.nh;
  return d;
}

__device__ __forceinline__ float silu_f(float x) { return x / (1.f + __expf(-x)); }
__device__ __forceinline__ float softplus_f(float x) { return x > 20.f ? x : log1pf(__expf(x)); }

// one thread per (row, channel); window = [state (W-1, oldest first), x]
__global__ void conv_kernel(const __nv_bfloat16* __restrict__ zx, const __nv_bfloat16* __restrict__ w,
                            const __nv_bfloat16* __restrict__ bias, __nv_bfloat16* __restrict__ state,
                            __nv_bfloat16* __restrict__ out, Dims d, Epi epi) {
  pdl_launch_dependents();
  pdl_wait();
  const size_t n = (size_t)d.rows * d.ch;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < n; t += (size_t)gridDim.x * blockDim.x) {
    const int b = (int)(t / d.ch), c = (int)(t % d.ch);
    const float x = __bfloat162float(zx[(size_t)b * d.pin + d.di + c]);
    __nv_bfloat16* st = state + t * (d.W - 1);
    float acc = __bfloat162float(bias[c]);
    float prev[8];
    for (int k = 0; k < d.W - 1; ++k) {
      prev[k] = __bfloat162float(st[k]);
      acc += prev[k] * __bfloat162float(w[(size_t)c * d.W + k]);
    }
    acc += x * __bfloat162float(w[(size_t)c * d.W + d.W - 1]);
    for (int k = 0; k < d.W - 2; ++k) st[k] = __float2bfloat16_rn(prev[k + 1]);
    st[d.W - 2] = __float2bfloat16_rn(x);
    const __nv_bfloat16 o = __float2bfloat16_rn(silu_f(acc));
    out[t] = o;
    for (int p = 0; p < epi.n; ++p) ((__nv_bfloat16*)epi.dst[p])[t] = o;
  }
  epi_signal(epi);
}

// 8 channels per thread (16-byte loads of x, the 3-deep state, the 4 taps and
// the bias): the same per-channel arithmetic as conv_kernel, in the same
// order (bitwise equal); used when d_conv == 4 and the rows are 16-byte aligned
__global__ void conv8_kernel(const __nv_bfloat16* __restrict__ zx, const __nv_bfloat16* __restrict__ w,
                             const __nv_bfloat16* __restrict__ bias, __nv_bfloat16* __restrict__ state,
                             __nv_bfloat16* __restrict__ out, Dims d, Epi epi) {
  pdl_launch_dependents();
  pdl_wait();
  const int c8n = d.ch / 8;
  const size_t n = (size_t)d.rows * c8n;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < n; t += (size_t)gridDim.x * blockDim.x) {
    const int b = (int)(t / c8n), c0 = (int)(t % c8n) * 8;
    const uint4 xv = *reinterpret_cast<const uint4*>(zx + (size_t)b * d.pin + d.di + c0);
    const size_t e0 = (size_t)b * d.ch + c0;                    // first element of this thread's 8 channels
    uint4 sv[3], wv[4];
#pragma unroll
    for (int i = 0; i < 3; ++i) sv[i] = reinterpret_cast<const uint4*>(state + e0 * 3)[i];   // [8 ch][3]
#pragma unroll
    for (int i = 0; i < 4; ++i) wv[i] = reinterpret_cast<const uint4*>(w + (size_t)c0 * 4)[i];  // [8 ch][4]
    const uint4 bv = *reinterpret_cast<const uint4*>(bias + c0);
    const __nv_bfloat16* xs = reinterpret_cast<const __nv_bfloat16*>(&xv);
    const __nv_bfloat16* ss = reinterpret_cast<const __nv_bfloat16*>(sv);
    const __nv_bfloat16* ws = reinterpret_cast<const __nv_bfloat16*>(wv);
    const __nv_bfloat16* bs = reinterpret_cast<const __nv_bfloat16*>(&bv);
    __align__(16) __nv_bfloat16 ns[24];
    __align__(16) __nv_bfloat16 o[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float x = __bfloat162float(xs[j]);
      float acc = __bfloat162float(bs[j]);
      float prev[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        prev[k] = __bfloat162float(ss[j * 3 + k]);
        acc += prev[k] * __bfloat162float(ws[j * 4 + k]);
      }
      acc += x * __bfloat162float(ws[j * 4 + 3]);
      ns[j * 3 + 0] = __float2bfloat16_rn(prev[1]);
      ns[j * 3 + 1] = __float2bfloat16_rn(prev[2]);
      ns[j * 3 + 2] = __float2bfloat16_rn(x);
      o[j] = __float2bfloat16_rn(silu_f(acc));
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) reinterpret_cast<uint4*>(state + e0 * 3)[i] = reinterpret_cast<const uint4*>(ns)[i];
    const uint4 ov = *reinterpret_cast<const uint4*>(o);
    *reinterpret_cast<uint4*>(out + e0) = ov;
    for (int p = 0; p < epi.n; ++p) *reinterpret_cast<uint4*>((__nv_bfloat16*)epi.dst[p] + e0) = ov;
  }
  epi_signal(epi);
}

// one CTA per (head, row): S [P][N] fp32; 4 threads per state row, each owning
// N/4 columns as interleaved float4s (lanes of a quad read 64 contiguous bytes)
template <int P, int N>
__global__ void __launch_bounds__(P * 4) update_kernel(const __nv_bfloat16* __restrict__ xbc,
                                                       const __nv_bfloat16* __restrict__ zx,
                                                       const float* __restrict__ dt_bias,
                                                       const float* __restrict__ A_log, const float* __restrict__ Dp,
                                                       float* __restrict__ state, __nv_bfloat16* __restrict__ y,
                                                       Dims d, Epi epi) {
  pdl_launch_dependents();
  constexpr int V = N / 16;  // float4s per thread
  __shared__ float sB[N], sC[N];
  const int h = blockIdx.x, b = blockIdx.y;
  const int p = threadIdx.x >> 2, q = threadIdx.x & 3;
  const int g = h / (d.nh / d.G);
  const float dtb = dt_bias[h], A = -__expf(A_log[h]), Dh = Dp[h];  // weights: before the wait
  pdl_wait();
  const __nv_bfloat16* row = xbc + (size_t)b * d.ch;
  for (int n = threadIdx.x; n < N; n += blockDim.x) {
    sB[n] = __bfloat162float(row[d.di + g * N + n]);
    sC[n] = __bfloat162float(row[d.di + d.G * N + g * N + n]);
  }
  float4* S = reinterpret_cast<float4*>(state + (((size_t)b * d.nh + h) * P + p) * N);
  float4 s[V];
#pragma unroll
  for (int i = 0; i < V; ++i) s[i] = S[i * 4 + q];
  const float dt = softplus_f(__bfloat162float(zx[(size_t)b * d.pin + 2 * d.di + 2 * d.G * N + h]) + dtb);
  const float dA = __expf(dt * A);
  const float x = __bfloat162float(row[h * P + p]);
  const float dx = dt * x;
  __syncthreads();
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int n0 = (i * 4 + q) * 4;
    s[i].x = s[i].x * dA + dx * sB[n0 + 0];
    s[i].y = s[i].y * dA + dx * sB[n0 + 1];
    s[i].z = s[i].z * dA + dx * sB[n0 + 2];
    s[i].w = s[i].w * dA + dx * sB[n0 + 3];
    acc += s[i].x * sC[n0 + 0] + s[i].y * sC[n0 + 1] + s[i].z * sC[n0 + 2] + s[i].w * sC[n0 + 3];
    S[i * 4 + q] = s[i];
  }
  acc += __shfl_xor_sync(0xffffffffu, acc, 1);
  acc += __shfl_xor_sync(0xffffffffu, acc, 2);
  if (q == 0) {
    const __nv_bfloat16 o = __float2bfloat16_rn(acc + Dh * x);
    const size_t yi = (size_t)b * d.di + h * P + p;
    y[yi] = o;
    for (int pp = 0; pp < epi.n; ++pp) ((__nv_bfloat16*)epi.dst[pp])[yi] = o;
  }
  epi_signal(epi);
}

// one CTA per (row, group): g = y·silu(z); out = g·rsqrt(mean g² + eps)·w
__global__ void __launch_bounds__(256) gnorm_kernel(const __nv_bfloat16* __restrict__ y,
                                                    const __nv_bfloat16* __restrict__ zx,
                                                    const __nv_bfloat16* __restrict__ w,
                                                    __nv_bfloat16* __restrict__ out, Dims d, float eps, Epi epi) {
  pdl_launch_dependents();
  pdl_wait();
  const int b = blockIdx.x, grp = blockIdx.y;
  const int gs = d.di / d.G;
  const int c0 = grp * gs;
  __shared__ float red[8];
  float vals[16];
  float ss = 0.f;
  int cnt = 0;
  for (int c = threadIdx.x; c < gs && cnt < 16; c += blockDim.x, ++cnt) {
    const float yv = __bfloat162float(y[(size_t)b * d.di + c0 + c]);
    const float zv = __bfloat162float(zx[(size_t)b * d.pin + c0 + c]);
    const float gv = yv * silu_f(zv);
    vals[cnt] = gv;
    ss += gv * gv;
  }
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) tot += red[i];
  const float inv = rsqrtf(tot / (float)gs + eps);
  cnt = 0;
  for (int c = threadIdx.x; c < gs && cnt < 16; c += blockDim.x, ++cnt) {
    const __nv_bfloat16 o = __float2bfloat16_rn(vals[cnt] * inv * __bfloat162float(w[c0 + c]));
    const size_t oi = (size_t)b * d.di + c0 + c;
    out[oi] = o;
    for (int p = 0; p < epi.n; ++p) ((__nv_bfloat16*)epi.dst[p])[oi] = o;
  }
  epi_signal(epi);
}

static kd_status check(const kd_attr_ssm& a) {
  if (a.dtype != KD_BF16) return fail(KD_ERR_UNSUPPORTED, "ssm: only bf16 activations");
  if (a.rows == 0 || a.nheads == 0 || a.ngroups == 0 || a.nheads % a.ngroups || a.d_conv < 2 || a.d_conv > 8)
    return fail(KD_ERR_UNSUPPORTED, "ssm: need nheads % ngroups == 0 and 2 <= d_conv <= 8");
  const bool ok_pn = (a.head_dim == 64 && (a.d_state == 128 || a.d_state == 64)) ||
                     (a.head_dim == 32 && (a.d_state == 32 || a.d_state == 64 || a.d_state == 128));
  if (!ok_pn) return fail(KD_ERR_UNSUPPORTED, "ssm: (head_dim, d_state) in {64}x{64,128} or {32}x{32,64,128}");
  if ((a.nheads * a.head_dim / a.ngroups) > 256 * 16) return fail(KD_ERR_UNSUPPORTED, "ssm: group too large");
  return KD_OK;
}

// the 8-channel kernel when the shape allows (d_conv 4, channel counts and
// row pitches multiples of 8); decided from the attrs alone so the signal
// count (= grid) is known to the runtime
static bool conv8(const kd_attr_ssm& a) {
  const Dims d = dims(a);
  return d.W == 4 && d.ch % 8 == 0 && d.pin % 8 == 0 && d.di % 8 == 0;
}

static int conv_grid(const kd_attr_ssm& a) {
  const Dims d = dims(a);
  const size_t n = (size_t)d.rows * d.ch / (conv8(a) ? 8 : 1);
  return (int)std::max<size_t>(1, std::min<size_t>((n + 255) / 256, 8 * kNumSMs));
}

}  // namespace ssm

kd_status launch_ssm_conv(const kd_attr_ssm& a, const void* zx, const void* w, const void* bias, void* state,
                          void* out, const LaunchCtx& c, uint32_t* signals) {
  kd_status s = ssm::check(a);
  if (s) return s;
  if (!zx || !w || !bias || !state || !out) return fail(KD_ERR_INVALID_ARG, "ssm_conv: NULL pointer");
  const int grid = ssm::conv_grid(a);
  const bool v8 = ssm::conv8(a);
  if (v8 && (((uintptr_t)zx | (uintptr_t)w | (uintptr_t)bias | (uintptr_t)state | (uintptr_t)out) & 15))
    return fail(KD_ERR_INVALID_ARG, "ssm_conv: operands must be 16-byte aligned");
  KD_CUDA_CHECK(kd_launch(v8 ? ssm::conv8_kernel : ssm::conv_kernel, dim3(grid), dim3(256), 0, c.stream,
                          (const __nv_bfloat16*)zx,
                          (const __nv_bfloat16*)w, (const __nv_bfloat16*)bias, (__nv_bfloat16*)state,
                          (__nv_bfloat16*)out, ssm::dims(a), c.epi),
                "ssm_conv launch");
  if (signals) *signals = grid;
  return KD_OK;
}

kd_status launch_ssm_update(const kd_attr_ssm& a, const void* xbc, const void* zx, const float* dt_bias,
                            const float* A_log, const float* D, float* state, void* y, const LaunchCtx& c,
                            uint32_t* signals) {
  kd_status s = ssm::check(a);
  if (s) return s;
  if (!xbc || !zx || !dt_bias || !A_log || !D || !state || !y) return fail(KD_ERR_INVALID_ARG, "ssm_update: NULL pointer");
  const ssm::Dims d = ssm::dims(a);
  dim3 grid(a.nheads, a.rows);
  cudaError_t e;
#define KD_SSM_CASE(P_, N_)                                                                                        \
  if (a.head_dim == P_ && a.d_state == N_)                                                                         \
    e = kd_launch(ssm::update_kernel<P_, N_>, grid, dim3(P_ * 4), 0, c.stream, (const __nv_bfloat16*)xbc,          \
                  (const __nv_bfloat16*)zx, dt_bias, A_log, D, state, (__nv_bfloat16*)y, d, c.epi);               \
  else
  KD_SSM_CASE(64, 128) KD_SSM_CASE(64, 64) KD_SSM_CASE(32, 32) KD_SSM_CASE(32, 64) KD_SSM_CASE(32, 128)
  return fail(KD_ERR_UNSUPPORTED, "ssm_update: shape");
#undef KD_SSM_CASE
  KD_CUDA_CHECK(e, "ssm_update launch");
  if (signals) *signals = a.nheads * a.rows;
  return KD_OK;
}

kd_status launch_gated_norm(const kd_attr_ssm& a, const void* y, const void* zx, const void* w, void* out,
                            const LaunchCtx& c, uint32_t* signals) {
  kd_status s = ssm::check(a);
  if (s) return s;
  if (!y || !zx || !w || !out) return fail(KD_ERR_INVALID_ARG, "gated_norm: NULL pointer");
  KD_CUDA_CHECK(kd_launch(ssm::gnorm_kernel, dim3(a.rows, a.ngroups), dim3(256), 0, c.stream, (const __nv_bfloat16*)y,
                          (const __nv_bfloat16*)zx, (const __nv_bfloat16*)w, (__nv_bfloat16*)out, ssm::dims(a),
                          a.eps, c.epi),
                "gated_norm launch");
  if (signals) *signals = a.rows * a.ngroups;
  return KD_OK;
}

kd_status ssm_init_attrs() {
  const void* fns[] = {(const void*)ssm::conv_kernel, (const void*)ssm::conv8_kernel, (const void*)ssm::update_kernel<64, 128>,
                       (const void*)ssm::update_kernel<64, 64>, (const void*)ssm::update_kernel<32, 32>,
                       (const void*)ssm::update_kernel<32, 64>, (const void*)ssm::update_kernel<32, 128>,
                       (const void*)ssm::gnorm_kernel};
  for (const void* f : fns)
    KD_CUDA_CHECK(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100), "carveout");
  return KD_OK;
}

kd_status ssm_signals(uint32_t op, const std::vector<uint8_t>& attrs, uint32_t* s) {
  if (attrs.size() != sizeof(kd_attr_ssm)) return fail(KD_ERR_INVALID_ARG, "ssm: attrs have the wrong size");
  kd_attr_ssm a;
  std::memcpy(&a, attrs.data(), sizeof a);
  if (op == KD_OP_SSM_CONV) *s = (uint32_t)ssm::conv_grid(a);
  else if (op == KD_OP_SSM_UPDATE) *s = a.nheads * a.rows;
  else *s = a.rows * a.ngroups;
  return KD_OK;
}

}  // namespace kd

using namespace kd;

extern "C" {

kd_status kd_op_ssm_conv(const kd_attr_ssm* a, const void* zxbcdt, const void* conv_w, const void* conv_b,
                         void* conv_state, void* xbc, void* stream) {
  if (!a) return fail(KD_ERR_INVALID_ARG, "kd_op_ssm_conv: NULL attrs");
  LaunchCtx c;
  c.stream = (cudaStream_t)stream;
  return launch_ssm_conv(*a, zxbcdt, conv_w, conv_b, conv_state, xbc, c, nullptr);
}

kd_status kd_op_ssm_update(const kd_attr_ssm* a, const void* xbc, const void* zxbcdt, const float* dt_bias,
                           const float* A_log, const float* D, float* ssm_state, void* y, void* stream) {
  if (!a) return fail(KD_ERR_INVALID_ARG, "kd_op_ssm_update: NULL attrs");
  LaunchCtx c;
  c.stream = (cudaStream_t)stream;
  return launch_ssm_update(*a, xbc, zxbcdt, dt_bias, A_log, D, ssm_state, y, c, nullptr);
}

kd_status kd_op_gated_norm(const kd_attr_ssm* a, const void* y, const void* zxbcdt, const void* norm_w, void* yn,
                           void* stream) {
  if (!a) return fail(KD_ERR_INVALID_ARG, "kd_op_gated_norm: NULL attrs");
  LaunchCtx c;
  c.stream = (cudaStream_t)stream;
  return launch_gated_norm(*a, y, zxbcdt, norm_w, yn, c, nullptr);
}

}  // extern "C"
