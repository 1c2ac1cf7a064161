// elementwise.cu — the memory-role kernels other than attention:
//   a3  fused residual add + RMSNorm
//   a5  NeoX RoPE + paged KV append      (a5, C1.3-C1.4)
//   a8  SiLU·mul on 64-col gate/up blocks (a8, C1.9)
//   C1.11 final residual add
// plus the runtime's step-begin barrier and flag-wait kernels (a13/a15).
// All are HBM- or launch-bound: 16-byte vector loads, fp32 math, one pass.
#include <math.h>
#include <cmath>
#include <cstdlib>

#include "launch.hpp"

namespace kd {

static bool pdl_default() {
  const char* e = getenv("KD_PDL");
  return e ? atoi(e) != 0 : true;
}
bool g_pdl = pdl_default();

kd_status set_cuda_error(cudaError_t e, const char* where) {
  return fail(KD_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

// ------------------------------------------------------------------ a3
// one CTA per row; each thread keeps up to 4 chunks of 8 elements in registers
constexpr int kNormThreads = 256;
constexpr int kNormChunks = 4;  // H <= 8 * 256 * 4 = 8192

__global__ void __launch_bounds__(kNormThreads) add_rmsnorm_kernel(float* __restrict__ r, Deltas deltas,
                                                                  const __nv_bfloat16* __restrict__ gamma,
                                                                  __nv_bfloat16* __restrict__ h, int H, float eps,
                                                                  Epi epi, Acq acq) {
  pdl_launch_dependents();
  epi_started(epi);
  const int row = blockIdx.x, tid = threadIdx.x;
  const int nch = H / 8;
  // gamma is a weight (never written in a step): fetch it before the
  // dependency wait so it is in registers when the reduction finishes
  uint4 gm[kNormChunks];
#pragma unroll
  for (int c = 0; c < kNormChunks; ++c) {
    int ch = tid + c * kNormThreads;
    if (ch < nch) gm[c] = reinterpret_cast<const uint4*>(gamma)[ch];
  }
  pdl_wait();
  float v[kNormChunks][8];
  float ss = 0.f;
  float* rr = r + (size_t)row * H;
  uint32_t held[kMaxAcqIn] = {};  // chunks thread 0 acquired, per remote delta
#pragma unroll
  for (int c = 0; c < kNormChunks; ++c) {
    // remote deltas (a13 consumer side): column group c of every thread is the
    // byte range [16·256c, 16·256(c+1)) of the row; thread 0 acquires the
    // chunks it touches (ascending), the barrier orders the others behind it
    if (acq.n && c * kNormThreads < nch) {
      if (tid == 0)
        for (int i = 0; i < acq.n; ++i)
          acq_range(acq, i, 16u * (c * kNormThreads), 16u * min(nch, (c + 1) * kNormThreads), &held[i]);
      __syncthreads();
    }
    int ch = tid + c * kNormThreads;
    if (ch < nch) {
      float4 a = reinterpret_cast<const float4*>(rr)[2 * ch];
      float4 b = reinterpret_cast<const float4*>(rr)[2 * ch + 1];
      v[c][0] = a.x; v[c][1] = a.y; v[c][2] = a.z; v[c][3] = a.w;
      v[c][4] = b.x; v[c][5] = b.y; v[c][6] = b.z; v[c][7] = b.w;
      if (deltas.n) {
        uint4 dv[kMaxDeltas];
        for (int i = 0; i < deltas.n; ++i) dv[i] = reinterpret_cast<const uint4*>(deltas.p[i] + (size_t)row * H)[ch];
        for (int i = 0; i < deltas.n; ++i) {  // index order: bitwise reproducible
          const uint4 d = dv[i];
          v[c][0] += bf16lo(d.x); v[c][1] += bf16hi(d.x);
          v[c][2] += bf16lo(d.y); v[c][3] += bf16hi(d.y);
          v[c][4] += bf16lo(d.z); v[c][5] += bf16hi(d.z);
          v[c][6] += bf16lo(d.w); v[c][7] += bf16hi(d.w);
        }
        reinterpret_cast<float4*>(rr)[2 * ch] = make_float4(v[c][0], v[c][1], v[c][2], v[c][3]);
        reinterpret_cast<float4*>(rr)[2 * ch + 1] = make_float4(v[c][4], v[c][5], v[c][6], v[c][7]);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) ss += v[c][j] * v[c][j];
    }
  }
  __shared__ float red[kNormThreads / 32];
  ss = warp_sum(ss);
  if ((tid & 31) == 0) red[tid >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int w = 0; w < kNormThreads / 32; ++w) tot += red[w];  // fixed order: deterministic
  const float inv = rsqrtf(tot / (float)H + eps);
#pragma unroll
  for (int c = 0; c < kNormChunks; ++c) {
    int ch = tid + c * kNormThreads;
    if (ch < nch) {
      const uint4 g = gm[c];
      uint4 o;
      o.x = pack_bf16(v[c][0] * inv * bf16lo(g.x), v[c][1] * inv * bf16hi(g.x));
      o.y = pack_bf16(v[c][2] * inv * bf16lo(g.y), v[c][3] * inv * bf16hi(g.y));
      o.z = pack_bf16(v[c][4] * inv * bf16lo(g.z), v[c][5] * inv * bf16hi(g.z));
      o.w = pack_bf16(v[c][6] * inv * bf16lo(g.w), v[c][7] * inv * bf16hi(g.w));
      size_t e = (size_t)row * nch + ch;
      reinterpret_cast<uint4*>(h)[e] = o;
      for (int p = 0; p < epi.n; ++p) reinterpret_cast<uint4*>(epi.dst[p])[e] = o;
    }
  }
  epi_signal(epi, 0u, (uint32_t)H * 2u, (uint32_t)row, (uint32_t)row + 1u);  // COUNT: this CTA wrote the whole row
}

static DeltasF as_f32(const Deltas& d) {
  DeltasF f;
  f.n = d.n;
  for (int i = 0; i < d.n; ++i) f.p[i] = reinterpret_cast<const float*>(d.p[i]);
  return f;
}

kd_status launch_add_rmsnorm(const kd_attr_add_rmsnorm& a, float* r, const Deltas& d, const void* gamma, void* h,
                             const LaunchCtx& c, uint32_t* signals) {
  if (a.dtype != KD_BF16 && a.dtype != KD_F32) return fail(KD_ERR_UNSUPPORTED, "add_rmsnorm: dtype must be bf16 or fp32");
  if (a.n_delta > (uint32_t)kMaxDeltas || (int)a.n_delta != d.n)
    return fail(KD_ERR_INVALID_ARG, "add_rmsnorm: n_delta must match the deltas given (<= 8)");
  for (int i = 0; i < d.n; ++i)
    if (!d.p[i]) return fail(KD_ERR_INVALID_ARG, "add_rmsnorm: NULL delta");
  if (a.dtype == KD_F32) return launch_add_rmsnorm_f32(a, r, as_f32(d), (const float*)gamma, (float*)h, c, signals);
  if (a.rows == 0 || a.hidden == 0 || a.hidden % 8 || a.hidden > 8 * kNormThreads * kNormChunks)
    return fail(KD_ERR_UNSUPPORTED, "add_rmsnorm: hidden must be a multiple of 8 and <= 8192");
  if (!r || !gamma || !h) return fail(KD_ERR_INVALID_ARG, "add_rmsnorm: NULL pointer");
  KD_CUDA_CHECK(kd_launch(add_rmsnorm_kernel, dim3(a.rows), dim3(kNormThreads), 0, c.stream, r, d,
                          (const __nv_bfloat16*)gamma, (__nv_bfloat16*)h, (int)a.hidden, a.eps, c.epi, c.acq),
                "add_rmsnorm launch");
  if (signals) *signals = a.rows;
  return KD_OK;
}

// ------------------------------------------------------------------ C1.11
__global__ void residual_add_kernel(float* __restrict__ r, Deltas d, size_t n8, Epi epi, Acq acq) {
  pdl_launch_dependents();
  pdl_wait();
  if (acq.n) {  // remote deltas: thread 0 acquires every chunk of each (the final add is tiny)
    if (threadIdx.x == 0)
      for (int i = 0; i < acq.n; ++i) {
        uint32_t held = 0;
        acq_range(acq, i, 0u, acq.in[i].row_bytes, &held);
      }
    __syncthreads();
  }
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n8; i += (size_t)gridDim.x * blockDim.x) {
    float4 a = reinterpret_cast<float4*>(r)[2 * i];
    float4 b = reinterpret_cast<float4*>(r)[2 * i + 1];
    for (int k = 0; k < d.n; ++k) {  // index order
      const uint4 x = reinterpret_cast<const uint4*>(d.p[k])[i];
      a.x += bf16lo(x.x); a.y += bf16hi(x.x); a.z += bf16lo(x.y); a.w += bf16hi(x.y);
      b.x += bf16lo(x.z); b.y += bf16hi(x.z); b.z += bf16lo(x.w); b.w += bf16hi(x.w);
    }
    reinterpret_cast<float4*>(r)[2 * i] = a;
    reinterpret_cast<float4*>(r)[2 * i + 1] = b;
    for (int p = 0; p < epi.n; ++p) {
      reinterpret_cast<float4*>(epi.dst[p])[2 * i] = a;
      reinterpret_cast<float4*>(epi.dst[p])[2 * i + 1] = b;
    }
  }
  epi_signal(epi);  // CTA mode (the residual stream is never streamed in the decoder graphs)
}

static int residual_grid(const kd_attr_residual_add& a) {
  size_t n8 = (size_t)a.rows * a.hidden / 8;
  return (int)std::max<size_t>(1, std::min<size_t>((n8 + 255) / 256, 4 * kNumSMs));
}

kd_status launch_residual_add(const kd_attr_residual_add& a, float* r, const Deltas& d, const LaunchCtx& c,
                              uint32_t* signals) {
  size_t n = (size_t)a.rows * a.hidden;
  if (n == 0 || a.hidden % 8) return fail(KD_ERR_UNSUPPORTED, "residual_add: hidden must be a multiple of 8");
  if (a.n_delta == 0 || a.n_delta > (uint32_t)kMaxDeltas || (int)a.n_delta != d.n)
    return fail(KD_ERR_INVALID_ARG, "residual_add: need 1..8 deltas matching n_delta");
  for (int i = 0; i < d.n; ++i)
    if (!d.p[i]) return fail(KD_ERR_INVALID_ARG, "residual_add: NULL delta");
  if (!r) return fail(KD_ERR_INVALID_ARG, "residual_add: NULL pointer");
  if (a.dtype != KD_BF16 && a.dtype != KD_F32) return fail(KD_ERR_UNSUPPORTED, "residual_add: deltas bf16 or fp32");
  size_t n8 = n / 8;
  int grid = residual_grid(a);
  if (a.dtype == KD_F32) {
    kd_status st = launch_residual_add_f32(r, as_f32(d), n, grid, c);
    if (!st && signals) *signals = grid;
    return st;
  }
  KD_CUDA_CHECK(kd_launch(residual_add_kernel, dim3(grid), dim3(256), 0, c.stream, r, d, n8, c.epi, c.acq),
                "residual_add launch");
  if (signals) *signals = grid;
  return KD_OK;
}

// ------------------------------------------------------------------ a8
__global__ void silu_mul_kernel(const __nv_bfloat16* __restrict__ gu, __nv_bfloat16* __restrict__ out, int rows,
                                int F, Epi epi, Acq acq) {
  // one thread = 8 consecutive outputs; block j of 64 outputs reads gate
  // columns [128j, 128j+64) and up columns [128j+64, 128j+128). Work is
  // ordered block-major (t → block j, row, 8-column group), so the grid sweeps
  // the gu chunks in ascending order: a warp covers 4 rows of one block, and
  // its lane 0 acquires that block's chunk once (a13 consumer side).
  __shared__ unsigned s_cnt[kMaxChunks];
  pdl_launch_dependents();
  epi_started(epi);
  if (threadIdx.x < kMaxChunks) s_cnt[threadIdx.x] = 0u;
  if (epi.nch) __syncthreads();
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const size_t n = (size_t)rows * (F / 8);
  uint32_t held = 0;
  for (size_t t0 = blockIdx.x * (size_t)blockDim.x + (threadIdx.x & ~31u); t0 < n; t0 += (size_t)gridDim.x * blockDim.x) {
    const size_t t = t0 + lane;
    const int jw = (int)(t0 / ((size_t)rows * 8));  // the warp's first block (a warp spans ≤ 2 blocks when rows < 4)
    if (acq.n) {
      if (lane == 0) {
        const int jl = (int)(min(t0 + 31, n - 1) / ((size_t)rows * 8));
        acq_range(acq, 0, 256u * jw, 256u * (jl + 1), &held);
      }
      __syncwarp();
    }
    if (t < n) {
      const int j = (int)(t / ((size_t)rows * 8));
      const int rem = (int)(t - (size_t)j * rows * 8);
      const int row = rem >> 3, i = (rem & 7) * 8;
      const __nv_bfloat16* g = gu + (size_t)row * 2 * F + 128 * j + i;
      uint4 gv = *reinterpret_cast<const uint4*>(g);
      uint4 uv = *reinterpret_cast<const uint4*>(g + 64);
      const uint32_t* gp = &gv.x;
      const uint32_t* up = &uv.x;
      uint4 o;
      uint32_t* op = &o.x;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float g0 = bf16lo(gp[q]), g1 = bf16hi(gp[q]);
        float s0 = silu_fast(g0), s1 = silu_fast(g1);
        op[q] = pack_bf16(s0 * bf16lo(up[q]), s1 * bf16hi(up[q]));
      }
      const size_t e = ((size_t)row * F + 64 * j + i) / 8;
      reinterpret_cast<uint4*>(out)[e] = o;
      for (int p = 0; p < epi.n; ++p) reinterpret_cast<uint4*>(epi.dst[p])[e] = o;
      if (epi.nch) atomicAdd(&s_cnt[epi_chunk_of(epi, (uint32_t)(64 * j + i) * 2u)], 16u);
    }
  }
  epi_signal_counts(epi, s_cnt);
}

static int silu_grid(const kd_attr_silu_mul& a) {
  size_t n = (size_t)a.rows * a.ffn / 8;
  return (int)std::max<size_t>(1, std::min<size_t>((n + 255) / 256, 4 * kNumSMs));
}

kd_status launch_silu_mul(const kd_attr_silu_mul& a, const void* gu, void* out, const LaunchCtx& c,
                          uint32_t* signals) {
  if (a.dtype != KD_BF16 && a.dtype != KD_F32) return fail(KD_ERR_UNSUPPORTED, "silu_mul: dtype must be bf16 or fp32");
  if (a.rows == 0 || a.ffn == 0 || a.ffn % 64) return fail(KD_ERR_UNSUPPORTED, "silu_mul: ffn must be a multiple of 64");
  if (!gu || !out) return fail(KD_ERR_INVALID_ARG, "silu_mul: NULL pointer");
  int grid = silu_grid(a);
  if (a.dtype == KD_F32) {
    kd_status st = launch_silu_mul_f32(a, (const float*)gu, (float*)out, grid, c);
    if (!st && signals) *signals = grid;
    return st;
  }
  KD_CUDA_CHECK(kd_launch(silu_mul_kernel, dim3(grid), dim3(256), 0, c.stream, (const __nv_bfloat16*)gu,
                          (__nv_bfloat16*)out, (int)a.rows, (int)a.ffn, c.epi, c.acq),
                "silu_mul launch");
  if (signals) *signals = grid;
  return KD_OK;
}

// ------------------------------------------------------------------ a5
// grid (row, head group of 8): 16 threads per head. A rotated head (q or k)
// uses threads 0..D/16-1, each rotating 8 dims i..i+7 of the first half with
// their partners i+D/2.. (two 16-byte loads, two 16-byte stores); a v head is
// a 16-byte-vector copy into the cache slot. cos/sin of pos·θ^(−2i/D) are
// formed per thread in fp64 (R12), overlapping the loads.
constexpr int kRopeHeadsPerCta = 8;
struct RopeFreq {  // θ^(−2i/D), i < D/2, fp64, formed once per launch on the host
  double f[128];
};

__global__ void __launch_bounds__(kRopeHeadsPerCta * 16)
    rope_append_kernel(const __nv_bfloat16* __restrict__ qkv, const int32_t* __restrict__ bt,
                       const int32_t* __restrict__ sl, __nv_bfloat16* __restrict__ q_out,
                       __nv_bfloat16* __restrict__ kc, __nv_bfloat16* __restrict__ vc, int Hq, int Hkv, int D,
                       int page, int pps, int slot_offset, const __grid_constant__ RopeFreq fr, Epi epi, Acq acq) {
  __shared__ unsigned s_cnt[kMaxChunks];
  pdl_launch_dependents();
  epi_started(epi);
  const int b = blockIdx.x, half = D / 2, G = Hq / Hkv;
  const int hh = blockIdx.y * kRopeHeadsPerCta + (int)(threadIdx.x >> 4), t16 = threadIdx.x & 15;
  const int n_rot = Hq + Hkv;
  if (threadIdx.x < kMaxChunks) s_cnt[threadIdx.x] = 0u;
  pdl_wait();
  if (acq.n) {
    // remote qkv (a13 consumer side): thread 0 acquires the chunks holding the
    // source columns of this CTA's heads (kv-group chunks of the grouped layout)
    if (threadIdx.x == 0) {
      uint32_t held = 0;
      for (int x = 0; x < kRopeHeadsPerCta; ++x) {
        const int h2 = blockIdx.y * kRopeHeadsPerCta + x;
        int col;
        if (h2 < Hq) col = ((h2 / G) * (G + 2) + h2 % G) * D;
        else if (h2 < n_rot) col = ((h2 - Hq) * (G + 2) + G) * D;
        else if (h2 < n_rot + Hkv) col = ((h2 - n_rot) * (G + 2) + G + 1) * D;
        else break;
        acq_range(acq, 0, 2u * col, 2u * (col + D), &held);
      }
    }
    __syncthreads();
  } else if (epi.nch) {
    __syncthreads();  // s_cnt zeroed
  }
  if (hh < n_rot && t16 * 8 < half) {
    const int i0 = t16 * 8;
    const int pos = sl[b] - 1;
    const __nv_bfloat16* src = qkv + (size_t)b * (Hq + 2 * Hkv) * D;
    const __nv_bfloat16* x;
    __nv_bfloat16* dst;
    bool is_q = hh < Hq;
    size_t qoff = 0;
    if (is_q) {
      const int g = hh / G, j = hh % G;
      x = src + (size_t)g * (G + 2) * D + (size_t)j * D;
      qoff = (size_t)b * Hq * D + (size_t)hh * D;
      dst = q_out + qoff;
    } else {
      const int g = hh - Hq, slot = pos - slot_offset;  // this shard's slot of the absolute position
      const int32_t pg = bt[(size_t)b * pps + slot / page];
      x = src + (size_t)g * (G + 2) * D + (size_t)G * D;
      dst = kc + (((size_t)pg * Hkv + g) * page + slot % page) * D;
    }
    const uint4 xa = *reinterpret_cast<const uint4*>(x + i0);
    const uint4 xb = *reinterpret_cast<const uint4*>(x + half + i0);
    // angle = pos·θ^(−2i/D) in fp64, reduced to [−π, π] in fp64, then fp32
    // sincos of the small reduced angle (≈ the fp64 value rounded to fp32)
    float c[8], sn[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double ang = (double)pos * fr.f[i0 + k];
      const double kk = rint(ang * 0.15915494309189535);  // 1/(2π)
      const double red = fma(-kk, 6.283185307179586, fma(-kk, 2.4492935982947064e-16, ang));
      sincosf((float)red, &sn[k], &c[k]);
    }
    const uint32_t* pa = &xa.x;
    const uint32_t* pb = &xb.x;
    uint4 lo, hi;
    uint32_t* plo = &lo.x;
    uint32_t* phi = &hi.x;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float x0 = bf16lo(pa[q]), x1 = bf16hi(pa[q]), y0 = bf16lo(pb[q]), y1 = bf16hi(pb[q]);
      const float c0 = c[2 * q], c1 = c[2 * q + 1], s0 = sn[2 * q], s1 = sn[2 * q + 1];
      plo[q] = pack_bf16(x0 * c0 - y0 * s0, x1 * c1 - y1 * s1);
      phi[q] = pack_bf16(y0 * c0 + x0 * s0, y1 * c1 + x1 * s1);
    }
    *reinterpret_cast<uint4*>(dst + i0) = lo;
    *reinterpret_cast<uint4*>(dst + half + i0) = hi;
    if (!is_q)  // delta replication of the K cache: the same slot in every peer replica
      for (int p = 0; p < epi.n; ++p)
        if (epi.mir[p][0]) {
          __nv_bfloat16* pd = (__nv_bfloat16*)epi.mir[p][0] + (dst - kc);
          *reinterpret_cast<uint4*>(pd + i0) = lo;
          *reinterpret_cast<uint4*>(pd + half + i0) = hi;
        }
    if (is_q) {
      for (int p = 0; p < epi.n; ++p) {
        __nv_bfloat16* pd = (__nv_bfloat16*)epi.dst[p] + qoff;
        *reinterpret_cast<uint4*>(pd + i0) = lo;
        *reinterpret_cast<uint4*>(pd + half + i0) = hi;
      }
      if (epi.nch) {  // COUNT: 16 bytes at q columns hh·D + i0 and hh·D + half + i0
        atomicAdd(&s_cnt[epi_chunk_of(epi, (uint32_t)(hh * D + i0) * 2u)], 16u);
        atomicAdd(&s_cnt[epi_chunk_of(epi, (uint32_t)(hh * D + half + i0) * 2u)], 16u);
      }
    }
  } else if (hh >= n_rot && hh < n_rot + Hkv) {
    // v: plain copy into the cache slot, 16 threads × 8 dims per pass
    const int g = hh - n_rot;
    const int slot = sl[b] - 1 - slot_offset;
    const int32_t pg = bt[(size_t)b * pps + slot / page];
    const __nv_bfloat16* x = qkv + (size_t)b * (Hq + 2 * Hkv) * D + (size_t)g * (G + 2) * D + (size_t)(G + 1) * D;
    __nv_bfloat16* dst = vc + (((size_t)pg * Hkv + g) * page + slot % page) * D;
    for (int c8 = t16 * 8; c8 < D; c8 += 128) {
      const uint4 v = *reinterpret_cast<const uint4*>(x + c8);
      *reinterpret_cast<uint4*>(dst + c8) = v;
      for (int p = 0; p < epi.n; ++p)  // delta replication of the V cache
        if (epi.mir[p][1]) *reinterpret_cast<uint4*>((__nv_bfloat16*)epi.mir[p][1] + (dst - vc) + c8) = v;
    }
  }
  epi_signal_counts(epi, s_cnt);
}

static dim3 rope_grid(const kd_attr_rope_append& a) {
  const int heads = (int)(a.n_heads + 2 * a.n_kv_heads);
  return dim3(a.rows, (heads + kRopeHeadsPerCta - 1) / kRopeHeadsPerCta);
}

kd_status launch_rope_append(const kd_attr_rope_append& a, const void* qkv, const int32_t* bt, const int32_t* sl,
                             void* q_out, void* kc, void* vc, const LaunchCtx& c, uint32_t* signals) {
  if (a.dtype != KD_BF16 && a.dtype != KD_F32) return fail(KD_ERR_UNSUPPORTED, "rope_append: dtype must be bf16 or fp32");
  if (a.rows == 0 || a.n_kv_heads == 0 || a.n_heads % a.n_kv_heads || a.head_dim % 16 || a.head_dim < 16 ||
      a.head_dim > 256 || a.page == 0 || a.pages_per_seq == 0)
    return fail(KD_ERR_UNSUPPORTED, "rope_append: unsupported shape (head_dim a multiple of 16, <= 256)");
  if (!qkv || !bt || !sl || !q_out || !kc || !vc) return fail(KD_ERR_INVALID_ARG, "rope_append: NULL pointer");
  const dim3 grid = rope_grid(a);
  if (a.slot_offset % a.page) return fail(KD_ERR_INVALID_ARG, "rope_append: slot_offset must be a multiple of the page");
  if (a.dtype == KD_F32) {
    if (a.slot_offset) return fail(KD_ERR_UNSUPPORTED, "rope_append (fp32): sharded caches are bf16-path only");
    kd_status st = launch_rope_append_f32(a, (const float*)qkv, bt, sl, (float*)q_out, (float*)kc, (float*)vc, grid, c);
    if (!st && signals) *signals = grid.x * grid.y;
    return st;
  }
  RopeFreq fr;
  const double l2t = std::log2(a.theta);
  for (uint32_t i = 0; i < a.head_dim / 2; ++i) fr.f[i] = std::exp2(-2.0 * (double)i / (double)a.head_dim * l2t);
  KD_CUDA_CHECK(kd_launch(rope_append_kernel, grid, dim3(kRopeHeadsPerCta * 16), 0, c.stream, (const __nv_bfloat16*)qkv,
                          bt, sl, (__nv_bfloat16*)q_out, (__nv_bfloat16*)kc, (__nv_bfloat16*)vc, (int)a.n_heads,
                          (int)a.n_kv_heads, (int)a.head_dim, (int)a.page, (int)a.pages_per_seq, (int)a.slot_offset,
                          fr, c.epi, c.acq),
                "rope_append launch");
  if (signals) *signals = grid.x * grid.y;
  return KD_OK;
}

// ------------------------------------------------------------------ f2: KV-shard merge
// out = Σ_s 2^(lse_s − M)·out_s / Σ_s 2^(lse_s − M), M = max_s lse_s, shards in
// index order (deterministic); a shard with an empty context has lse = −inf
constexpr int kMaxParts = 8;
struct Parts {
  const uint8_t* p[kMaxParts];
};

__global__ void attn_merge_kernel(Parts ps, int n, __nv_bfloat16* __restrict__ out, int rows, int Hq, int D, Epi epi) {
  __shared__ unsigned s_cnt[kMaxChunks];
  pdl_launch_dependents();
  epi_started(epi);
  if (threadIdx.x < kMaxChunks) s_cnt[threadIdx.x] = 0u;
  if (epi.nch) __syncthreads();
  pdl_wait();
  const size_t lse_off = (size_t)rows * Hq * D * 2;
  const int d4n = D / 4;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < (size_t)rows * Hq * d4n;
       e += (size_t)gridDim.x * blockDim.x) {
    const size_t rh = e / d4n;
    const int d0 = (int)(e % d4n) * 4;
    float M = -INFINITY;
    for (int s = 0; s < n; ++s) M = fmaxf(M, reinterpret_cast<const float*>(ps.p[s] + lse_off)[rh]);
    float ax = 0.f, ay = 0.f, az = 0.f, aw = 0.f, wsum = 0.f;
    for (int s = 0; s < n; ++s) {
      const float l = reinterpret_cast<const float*>(ps.p[s] + lse_off)[rh];
      const float w = (M == -INFINITY || l == -INFINITY) ? 0.f : exp2f(l - M);
      const uint2 v = *reinterpret_cast<const uint2*>(ps.p[s] + (rh * D + d0) * 2);
      ax += w * bf16lo(v.x), ay += w * bf16hi(v.x), az += w * bf16lo(v.y), aw += w * bf16hi(v.y);
      wsum += w;
    }
    const float inv = wsum > 0.f ? 1.f / wsum : 0.f;
    uint2 o;
    o.x = pack_bf16(ax * inv, ay * inv);
    o.y = pack_bf16(az * inv, aw * inv);
    const size_t oi = rh * D + d0;
    *reinterpret_cast<uint2*>(out + oi) = o;
    for (int p = 0; p < epi.n; ++p) *reinterpret_cast<uint2*>((__nv_bfloat16*)epi.dst[p] + oi) = o;
    if (epi.nch) atomicAdd(&s_cnt[epi_chunk_of(epi, (uint32_t)(oi % ((size_t)Hq * D)) * 2u)], 8u);
  }
  epi_signal_counts(epi, s_cnt);
}

static int merge_grid(const kd_attr_attn_merge& a) {
  const size_t n = (size_t)a.rows * a.n_heads * (a.head_dim / 4);
  return (int)std::max<size_t>(1, std::min<size_t>((n + 255) / 256, 4 * kNumSMs));
}

kd_status launch_attn_merge(const kd_attr_attn_merge& a, const void* const* parts, void* out, const LaunchCtx& c,
                            uint32_t* signals) {
  if (a.n_parts == 0 || a.n_parts > (uint32_t)kMaxParts) return fail(KD_ERR_INVALID_ARG, "attn_merge: 1..8 parts");
  if (a.rows == 0 || a.n_heads == 0 || a.head_dim % 4) return fail(KD_ERR_UNSUPPORTED, "attn_merge: unsupported shape");
  if (!out) return fail(KD_ERR_INVALID_ARG, "attn_merge: NULL output");
  Parts ps{};
  for (uint32_t s = 0; s < a.n_parts; ++s) {
    if (!parts[s]) return fail(KD_ERR_INVALID_ARG, "attn_merge: NULL part");
    ps.p[s] = (const uint8_t*)parts[s];
  }
  const int grid = merge_grid(a);
  KD_CUDA_CHECK(kd_launch(attn_merge_kernel, dim3(grid), dim3(256), 0, c.stream, ps, (int)a.n_parts,
                          (__nv_bfloat16*)out, (int)a.rows, (int)a.n_heads, (int)a.head_dim, c.epi),
                "attn_merge launch");
  if (signals) *signals = grid;
  return KD_OK;
}

// ------------------------------------------------------------------ runtime support
struct PeerSlots {
  unsigned* slot[8];     // &peer.ctrl.barrier[me]
  unsigned* mine[8];     // &my.ctrl.barrier[peer]
};

__global__ void step_begin_kernel2(unsigned* epoch, PeerSlots ps, int n_peers) {
  if (threadIdx.x != 0) return;
  unsigned e = *epoch + 1;
  *epoch = e;
  if (n_peers == 0) return;
  fence_acq_rel_sys();
  for (int p = 0; p < n_peers; ++p) red_release_sys_add(ps.slot[p], 1u);
  for (int p = 0; p < n_peers; ++p) {
    long long spins = 0;
    while (ld_acquire_sys(ps.mine[p]) < e) {
      if (++spins > (1ll << 28)) {  // watchdog (~20 s): record (KD_ERR_TIMEOUT at kd_runtime_check) and give up
        atomicExch(epoch + 1, 3u);  // the error word follows the epoch word in the control block
        break;
      }
      __nanosleep(64);
    }
  }
}

kd_status launch_step_begin(unsigned* epoch, unsigned* const* mine, unsigned* const* peer_slots, int n_peers,
                            cudaStream_t s) {
  // mine[j] = my barrier word counting peer j's arrivals; peer_slots[j] = peer j's word for me
  if (n_peers > 8) return fail(KD_ERR_UNSUPPORTED, "step_begin: more than 8 peers");
  PeerSlots ps{};
  for (int j = 0; j < n_peers; ++j) {
    ps.slot[j] = peer_slots[j];
    ps.mine[j] = mine[j];
  }
  step_begin_kernel2<<<1, 32, 0, s>>>(epoch, ps, n_peers);
  KD_CUDA_CHECK(cudaGetLastError(), "step_begin launch");
  return KD_OK;
}

__global__ void wait_kernel(WaitList w, const unsigned* epoch, unsigned base, unsigned* err) {
  if ((int)threadIdx.x >= w.n) return;
  const unsigned e = *epoch;
  const unsigned long long target = (unsigned long long)(e - base) * w.mult[threadIdx.x];
  unsigned long long* log = w.log[threadIdx.x];
  const unsigned long long t0 = log ? gtimer_ns() : 0ull;
  long long spins = 0;
  while (ld_acquire_sys64(w.flag[threadIdx.x]) < target) {
    if (++spins > (1ll << 30)) {  // watchdog: record and give up (KD_ERR_TIMEOUT at kd_runtime_check)
      atomicExch(err, 1u);
      break;
    }
    __nanosleep(32);
  }
  if (log && atomicMax(log, (unsigned long long)e) < e) {  // first acquire of this chunk in this step
    log[1] = t0;
    log[2] = gtimer_ns();
  }
}

kd_status launch_wait(const WaitList& w, const unsigned* epoch, unsigned base, unsigned* err, cudaStream_t s) {
  if (w.n <= 0) return KD_OK;
  if (w.n > kMaxWait) return fail(KD_ERR_UNSUPPORTED, "wait: more than 32 flags");
  wait_kernel<<<1, 32, 0, s>>>(w, epoch, base, err);
  KD_CUDA_CHECK(cudaGetLastError(), "wait launch");
  return KD_OK;
}

kd_status ssm_init_attrs();  // ssm.cu

kd_status elementwise_init_attrs() {
  const void* fns[] = {(const void*)add_rmsnorm_kernel, (const void*)residual_add_kernel, (const void*)silu_mul_kernel,
                       (const void*)rope_append_kernel, (const void*)step_begin_kernel2, (const void*)wait_kernel};
  for (const void* f : fns)
    KD_CUDA_CHECK(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100), "carveout");
  return ssm_init_attrs();
}

template <typename T>
static kd_status attrs_of(const std::vector<uint8_t>& v, T* out) {
  if (v.size() != sizeof(T)) return fail(KD_ERR_INVALID_ARG, "op attrs have the wrong size for the op");
  std::memcpy(out, v.data(), sizeof(T));
  return KD_OK;
}

kd_status attention_signals(const kd_attr_attention& a, uint32_t* s);  // attention.cu

kd_status attention_grid(const kd_attr_attention& a, uint32_t* grid);  // attention.cu
kd_status gemm_grid(const GemmShape& sh, uint32_t* grid);              // gemm.cu

// CTAs one launch of a COUNT-release producer runs (the loopback residency
// gate waits for all of them to have started, runtime.cu)
kd_status op_grid(uint32_t op, const std::vector<uint8_t>& attrs, uint32_t* grid) {
  kd_status st = KD_OK;
  switch (op) {
    case KD_OP_ADD_RMSNORM: { kd_attr_add_rmsnorm a; if ((st = attrs_of(attrs, &a))) return st; *grid = a.rows; return KD_OK; }
    case KD_OP_SILU_MUL: { kd_attr_silu_mul a; if ((st = attrs_of(attrs, &a))) return st; *grid = silu_grid(a); return KD_OK; }
    case KD_OP_ROPE_APPEND: {
      kd_attr_rope_append a;
      if ((st = attrs_of(attrs, &a))) return st;
      const dim3 g = rope_grid(a);
      *grid = g.x * g.y;
      return KD_OK;
    }
    case KD_OP_ATTN_MERGE: { kd_attr_attn_merge a; if ((st = attrs_of(attrs, &a))) return st; *grid = merge_grid(a); return KD_OK; }
    case KD_OP_ATTENTION: { kd_attr_attention a; if ((st = attrs_of(attrs, &a))) return st; return attention_grid(a, grid); }
    case KD_OP_GEMM: { kd_attr_gemm a; if ((st = attrs_of(attrs, &a))) return st; return gemm_grid(gemm_shape(a), grid); }
    case KD_OP_GEMM_SILU: { kd_attr_gemm a; if ((st = attrs_of(attrs, &a))) return st; return gemm_grid(gemm_shape(a, true), grid); }
    case KD_OP_GEMM_RMSNORM: { kd_attr_gemm_rmsnorm a; if ((st = attrs_of(attrs, &a))) return st; return gemm_grid(gemm_shape(a), grid); }
  }
  return fail(KD_ERR_UNSUPPORTED, "op_grid: not a COUNT-release producer");
}

kd_status op_signals(uint32_t op, const std::vector<uint8_t>& attrs, uint32_t* signals) {
  kd_status st = KD_OK;
  switch (op) {
    case KD_OP_ADD_RMSNORM: { kd_attr_add_rmsnorm a; if ((st = attrs_of(attrs, &a))) return st; *signals = a.rows; return KD_OK; }
    case KD_OP_ATTN_MERGE: {
      kd_attr_attn_merge a;
      if ((st = attrs_of(attrs, &a))) return st;
      *signals = merge_grid(a);
      return KD_OK;
    }
    case KD_OP_ROPE_APPEND: {
      kd_attr_rope_append a;
      if ((st = attrs_of(attrs, &a))) return st;
      const dim3 g = rope_grid(a);
      *signals = g.x * g.y;
      return KD_OK;
    }
    case KD_OP_SILU_MUL: { kd_attr_silu_mul a; if ((st = attrs_of(attrs, &a))) return st; *signals = silu_grid(a); return KD_OK; }
    case KD_OP_RESIDUAL_ADD: { kd_attr_residual_add a; if ((st = attrs_of(attrs, &a))) return st; *signals = residual_grid(a); return KD_OK; }
    case KD_OP_ATTENTION: { kd_attr_attention a; if ((st = attrs_of(attrs, &a))) return st; return attention_signals(a, signals); }
    case KD_OP_GEMM: { kd_attr_gemm a; if ((st = attrs_of(attrs, &a))) return st; return gemm_signals(gemm_shape(a), signals); }
    case KD_OP_GEMM_SILU: { kd_attr_gemm a; if ((st = attrs_of(attrs, &a))) return st; return gemm_signals(gemm_shape(a, true), signals); }
    case KD_OP_QKV_ROPE: { kd_attr_qkv_rope a; if ((st = attrs_of(attrs, &a))) return st; return gemm_signals(gemm_shape(a), signals); }
    case KD_OP_GEMM_RMSNORM: { kd_attr_gemm_rmsnorm a; if ((st = attrs_of(attrs, &a))) return st; return gemm_signals(gemm_shape(a), signals); }
    case KD_OP_GROUPED_GEMM: { kd_attr_grouped_gemm a; if ((st = attrs_of(attrs, &a))) return st; return gemm_signals(gemm_shape(a), signals); }
    case KD_OP_MOE_ROUTE:
    case KD_OP_MOE_DISPATCH:
    case KD_OP_MOE_COMBINE: return moe_signals(op, attrs, signals);
    case KD_OP_SSM_CONV:
    case KD_OP_SSM_UPDATE:
    case KD_OP_GATED_NORM: return ssm_signals(op, attrs, signals);
    case KD_OP_ROPE_PREFILL: {
      kd_attr_rope_prefill a;
      if ((st = attrs_of(attrs, &a)) || (st = rope_prefill_validate(a))) return st;
      *signals = rope_prefill_signals(a);
      return KD_OK;
    }
    case KD_OP_PREFILL_ATTENTION: {
      kd_attr_prefill_attention a;
      if ((st = attrs_of(attrs, &a)) || (st = prefill_attention_validate(a))) return st;
      *signals = prefill_attention_signals(a);
      return KD_OK;
    }
  }
  *signals = 0;
  return KD_OK;
}

}  // namespace kd

extern "C" kd_status kd_set_pdl(int32_t enable) {
  kd::g_pdl = enable != 0;
  return KD_OK;
}
