// attention.cu — paged GQA decode attention (C1.5).
//
// For sequence b, kv head g and the G = Hq/Hkv query heads sharing it:
//   s_t = q_h·k_t/√D (t < seq_len[b]); p = softmax(s); out_h = Σ_t p_t v_t.
//
// B200 design (HBM-bound: 4 FLOP/B at G=4, 8 at G=8):
//  * grid = (split, kv head, sequence); each CTA streams the KV pages of its
//    split exactly once for all G heads (GQA reuse).
//  * HND cache [page][Hkv][16][D]: one page's K (or V) slab for one kv head is
//    16·D·2 contiguous bytes → one cp.async.bulk (TMA bulk copy) per slab into a
//    8-stage shared-memory ring guarded by mbarriers (stage s always feeds
//    warp s % 4); a single producer lane keeps up to 64 KB per CTA in flight.
//  * 4 consumer warps own alternate pages. Sᵀ = Q·Kᵀ and O += P·V use
//    mma.sync m16n8k16 (bf16 → fp32) with the G heads as MMA rows (padded
//    to 16): Q is a register-resident A operand, P stays in registers between
//    the two MMAs (C-fragment layout == A-fragment layout). The head-dim is
//    permuted consistently on q and K so each lane reads 16 contiguous bytes
//    per K row; the output dims are permuted so each lane owns 2·(D/8)
//    contiguous output dims.
//  * online softmax in fp32 with exp2; per-warp states merged in fixed warp
//    order; splits merged in fixed split order by whichever CTA of the
//    (b, g) unit arrives last (counter returns to 0) → bitwise deterministic.
#include <math.h>

#include "launch.hpp"

namespace kd {
namespace attn {

constexpr int kWarps = 4;           // consumer warps
constexpr int kThreads = (kWarps + 1) * 32;
constexpr int kStages = 8;
// Page j lives in stage j % kStages and is consumed by warp j % kWarps. With
// kStages % kWarps == 0 every stage is always consumed by the SAME warp, in
// round order, so no waiter can run two mbarrier phases ahead (parity waits
// alias after two phases).
static_assert(kStages % kWarps == 0, "each stage must belong to one consumer warp");
constexpr int kPage = 16;
constexpr int kMaxG = 8;
constexpr int kMaxPagesPerSplit = 512;

struct Params {
  const __nv_bfloat16* q;
  const __nv_bfloat16* kc;
  const __nv_bfloat16* vc;
  const int32_t* bt;
  const int32_t* sl;
  __nv_bfloat16* out;
  float* part_o;      // [rows][Hkv][splits][G][D]
  float* part_lse;    // [rows][Hkv][splits][G]
  unsigned* counter;  // [rows][Hkv]
  int Hq, Hkv, G, pps, splits, pages_per_split;
  float scale_log2;   // log2(e)/sqrt(D)
  Epi epi;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// D[16x8] += A[16x16] · B[16x8], bf16 inputs, fp32 accumulate.
// Rows 8..15 of A are zero padding (heads ≥ 8 never exist), so their
// accumulators (c2, c3) are bound to throw-away registers.
__device__ __forceinline__ void mma_rows8(float& c0, float& c1, float& z0, float& z1, uint32_t a0, uint32_t a2,
                                          uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c0), "+f"(c1), "+f"(z0), "+f"(z1)
      : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}

template <int D>
__global__ void __launch_bounds__(kThreads) decode_attention_kernel(Params P) {
  constexpr int NB = D / 8;        // PV n-blocks; each lane owns 2*NB output dims
  constexpr int KJ = D / 32;       // QK k-step pairs
  constexpr int SLAB = kPage * D;  // elements per page slab
  extern __shared__ __align__(128) uint8_t smem[];
  __nv_bfloat16* ks = reinterpret_cast<__nv_bfloat16*>(smem);
  __nv_bfloat16* vs = ks + kStages * SLAB;
  float* comb = reinterpret_cast<float*>(vs + kStages * SLAB);      // [kWarps][kMaxG][D]
  float* comb_ml = comb + kWarps * kMaxG * D;                        // [kWarps][kMaxG][2]
  int32_t* pages = reinterpret_cast<int32_t*>(comb_ml + kWarps * kMaxG * 2);
  uint64_t* full = reinterpret_cast<uint64_t*>(pages + kMaxPagesPerSplit);
  uint64_t* empty = full + kStages;
  __shared__ int s_last;

  pdl_launch_dependents();
  pdl_wait();
  const int split = blockIdx.x, g = blockIdx.y, b = blockIdx.z;
  const int G = P.G, Hkv = P.Hkv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int len = P.sl[b];
  const int n_pages_seq = (len + kPage - 1) / kPage;
  const int p0 = split * P.pages_per_split;
  const int p1 = min(n_pages_seq, p0 + P.pages_per_split);
  const int np = max(0, p1 - p0);

  for (int i = threadIdx.x; i < np; i += blockDim.x) pages[i] = P.bt[(size_t)b * P.pps + p0 + i];
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kWarps) {
    // ---------------- producer: one lane streams K/V page slabs
    if (lane == 0) {
      const size_t slab_stride = (size_t)Hkv * SLAB;
      for (int j = 0; j < np; ++j) {
        int st = j % kStages, round = j / kStages;
        if (round > 0) mbar_wait(&empty[st], (round - 1) & 1);
        size_t base = (size_t)pages[j] * slab_stride + (size_t)g * SLAB;
        mbar_expect_tx(&full[st], 2u * SLAB * 2u);
        bulk_g2s(ks + st * SLAB, P.kc + base, SLAB * 2u, &full[st]);
        bulk_g2s(vs + st * SLAB, P.vc + base, SLAB * 2u, &full[st]);
      }
    }
  } else {
    // ---------------- consumers
    const int gid = lane >> 2, c = lane & 3;
    // Q as the A operand: row gid = head g*G+gid; dims permuted (see header)
    uint32_t qa[2 * KJ][2];
    {
      const __nv_bfloat16* qh = P.q + (size_t)b * P.Hq * D + (size_t)(g * G + gid) * D;
#pragma unroll
      for (int J = 0; J < KJ; ++J) {
        uint4 v = make_uint4(0, 0, 0, 0);
        if (gid < G) v = *reinterpret_cast<const uint4*>(qh + 32 * J + 8 * c);
        qa[2 * J][0] = v.x;
        qa[2 * J][1] = v.y;
        qa[2 * J + 1][0] = v.z;
        qa[2 * J + 1][1] = v.w;
      }
    }
    float o[NB][2];
#pragma unroll
    for (int j = 0; j < NB; ++j) o[j][0] = o[j][1] = 0.f;
    float m_run = -INFINITY, l_run = 0.f;
    float z0 = 0.f, z1 = 0.f;  // throw-away accumulators of padding rows

    for (int j = warp; j < np; j += kWarps) {
      const int st = j % kStages;
      mbar_wait(&full[st], (j / kStages) & 1);
      const __nv_bfloat16* kp = ks + st * SLAB;
      __nv_bfloat16* vp = vs + st * SLAB;
      const int tok0 = (p0 + j) * kPage;
      const int valid = min(kPage, len - tok0);
      if (valid < kPage) {  // zero the V rows past the end (0·garbage must not be NaN)
        for (int e = lane; e < (kPage - valid) * D / 8; e += 32)
          reinterpret_cast<uint4*>(vp + valid * D)[e] = make_uint4(0, 0, 0, 0);
        __syncwarp();
      }
      // ---- S = Q Kᵀ : two n-blocks of 8 tokens
      float s0[2] = {0.f, 0.f}, s1[2] = {0.f, 0.f};
#pragma unroll
      for (int J = 0; J < KJ; ++J) {
        uint4 k0 = *reinterpret_cast<const uint4*>(kp + gid * D + 32 * J + 8 * c);
        uint4 k1 = *reinterpret_cast<const uint4*>(kp + (gid + 8) * D + 32 * J + 8 * c);
        mma_rows8(s0[0], s0[1], z0, z1, qa[2 * J][0], qa[2 * J][1], k0.x, k0.y);
        mma_rows8(s0[0], s0[1], z0, z1, qa[2 * J + 1][0], qa[2 * J + 1][1], k0.z, k0.w);
        mma_rows8(s1[0], s1[1], z0, z1, qa[2 * J][0], qa[2 * J][1], k1.x, k1.y);
        mma_rows8(s1[0], s1[1], z0, z1, qa[2 * J + 1][0], qa[2 * J + 1][1], k1.z, k1.w);
      }
      // tokens held by this lane: 2c, 2c+1 (block 0) and 8+2c, 9+2c (block 1)
      float sv[4] = {s0[0] * P.scale_log2, s0[1] * P.scale_log2, s1[0] * P.scale_log2, s1[1] * P.scale_log2};
      const int tl[4] = {2 * c, 2 * c + 1, 8 + 2 * c, 9 + 2 * c};
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (tl[i] >= valid) sv[i] = -INFINITY;
      float mx = fmaxf(fmaxf(sv[0], sv[1]), fmaxf(sv[2], sv[3]));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      const float m_new = fmaxf(m_run, mx);
      const float m_use = (m_new == -INFINITY) ? 0.f : m_new;
      const float alpha = exp2f(m_run - m_use);
      float p[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) p[i] = exp2f(sv[i] - m_use);
      l_run = l_run * alpha + (p[0] + p[1]) + (p[2] + p[3]);
      m_run = m_new;
#pragma unroll
      for (int jj = 0; jj < NB; ++jj) {
        o[jj][0] *= alpha;
        o[jj][1] *= alpha;
      }
      const uint32_t pa0 = pack_bf16(p[0], p[1]);  // A row gid, k = tokens 2c, 2c+1
      const uint32_t pa2 = pack_bf16(p[2], p[3]);  // A row gid, k = tokens 8+2c, 9+2c
      // ---- O += P V : lane supplies dims gid*NB + jj for tokens 2c,2c+1,2c+8,2c+9
      uint32_t vr[4][NB / 2];
      const int vt[4] = {2 * c, 2 * c + 1, 2 * c + 8, 2 * c + 9};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
#pragma unroll
        for (int q8 = 0; q8 < NB / 8; ++q8) {
          uint4 v = *reinterpret_cast<const uint4*>(vp + vt[i] * D + gid * NB + 8 * q8);
          vr[i][4 * q8 + 0] = v.x;
          vr[i][4 * q8 + 1] = v.y;
          vr[i][4 * q8 + 2] = v.z;
          vr[i][4 * q8 + 3] = v.w;
        }
      }
#pragma unroll
      for (int jj = 0; jj < NB; ++jj) {
        const uint32_t sel = (jj & 1) ? 0x7632u : 0x5410u;
        uint32_t b0 = __byte_perm(vr[0][jj >> 1], vr[1][jj >> 1], sel);
        uint32_t b1 = __byte_perm(vr[2][jj >> 1], vr[3][jj >> 1], sel);
        mma_rows8(o[jj][0], o[jj][1], z0, z1, pa0, pa2, b0, b1);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    // per-warp state → shared memory (unnormalised O, m, l)
    l_run += __shfl_xor_sync(0xffffffffu, l_run, 1);
    l_run += __shfl_xor_sync(0xffffffffu, l_run, 2);
    if (gid < G) {
      float* dst = comb + ((size_t)warp * kMaxG + gid) * D;
#pragma unroll
      for (int jj = 0; jj < NB; ++jj) {
        dst[(2 * c) * NB + jj] = o[jj][0];      // dim (2c)·NB + jj
        dst[(2 * c + 1) * NB + jj] = o[jj][1];  // dim (2c+1)·NB + jj
      }
      if (c == 0) {
        comb_ml[(warp * kMaxG + gid) * 2 + 0] = m_run;
        comb_ml[(warp * kMaxG + gid) * 2 + 1] = l_run;
      }
    }
  }
  __syncthreads();

  // ---------------- merge warps (fixed order), then splits (fixed order)
  const int nthr = kWarps * 32;
  const bool single = (P.splits == 1);
  const size_t unit = (size_t)b * Hkv + g;
  if (threadIdx.x < nthr) {
    for (int e = threadIdx.x; e < G * D; e += nthr) {
      const int h = e / D, d = e % D;
      float M = -INFINITY;
      for (int w = 0; w < kWarps; ++w) M = fmaxf(M, comb_ml[(w * kMaxG + h) * 2]);
      const float Mu = (M == -INFINITY) ? 0.f : M;
      float acc = 0.f, L = 0.f;
      for (int w = 0; w < kWarps; ++w) {
        const float sc = exp2f(comb_ml[(w * kMaxG + h) * 2] - Mu);
        acc += sc * comb[((size_t)w * kMaxG + h) * D + d];
        L += sc * comb_ml[(w * kMaxG + h) * 2 + 1];
      }
      if (single) {
        const float r = L > 0.f ? acc / L : 0.f;
        const size_t oi = (size_t)b * P.Hq * D + (size_t)(g * G + h) * D + d;
        __nv_bfloat16 ob = __float2bfloat16_rn(r);
        P.out[oi] = ob;
        for (int pp = 0; pp < P.epi.n; ++pp) ((__nv_bfloat16*)P.epi.dst[pp])[oi] = ob;
      } else {
        const size_t pi = ((unit * P.splits + split) * G + h);
        P.part_o[pi * D + d] = L > 0.f ? acc / L : 0.f;
        if (d == 0) P.part_lse[pi] = L > 0.f ? M + log2f(L) : -INFINITY;
      }
    }
  }
  if (single) {
    epi_signal(P.epi);
    return;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_acq_rel_gpu();
    unsigned prev = atom_add_acq_rel_gpu(&P.counter[unit], 1u);
    s_last = (prev == (unsigned)P.splits - 1);
  }
  __syncthreads();
  if (!s_last) return;
  fence_acq_rel_gpu();
  for (int e = threadIdx.x; e < G * D; e += blockDim.x) {
    const int h = e / D, d = e % D;
    float M = -INFINITY;
    for (int s = 0; s < P.splits; ++s) M = fmaxf(M, __ldcg(&P.part_lse[(unit * P.splits + s) * G + h]));
    const float Mu = (M == -INFINITY) ? 0.f : M;
    float acc = 0.f, L = 0.f;
    for (int s = 0; s < P.splits; ++s) {
      const size_t pi = (unit * P.splits + s) * G + h;
      const float sc = exp2f(__ldcg(&P.part_lse[pi]) - Mu);
      acc += sc * __ldcg(&P.part_o[pi * D + d]);
      L += sc;
    }
    const size_t oi = (size_t)b * P.Hq * D + (size_t)(g * G + h) * D + d;
    __nv_bfloat16 ob = __float2bfloat16_rn(L > 0.f ? acc / L : 0.f);
    P.out[oi] = ob;
    for (int pp = 0; pp < P.epi.n; ++pp) ((__nv_bfloat16*)P.epi.dst[pp])[oi] = ob;
  }
  if (threadIdx.x == 0) P.counter[unit] = 0u;  // ready for the next launch
  epi_signal(P.epi);
}

template <int D>
size_t smem_bytes() {
  return (size_t)2 * kStages * kPage * D * 2 + (size_t)kWarps * kMaxG * D * 4 + kWarps * kMaxG * 2 * 4 +
         kMaxPagesPerSplit * 4 + 2 * kStages * 8 + 64;
}

struct Shape {
  int splits, pages_per_split;
};

// Split count: enough CTAs for ~4 waves of 3 resident CTAs per SM, at least
// 16 pages per split, at most kMaxPagesPerSplit pages per split.
static Shape choose(const kd_attr_attention& a) {
  const int pages = (int)a.pages_per_seq;
  const long units = (long)a.rows * a.n_kv_heads;
  const long target = 4L * 3 * kNumSMs;
  int splits = (int)std::max<long>(1, (target + units - 1) / units);
  splits = std::min(splits, std::max(1, pages / 16));
  int pps = (pages + splits - 1) / splits;
  if (pps > kMaxPagesPerSplit) pps = kMaxPagesPerSplit;
  splits = (pages + pps - 1) / pps;
  return {splits, pps};
}

static kd_status validate(const kd_attr_attention& a) {
  if (a.dtype != KD_BF16) return fail(KD_ERR_UNSUPPORTED, "attention: only bf16 KV/activations");
  if (a.head_dim != 128 && a.head_dim != 64) return fail(KD_ERR_UNSUPPORTED, "attention: head_dim must be 64 or 128");
  if (a.page != kPage) return fail(KD_ERR_UNSUPPORTED, "attention: page size must be 16");
  if (a.n_kv_heads == 0 || a.n_heads % a.n_kv_heads || a.n_heads / a.n_kv_heads > kMaxG)
    return fail(KD_ERR_UNSUPPORTED, "attention: need Hq % Hkv == 0 and Hq/Hkv <= 8");
  if (a.rows == 0 || a.pages_per_seq == 0) return fail(KD_ERR_INVALID_ARG, "attention: empty shape");
  return KD_OK;
}

}  // namespace attn

kd_status attention_scratch_bytes(const kd_attr_attention& a, uint64_t* bytes) {
  kd_status s = attn::validate(a);
  if (s) return s;
  attn::Shape sh = attn::choose(a);
  const uint64_t units = (uint64_t)a.rows * a.n_kv_heads, G = a.n_heads / a.n_kv_heads;
  if (units > kMaxCounters) return fail(KD_ERR_UNSUPPORTED, "attention: too many (sequence, kv head) units");
  uint64_t n = 0;
  if (sh.splits > 1) n = kScratchCounterBytes + units * sh.splits * G * (a.head_dim + 1) * 4;
  *bytes = (n + 255) / 256 * 256;
  return KD_OK;
}

kd_status launch_attention(const kd_attr_attention& a, const void* q, const void* kc, const void* vc,
                           const int32_t* bt, const int32_t* sl, void* out, const LaunchCtx& c, uint32_t* signals) {
  kd_status s = attn::validate(a);
  if (s) return s;
  if (!q || !kc || !vc || !bt || !sl || !out) return fail(KD_ERR_INVALID_ARG, "attention: NULL pointer");
  attn::Shape sh = attn::choose(a);
  const int G = a.n_heads / a.n_kv_heads;
  if (sh.splits > 1 && !c.scratch) return fail(KD_ERR_INVALID_ARG, "attention: scratch required");
  attn::Params P;
  P.q = (const __nv_bfloat16*)q;
  P.kc = (const __nv_bfloat16*)kc;
  P.vc = (const __nv_bfloat16*)vc;
  P.bt = bt;
  P.sl = sl;
  P.out = (__nv_bfloat16*)out;
  const uint64_t units = (uint64_t)a.rows * a.n_kv_heads;
  if (units > kMaxCounters) return fail(KD_ERR_UNSUPPORTED, "attention: too many (sequence, kv head) units");
  P.counter = (unsigned*)c.scratch;
  P.part_o = (float*)((uint8_t*)c.scratch + kScratchCounterBytes);
  P.part_lse = P.part_o + units * sh.splits * G * a.head_dim;
  P.Hq = a.n_heads;
  P.Hkv = a.n_kv_heads;
  P.G = G;
  P.pps = a.pages_per_seq;
  P.splits = sh.splits;
  P.pages_per_split = sh.pages_per_split;
  P.scale_log2 = (float)(1.4426950408889634 / sqrt((double)a.head_dim));
  P.epi = c.epi;
  dim3 grid(sh.splits, a.n_kv_heads, a.rows);
  kd_status ks = kernels_init();
  if (ks) return ks;
  if (a.head_dim == 128)
    KD_CUDA_CHECK(kd_launch(attn::decode_attention_kernel<128>, grid, dim3(attn::kThreads), attn::smem_bytes<128>(),
                            c.stream, P),
                  "attention launch");
  else
    KD_CUDA_CHECK(kd_launch(attn::decode_attention_kernel<64>, grid, dim3(attn::kThreads), attn::smem_bytes<64>(),
                            c.stream, P),
                  "attention launch");
  if (signals) return attention_signals(a, signals);
  return KD_OK;
}

kd_status attention_signals(const kd_attr_attention& a, uint32_t* s) {
  kd_status st = attn::validate(a);
  if (st) return st;
  *s = (uint32_t)a.rows * a.n_kv_heads;  // one finishing CTA per (sequence, kv head)
  return KD_OK;
}

kd_status attention_init_attrs() {
  KD_CUDA_CHECK(cudaFuncSetAttribute(attn::decode_attention_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)attn::smem_bytes<128>()),
                "attention smem attr");
  KD_CUDA_CHECK(cudaFuncSetAttribute(attn::decode_attention_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)attn::smem_bytes<64>()),
                "attention smem attr");
  // one carveout (max shared memory) for every kernel of the step: the SM never
  // has to drain and re-split L1/shared memory between consecutive launches
  KD_CUDA_CHECK(cudaFuncSetAttribute(attn::decode_attention_kernel<128>, cudaFuncAttributePreferredSharedMemoryCarveout, 100),
                "attention carveout");
  KD_CUDA_CHECK(cudaFuncSetAttribute(attn::decode_attention_kernel<64>, cudaFuncAttributePreferredSharedMemoryCarveout, 100),
                "attention carveout");
  return KD_OK;
}

}  // namespace kd
