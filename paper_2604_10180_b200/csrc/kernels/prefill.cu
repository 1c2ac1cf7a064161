// prefill.cu — f4: the prefill kernel graph's compute-bound kernels (SURVEY
// §8(f) f4; §2: prefill kernels span memory-bound GEMV and
// compute-bound FlashAttention). Prefill runs the same layer as decode over S
// prompt tokens per sequence (oracle/prefill.py): token row r = b·S + t.
//  * large-M GEMM (KD_OP_GEMM with M > 256 rows): Y[M,N] = X[M,K]·W[N,K]ᵀ is
//    tensor-bound (arithmetic intensity ~M), so tokens are the MMA rows:
//    persistent CTAs walk 128-token × 256-feature tiles; TMA (128-byte swizzle)
//    feeds a 4-stage ring of X (16 KB) + W (32 KB) k-blocks; one elected lane
//    issues tcgen05.mma.cta_group::1.kind::f16 M=128 N=256 into one of two
//    256-column TMEM accumulators, so the 4 epilogue warps (tcgen05.ld →
//    bf16 → global) drain tile i while tile i+1 accumulates.
//  * RoPE at every prompt position + paged KV fill (KD_OP_ROPE_PREFILL):
//    rope_append_kernel's per-element arithmetic with position t = r mod S,
//    the row's (cos, sin) pairs formed once per token in shared memory.
//  * causal GQA attention (KD_OP_PREFILL_ATTENTION): FlashAttention-2 style —
//    a CTA owns 64 query tokens of one head, 4 consumer warps × 16 tokens;
//    a producer warp streams 64-key blocks of the paged K/V cache (one TMA per
//    16-token page slab) through a 3-stage mbarrier ring; S = Q·Kᵀ and O += P·V
//    on mma.sync m16n8k16 (bf16 → fp32), online softmax in fp32 with exp2,
//    P reused from the S accumulators as the A fragments; blocks above the
//    diagonal are skipped, the diagonal block masked.
// All three store their primary output into every consumer device's landing
// slot too and release one flag increment per CTA (Epi CTA mode).
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "launch.hpp"
#include "mmasync.cuh"
#include "tcgen05.cuh"

namespace kd {
namespace pre {

using gemm::mbar_arrive;
using gemm::mbar_expect_tx;
using gemm::mbar_init;
using gemm::mbar_wait;
using gemm::mbar_wait_sleep;
using gemm::mma_bf16;
using gemm::mma_bf16_ws;
using gemm::mma_commit_ws;
using gemm::mma_commit;
using gemm::policy_evict_first;
using gemm::policy_evict_last;
using gemm::smem_u32;
using gemm::sw128_desc;
using gemm::tma_load_2d;
using gemm::tmem_ld16_nowait;
using gemm::tmem_ld_wait;
using mmas::ldsm_x4;
using mmas::ldsm_x4_t;
using mmas::mma16816;
using mmas::tile_off;
using mmas::tma_3d;

// ======================================================================= GEMM
constexpr int kTM = 128, kTN = 256, kTK = 64, kStages = 4;
constexpr int kGThreads = 192;  // w0 TMA, w1 MMA (+TMEM), w2..w5 epilogue
constexpr int kXBytes = kTM * kTK * 2, kWBytes = kTN * kTK * 2;
constexpr size_t kGemmSmem = 1024 + (size_t)kStages * (kXBytes + kWBytes) + 256;

struct GArgs {
  __nv_bfloat16* Y;
  int M, N, K, tiles_m, tiles, kblocks;
  Epi epi;
};

__global__ void __launch_bounds__(kGThreads, 1)
    gemm_prefill_kernel(const __grid_constant__ CUtensorMap tx, const __grid_constant__ CUtensorMap tw,
                        const __grid_constant__ GArgs A) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sx = smem;                                 // [S][128 × 64] X
  uint8_t* sw = smem + (size_t)kStages * kXBytes;      // [S][256 × 64] W
  uint64_t* full = (uint64_t*)(sw + (size_t)kStages * kWBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;  // [2]
  uint64_t* tempty = tfull + 2;       // [2]
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pdl_launch_dependents();
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1), mbar_init(&empty[s], 1);
    for (int i = 0; i < 2; ++i) mbar_init(&tfull[i], 1), mbar_init(&tempty[i], 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tx) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tw) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  const int KB = A.kblocks;

  if (warp == 0) {
    // ---------------------------------------------------- TMA producer
    if (lane == 0) {
      const uint64_t pw = policy_evict_last(), px = policy_evict_last();
      pdl_wait();  // X is the previous kernel's output
      int s = 0;
      unsigned ph = 0;
      for (int tile = blockIdx.x; tile < A.tiles; tile += gridDim.x) {
        const int mt = tile % A.tiles_m, nt = tile / A.tiles_m;  // consecutive CTAs share the W tile
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&empty[s], ph ^ 1u);
          mbar_expect_tx(&full[s], (unsigned)(kXBytes + kWBytes));
          tma_load_2d(sx + (size_t)s * kXBytes, &tx, kb * kTK, mt * kTM, &full[s], px);
          tma_load_2d(sw + (size_t)s * kWBytes, &tw, kb * kTK, nt * kTN, &full[s], pw);
          if (++s == kStages) s = 0, ph ^= 1u;
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------- MMA issuer
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kTN >> 3) << 17) |
                           ((uint32_t)(kTM >> 4) << 24);
    int s = 0;
    unsigned ph = 0, tc = 0;
    for (int tile = blockIdx.x; tile < A.tiles; tile += gridDim.x, ++tc) {
      const unsigned acc = tc & 1u;
      if (tc >= 2) mbar_wait(&tempty[acc], ((tc >> 1) - 1u) & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t td = tmem + acc * kTN;
      for (int kb = 0; kb < KB; ++kb) {
        mbar_wait(&full[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;");
        {  // warp-uniform issue (elect.sync inside the asm: uniform descriptors, no waterfall)
          const uint64_t ad = sw128_desc(smem_u32(sx + (size_t)s * kXBytes));
          const uint64_t bd = sw128_desc(smem_u32(sw + (size_t)s * kWBytes));
#pragma unroll
          for (int k = 0; k < kTK / 16; ++k) mma_bf16_ws(td, ad + 2 * k, bd + 2 * k, idesc, (kb > 0 || k > 0) ? 1u : 0u);
          mma_commit_ws(&empty[s]);
        }
        __syncwarp();
        if (++s == kStages) s = 0, ph ^= 1u;
      }
      if (lane == 0) mma_commit(&tfull[acc]);
      __syncwarp();
    }
  } else {
    // ---------------------------------------------------- epilogue (warps 2..5)
    const int q = warp & 3;             // TMEM lane quarter of this warp
    const int row = q * 32 + lane;      // token within the tile
    unsigned tc = 0;
    for (int tile = blockIdx.x; tile < A.tiles; tile += gridDim.x, ++tc) {
      const int mt = tile % A.tiles_m, nt = tile / A.tiles_m;
      const unsigned acc = tc & 1u;
      mbar_wait_sleep(&tfull[acc], (tc >> 1) & 1u, 64);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t ta = tmem + acc * kTN + ((uint32_t)(q * 32) << 16);
      const int m = mt * kTM + row;
      const int n0 = nt * kTN;
      __nv_bfloat16* yrow = A.Y + (size_t)m * A.N + n0;
#pragma unroll 1
      for (int c0 = 0; c0 < kTN; c0 += 32) {
        uint32_t v[2][16];
        tmem_ld16_nowait(ta + c0, v[0]);
        tmem_ld16_nowait(ta + c0 + 16, v[1]);
        tmem_ld_wait();
        if (m < A.M) {
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            const int n = n0 + c0 + 16 * b;
            if (n >= A.N) continue;  // (N is a multiple of 16)
            uint4 lo, hi;
            lo.x = pack_bf16(__uint_as_float(v[b][0]), __uint_as_float(v[b][1]));
            lo.y = pack_bf16(__uint_as_float(v[b][2]), __uint_as_float(v[b][3]));
            lo.z = pack_bf16(__uint_as_float(v[b][4]), __uint_as_float(v[b][5]));
            lo.w = pack_bf16(__uint_as_float(v[b][6]), __uint_as_float(v[b][7]));
            hi.x = pack_bf16(__uint_as_float(v[b][8]), __uint_as_float(v[b][9]));
            hi.y = pack_bf16(__uint_as_float(v[b][10]), __uint_as_float(v[b][11]));
            hi.z = pack_bf16(__uint_as_float(v[b][12]), __uint_as_float(v[b][13]));
            hi.w = pack_bf16(__uint_as_float(v[b][14]), __uint_as_float(v[b][15]));
            uint4* d = reinterpret_cast<uint4*>(yrow + c0 + 16 * b);
            d[0] = lo;
            d[1] = hi;
            for (int p = 0; p < A.epi.n; ++p)
              if (epi_row_in(A.epi, p, (uint32_t)m)) {
                uint4* dp = reinterpret_cast<uint4*>((__nv_bfloat16*)A.epi.dst[p] + (size_t)m * A.N + n0 + c0 + 16 * b);
                dp[0] = lo;
                dp[1] = hi;
              }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
  epi_signal(A.epi);  // CTA mode: one release per CTA after all its tiles
}

static int device_sms() {
  static int n = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : kNumSMs;
  }();
  return n;
}

// ======================================================================= RoPE + KV fill
constexpr int kRopeThreads = 256;
struct RopeFreq {
  double f[128];
};

// one CTA per token row: the row's D/2 (cos, sin) pairs are computed once
// (rope_append_kernel's arithmetic: fp64 angle reduced to [−π, π], fp32
// sincos of the reduced angle) into shared memory, then every (head, 8-dim
// group) of the row is rotated / copied with 16-byte loads and stores
__global__ void __launch_bounds__(kRopeThreads)
    rope_prefill_kernel(const __nv_bfloat16* __restrict__ qkv, const int32_t* __restrict__ bt,
                        __nv_bfloat16* __restrict__ q_out, __nv_bfloat16* __restrict__ kc,
                        __nv_bfloat16* __restrict__ vc, int S, int Hq, int Hkv, int D, int page, int pps,
                        const __grid_constant__ RopeFreq fr, Epi epi) {
  __shared__ float s_c[128], s_s[128];
  pdl_launch_dependents();
  const int r = blockIdx.x, half = D / 2, G = Hq / Hkv;
  const int b = r / S, pos = r - b * S;
  for (int i = threadIdx.x; i < half; i += kRopeThreads) {
    const double ang = (double)pos * fr.f[i];
    const double kk = rint(ang * 0.15915494309189535);
    const double red = fma(-kk, 6.283185307179586, fma(-kk, 2.4492935982947064e-16, ang));
    sincosf((float)red, &s_s[i], &s_c[i]);
  }
  __syncthreads();
  pdl_wait();
  const __nv_bfloat16* src = qkv + (size_t)r * (Hq + 2 * Hkv) * D;
  const int32_t pg = __ldg(bt + (size_t)b * pps + pos / page);
  const int gpr = half / 8;                      // 8-dim groups per rotated half-head
  const int n_rot = (Hq + Hkv) * gpr;            // rotation work items: q heads, then k heads
  const int n_v = Hkv * (D / 8);                 // v copy items
  for (int w = threadIdx.x; w < n_rot + n_v; w += kRopeThreads) {
    if (w < n_rot) {
      const int hh = w / gpr, i0 = (w - hh * gpr) * 8;
      const __nv_bfloat16* x;
      __nv_bfloat16* dst;
      size_t qoff = 0;
      const bool is_q = hh < Hq;
      if (is_q) {
        const int g = hh / G, j = hh % G;
        x = src + (size_t)g * (G + 2) * D + (size_t)j * D;
        qoff = (size_t)r * Hq * D + (size_t)hh * D;
        dst = q_out + qoff;
      } else {
        const int g = hh - Hq;
        x = src + (size_t)g * (G + 2) * D + (size_t)G * D;
        dst = kc + (((size_t)pg * Hkv + g) * page + pos % page) * D;
      }
      const uint4 xa = *reinterpret_cast<const uint4*>(x + i0);
      const uint4 xb = *reinterpret_cast<const uint4*>(x + half + i0);
      const uint32_t* pa = &xa.x;
      const uint32_t* pb = &xb.x;
      uint4 lo, hi;
      uint32_t* plo = &lo.x;
      uint32_t* phi = &hi.x;
#pragma unroll
      for (int qq = 0; qq < 4; ++qq) {
        const float x0 = bf16lo(pa[qq]), x1 = bf16hi(pa[qq]), y0 = bf16lo(pb[qq]), y1 = bf16hi(pb[qq]);
        const float c0 = s_c[i0 + 2 * qq], c1 = s_c[i0 + 2 * qq + 1], s0 = s_s[i0 + 2 * qq], s1 = s_s[i0 + 2 * qq + 1];
        plo[qq] = pack_bf16(x0 * c0 - y0 * s0, x1 * c1 - y1 * s1);
        phi[qq] = pack_bf16(y0 * c0 + x0 * s0, y1 * c1 + x1 * s1);
      }
      *reinterpret_cast<uint4*>(dst + i0) = lo;
      *reinterpret_cast<uint4*>(dst + half + i0) = hi;
      if (is_q)
        for (int p = 0; p < epi.n; ++p) {
          __nv_bfloat16* pd = (__nv_bfloat16*)epi.dst[p] + qoff;
          *reinterpret_cast<uint4*>(pd + i0) = lo;
          *reinterpret_cast<uint4*>(pd + half + i0) = hi;
        }
    } else {
      const int v = w - n_rot, g = v / (D / 8), c8 = (v - g * (D / 8)) * 8;
      const __nv_bfloat16* x = src + (size_t)g * (G + 2) * D + (size_t)(G + 1) * D;
      __nv_bfloat16* dst = vc + (((size_t)pg * Hkv + g) * page + pos % page) * D;
      *reinterpret_cast<uint4*>(dst + c8) = *reinterpret_cast<const uint4*>(x + c8);
    }
  }
  epi_signal(epi);
}

// ======================================================================= causal attention
#ifndef KD_PA_WARPS
#define KD_PA_WARPS 11
#endif
// Registers are allocated to a CTA in groups of 4 warps: the 1 producer + 4
// consumer warps of a 64-query CTA (174 registers/thread) paid for 8 warps, so
// only one such CTA fit per SM (ncu: 7 % achieved occupancy). 7 consumer warps
// + the producer use those same registers: 112 queries per CTA, 1.75× the
// consumer warps per SM.
constexpr int kAWarps = KD_PA_WARPS;  // consumers (16 query rows each); + 1 producer warp
constexpr int kAQ = 16 * kAWarps;     // query tokens per CTA
constexpr int kAK = 64;               // keys per block (4 pages of 16)
constexpr int kAStages = 3;
constexpr int kAThreads = (kAWarps + 1) * 32;

struct AArgs {
  const __nv_bfloat16* q;
  const int32_t* bt;
  __nv_bfloat16* out;
  int S, Hq, Hkv, pps, n_qt;
  float scale_log2;
  Epi epi;
};

template <int D>
__global__ void __launch_bounds__(kAThreads)
    prefill_attention_kernel(const __grid_constant__ CUtensorMap tk, const __grid_constant__ CUtensorMap tv,
                             const __grid_constant__ AArgs A) {
  constexpr int KS = D / 16;           // k-steps of S = Q·Kᵀ
  constexpr int SLAB_B = 16 * D * 2;   // one 16-token page slab
  constexpr int BLK_B = 4 * SLAB_B;    // 64 keys
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* ks = smem;                                   // [stage][4 slabs] K
  uint8_t* vs = ks + (size_t)kAStages * BLK_B;           // [stage][4 slabs] V
  uint64_t* full = (uint64_t*)(vs + (size_t)kAStages * BLK_B);
  uint64_t* empty = full + kAStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // heavy (late) query tiles first: blockIdx.x 0 is the last tile
  const int qt = A.n_qt - 1 - (int)blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int G = A.Hq / A.Hkv, g = h / G;
  const int t0 = qt * kAQ;
  const int nkb = min((A.S + kAK - 1) / kAK, (t0 + kAQ + kAK - 1) / kAK);  // causal: keys < t0 + 64
  pdl_launch_dependents();
  if (threadIdx.x == 0) {
    for (int s = 0; s < kAStages; ++s) mbar_init(&full[s], 1), mbar_init(&empty[s], kAWarps);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();  // q and the cache are the previous kernels' outputs

  if (warp == kAWarps) {
    // ---------------------------------------------------- producer: 64-key blocks, one TMA per page slab
    const uint64_t pol = policy_evict_last();  // (a kv head's blocks are re-read by G heads × later tiles)
    int s = 0;
    unsigned ph = 0;
    for (int kb = 0; kb < nkb; ++kb) {
      const int pid = lane < 4 && kb * 4 + lane < A.pps ? __ldg(A.bt + (size_t)b * A.pps + kb * 4 + lane) : 0;
      const int np = min(4, (A.S - kb * kAK + 15) / 16);
      if (lane == 0) mbar_wait(&empty[s], ph ^ 1u);
      __syncwarp();
      if (np < 4) {  // keys past the prompt are masked, but 0·(stale smem) must not be NaN: zero their V rows
        uint4* z = reinterpret_cast<uint4*>(vs + (size_t)s * BLK_B + np * SLAB_B);
        for (int e = lane; e < (4 - np) * SLAB_B / 16; e += 32) z[e] = make_uint4(0u, 0u, 0u, 0u);
        __syncwarp();
      }
      if (lane == 0) mbar_expect_tx(&full[s], (unsigned)(np * 2 * SLAB_B));  // (its arrive releases the zeros)
      for (int p = 0; p < np; ++p) {
        const int pg = __shfl_sync(0xffffffffu, pid, p);
        if (lane == 0) {
          const int row = (pg * A.Hkv + g) * 16;
          tma_3d(ks + (size_t)s * BLK_B + p * SLAB_B, &tk, 0, 0, row, &full[s], pol);
          tma_3d(vs + (size_t)s * BLK_B + p * SLAB_B, &tv, 0, 0, row, &full[s], pol);
        }
      }
      __syncwarp();
      if (++s == kAStages) s = 0, ph ^= 1u;
    }
    return;
  }

  // ---------------------------------------------------- consumers: 16 query tokens each
  const int gid = lane >> 2, c4 = lane & 3;
  const int qr0 = t0 + warp * 16 + gid, qr1 = qr0 + 8;  // this thread's two query rows (positions)
  // Q as the A operand: qa[ks] = {Q[r0][16ks+2c..], Q[r1][16ks+2c..], Q[r0][16ks+8+2c..], Q[r1][16ks+8+2c..]}
  uint32_t qa[KS][4];
  {
    const size_t base0 = ((size_t)b * A.S + qr0) * A.Hq * D + (size_t)h * D;
    const size_t base1 = ((size_t)b * A.S + qr1) * A.Hq * D + (size_t)h * D;
    const uint32_t* q0 = reinterpret_cast<const uint32_t*>(A.q + base0);
    const uint32_t* q1 = reinterpret_cast<const uint32_t*>(A.q + base1);
#pragma unroll
    for (int s = 0; s < KS; ++s) {
      qa[s][0] = qr0 < A.S ? q0[8 * s + c4] : 0u;
      qa[s][1] = qr1 < A.S ? q1[8 * s + c4] : 0u;
      qa[s][2] = qr0 < A.S ? q0[8 * s + 4 + c4] : 0u;
      qa[s][3] = qr1 < A.S ? q1[8 * s + 4 + c4] : 0u;
    }
  }
  float o[D / 8][4];
#pragma unroll
  for (int j = 0; j < D / 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};
  // ldmatrix lane roles
  const int lk_key = lane & 7, lk_chk = lane >> 3;                      // K (B of S): key, 16-B dim chunk offset
  const int lv_key = (lane & 7) + ((lane >> 3) & 1) * 8, lv_chk = lane >> 4;  // V (B of O, .trans)
  int s = 0;
  unsigned ph = 0;
  for (int kb = 0; kb < nkb; ++kb) {
    mbar_wait(&full[s], ph);
    const uint32_t kt = smem_u32(ks + (size_t)s * BLK_B), vt = smem_u32(vs + (size_t)s * BLK_B);
    // ---- S = Q·Kᵀ: 16 tokens × 64 keys (8 key blocks of 8)
    float sc[8][4];
#pragma unroll
    for (int nb = 0; nb < 8; ++nb) {
      sc[nb][0] = sc[nb][1] = sc[nb][2] = sc[nb][3] = 0.f;
      const int key = nb * 8 + lk_key;  // within the 64-key block
      const uint32_t slab = kt + (key >> 4) * SLAB_B;
#pragma unroll
      for (int k2 = 0; k2 < KS; k2 += 2) {
        // matrices: (k2: dims 0-7), (k2: dims 8-15), (k2+1: dims 0-7), (k2+1: dims 8-15) of key rows nb·8..+7
        const int chunk = 2 * k2 + lk_chk;  // 16-byte chunk index over D
        uint32_t b0, b1, b2, b3;
        ldsm_x4(slab + tile_off<D>(chunk >> 3, key & 15, chunk & 7), b0, b1, b2, b3);
        mma16816(sc[nb], qa[k2][0], qa[k2][1], qa[k2][2], qa[k2][3], b0, b1);
        mma16816(sc[nb], qa[k2 + 1][0], qa[k2 + 1][1], qa[k2 + 1][2], qa[k2 + 1][3], b2, b3);
      }
    }
    // ---- scale, causal mask, online softmax (rows qr0: sc[.][0..1], qr1: sc[.][2..3])
    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int nb = 0; nb < 8; ++nb) {
      const int key0 = kb * kAK + nb * 8 + 2 * c4;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int key = key0 + e;
        float v0 = sc[nb][e] * A.scale_log2, v1 = sc[nb][2 + e] * A.scale_log2;
        if (key > qr0 || key >= A.S) v0 = -INFINITY;
        if (key > qr1 || key >= A.S) v1 = -INFINITY;
        sc[nb][e] = v0;
        sc[nb][2 + e] = v1;
        mx0 = fmaxf(mx0, v0);
        mx1 = fmaxf(mx1, v1);
      }
    }
#pragma unroll
    for (int x = 1; x < 4; x <<= 1) {
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, x));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, x));
    }
    const float mn0 = fmaxf(m_run[0], mx0), mn1 = fmaxf(m_run[1], mx1);
    const float mu0 = mn0 == -INFINITY ? 0.f : mn0, mu1 = mn1 == -INFINITY ? 0.f : mn1;
    const float al0 = exp2f(m_run[0] - mu0), al1 = exp2f(m_run[1] - mu1);
    m_run[0] = mn0, m_run[1] = mn1;
    float ls0 = 0.f, ls1 = 0.f;
    uint32_t pa[4][4];  // P as the A operand of O += P·V: 4 key steps of 16
#pragma unroll
    for (int nb = 0; nb < 8; ++nb) {
      const float p00 = exp2f(sc[nb][0] - mu0), p01 = exp2f(sc[nb][1] - mu0);
      const float p10 = exp2f(sc[nb][2] - mu1), p11 = exp2f(sc[nb][3] - mu1);
      ls0 += p00 + p01;
      ls1 += p10 + p11;
      const int kk = nb >> 1, hi = nb & 1;
      pa[kk][hi ? 2 : 0] = pack_bf16(p00, p01);  // row r0, keys 16kk + 8hi + 2c..
      pa[kk][hi ? 3 : 1] = pack_bf16(p10, p11);  // row r1
    }
    l_run[0] = l_run[0] * al0 + ls0;
    l_run[1] = l_run[1] * al1 + ls1;
#pragma unroll
    for (int j = 0; j < D / 8; ++j) o[j][0] *= al0, o[j][1] *= al0, o[j][2] *= al1, o[j][3] *= al1;
    // ---- O += P·V: per 16-key step, per pair of 8-dim blocks
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const int key = kk * 16 + lv_key;
      const uint32_t slab = vt + (key >> 4) * SLAB_B;
#pragma unroll
      for (int nd = 0; nd < D / 8; nd += 2) {
        const int chunk = nd + lv_chk;
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(slab + tile_off<D>(chunk >> 3, key & 15, chunk & 7), b0, b1, b2, b3);
        mma16816(o[nd], pa[kk][0], pa[kk][1], pa[kk][2], pa[kk][3], b0, b1);
        mma16816(o[nd + 1], pa[kk][0], pa[kk][1], pa[kk][2], pa[kk][3], b2, b3);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == kAStages) s = 0, ph ^= 1u;
  }
  // ---- normalise and store: o[nd] = rows (r0: [0..1], r1: [2..3]) × dims 8nd + 2c, +1
#pragma unroll
  for (int x = 1; x < 4; x <<= 1) {
    l_run[0] += __shfl_xor_sync(0xffffffffu, l_run[0], x);
    l_run[1] += __shfl_xor_sync(0xffffffffu, l_run[1], x);
  }
  const float i0 = l_run[0] > 0.f ? 1.f / l_run[0] : 0.f, i1 = l_run[1] > 0.f ? 1.f / l_run[1] : 0.f;
  const size_t ob0 = ((size_t)b * A.S + qr0) * A.Hq * D + (size_t)h * D;
  const size_t ob1 = ((size_t)b * A.S + qr1) * A.Hq * D + (size_t)h * D;
#pragma unroll
  for (int nd = 0; nd < D / 8; ++nd) {
    const int d = nd * 8 + 2 * c4;
    const uint32_t w0 = pack_bf16(o[nd][0] * i0, o[nd][1] * i0), w1 = pack_bf16(o[nd][2] * i1, o[nd][3] * i1);
    if (qr0 < A.S) {
      *reinterpret_cast<uint32_t*>(A.out + ob0 + d) = w0;
      for (int p = 0; p < A.epi.n; ++p) *reinterpret_cast<uint32_t*>((__nv_bfloat16*)A.epi.dst[p] + ob0 + d) = w0;
    }
    if (qr1 < A.S) {
      *reinterpret_cast<uint32_t*>(A.out + ob1 + d) = w1;
      for (int p = 0; p < A.epi.n; ++p) *reinterpret_cast<uint32_t*>((__nv_bfloat16*)A.epi.dst[p] + ob1 + d) = w1;
    }
  }
  // (the producer warp has returned; the consumers publish)
  if (A.epi.n) {
    asm volatile("bar.sync 1, %0;" ::"r"(kAWarps * 32) : "memory");
    if (threadIdx.x == 0) {
      fence_acq_rel_sys();
      epi_release_cta(A.epi);
    }
  }
}

template <int D>
constexpr size_t attn_smem() {
  return 1024 + (size_t)2 * kAStages * 4 * 16 * D * 2 + 2 * kAStages * 8 + 64;
}

}  // namespace pre

// ======================================================================= host
bool gemm_is_prefill(const GemmShape& a) {
  return a.M > 256 && !a.groups && !a.silu && !a.rope && !a.norm && a.dtype == KD_BF16;
}

static uint32_t prefill_grid(const GemmShape& a) {
  const int tiles = (int)(((a.M + pre::kTM - 1) / pre::kTM) * ((a.N + pre::kTN - 1) / pre::kTN));
  return (uint32_t)std::max(1, std::min(tiles, pre::device_sms()));
}

kd_status gemm_prefill_prepare(const GemmShape& a, const void* X, const void* W, GemmPlan* gp) {
  if (a.N % 16 || a.K % 8) return fail(KD_ERR_UNSUPPORTED, "prefill gemm: need N % 16 == 0 and K % 8 == 0");
  if (!X || !W) return fail(KD_ERR_INVALID_ARG, "prefill gemm: NULL operand");
  if (((uintptr_t)X | (uintptr_t)W) & 15) return fail(KD_ERR_INVALID_ARG, "prefill gemm: operands must be 16-byte aligned");
  gp->sh = a;
  gp->prefill = true;
  gp->dense = false;
  kd_status s = encode_bf16_2d_sw128(&gp->tmap_x, X, a.K, a.M, pre::kTK, pre::kTM);
  if (s) return s;
  return encode_bf16_2d_sw128(&gp->tmap_w, W, a.K, a.N, pre::kTK, pre::kTN);
}

uint32_t gemm_prefill_signals(const GemmShape& a) { return prefill_grid(a); }

kd_status launch_gemm_prefill(const GemmPlan& gp, void* Y, const LaunchCtx& c, uint32_t* signals) {
  static bool init = false;
  if (!init) {
    KD_CUDA_CHECK(cudaFuncSetAttribute(pre::gemm_prefill_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)pre::kGemmSmem),
                  "prefill gemm smem attr");
    init = true;
  }
  pre::GArgs A;
  A.Y = (__nv_bfloat16*)Y;
  A.M = (int)gp.sh.M;
  A.N = (int)gp.sh.N;
  A.K = (int)gp.sh.K;
  A.tiles_m = (A.M + pre::kTM - 1) / pre::kTM;
  A.tiles = A.tiles_m * ((A.N + pre::kTN - 1) / pre::kTN);
  A.kblocks = (A.K + pre::kTK - 1) / pre::kTK;
  A.epi = c.epi;
  const uint32_t grid = prefill_grid(gp.sh);
  KD_CUDA_CHECK(kd_launch(pre::gemm_prefill_kernel, dim3(grid), dim3(pre::kGThreads), pre::kGemmSmem, c.stream,
                          gp.tmap_x, gp.tmap_w, A),
                "prefill gemm launch");
  if (signals) *signals = grid;
  return KD_OK;
}

static dim3 rope_prefill_grid(const kd_attr_rope_prefill& a) { return dim3(a.seqs * a.seq_len); }

kd_status rope_prefill_validate(const kd_attr_rope_prefill& a) {
  if (a.dtype != KD_BF16) return fail(KD_ERR_UNSUPPORTED, "rope_prefill: bf16 only");
  if (a.seqs == 0 || a.seq_len == 0 || a.n_kv_heads == 0 || a.n_heads % a.n_kv_heads || a.head_dim % 16 ||
      a.head_dim > 256 || a.page == 0 || (uint64_t)a.pages_per_seq * a.page < a.seq_len)  // (D/2 ≤ 128 table)
    return fail(KD_ERR_UNSUPPORTED, "rope_prefill: unsupported shape (head_dim % 16, pages cover the prompt)");
  return KD_OK;
}

kd_status launch_rope_prefill(const kd_attr_rope_prefill& a, const void* qkv, const int32_t* bt, void* q_out, void* kc,
                              void* vc, const LaunchCtx& c, uint32_t* signals) {
  kd_status s = rope_prefill_validate(a);
  if (s) return s;
  if (!qkv || !bt || !q_out || !kc || !vc) return fail(KD_ERR_INVALID_ARG, "rope_prefill: NULL pointer");
  pre::RopeFreq fr;
  const double l2t = std::log2(a.theta);
  for (uint32_t i = 0; i < a.head_dim / 2; ++i) fr.f[i] = std::exp2(-2.0 * (double)i / (double)a.head_dim * l2t);
  const dim3 grid = rope_prefill_grid(a);
  KD_CUDA_CHECK(kd_launch(pre::rope_prefill_kernel, grid, dim3(pre::kRopeThreads), 0, c.stream,
                          (const __nv_bfloat16*)qkv, bt, (__nv_bfloat16*)q_out, (__nv_bfloat16*)kc, (__nv_bfloat16*)vc,
                          (int)a.seq_len, (int)a.n_heads, (int)a.n_kv_heads, (int)a.head_dim, (int)a.page,
                          (int)a.pages_per_seq, fr, c.epi),
                "rope_prefill launch");
  if (signals) *signals = grid.x * grid.y;
  return KD_OK;
}

uint32_t rope_prefill_signals(const kd_attr_rope_prefill& a) {
  const dim3 g = rope_prefill_grid(a);
  return g.x * g.y;
}

kd_status prefill_attention_validate(const kd_attr_prefill_attention& a) {
  if (a.dtype != KD_BF16) return fail(KD_ERR_UNSUPPORTED, "prefill_attention: bf16 only");
  if (a.head_dim != 64 && a.head_dim != 128) return fail(KD_ERR_UNSUPPORTED, "prefill_attention: head_dim 64 or 128");
  if (a.page != 16) return fail(KD_ERR_UNSUPPORTED, "prefill_attention: page size must be 16");
  if (a.seqs == 0 || a.seq_len == 0 || a.seq_len % 16 || a.n_kv_heads == 0 || a.n_heads % a.n_kv_heads ||
      (uint64_t)a.pages_per_seq * 16 < a.seq_len)
    return fail(KD_ERR_UNSUPPORTED, "prefill_attention: need seq_len % 16 == 0 and pages covering it");
  return KD_OK;
}

uint32_t prefill_attention_signals(const kd_attr_prefill_attention& a) {
  return ((a.seq_len + pre::kAQ - 1) / pre::kAQ) * a.n_heads * a.seqs;
}

kd_status launch_prefill_attention(const kd_attr_prefill_attention& a, const void* q, const void* kc, const void* vc,
                                   const int32_t* bt, void* out, const LaunchCtx& c, uint32_t* signals) {
  kd_status s = prefill_attention_validate(a);
  if (s) return s;
  if (!q || !kc || !vc || !bt || !out) return fail(KD_ERR_INVALID_ARG, "prefill_attention: NULL pointer");
  static bool init = false;
  if (!init) {
    KD_CUDA_CHECK(cudaFuncSetAttribute(pre::prefill_attention_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)pre::attn_smem<128>()),
                  "prefill attention smem attr");
    KD_CUDA_CHECK(cudaFuncSetAttribute(pre::prefill_attention_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)pre::attn_smem<64>()),
                  "prefill attention smem attr");
    // the whole shared-memory carveout: left to the driver, the 99 KB CTA got a
    // 102 KB configuration, i.e. one CTA (5 warps) per SM (ncu: 7 % achieved
    // occupancy, 5.3 cycles between issues); two fit in the full 228 KB
    KD_CUDA_CHECK(cudaFuncSetAttribute(pre::prefill_attention_kernel<128>,
                                       cudaFuncAttributePreferredSharedMemoryCarveout, 100),
                  "prefill attention carveout");
    KD_CUDA_CHECK(cudaFuncSetAttribute(pre::prefill_attention_kernel<64>,
                                       cudaFuncAttributePreferredSharedMemoryCarveout, 100),
                  "prefill attention carveout");
    init = true;
  }
  CUtensorMap tk, tv;
  const uint64_t dims[3] = {64, a.head_dim / 64u, 1ull << 30};
  const uint64_t strides[2] = {128, a.head_dim * 2u};
  const uint32_t box[3] = {64, a.head_dim / 64u, 16};
  s = encode_bf16_sw128(&tk, kc, 3, dims, strides, box);
  if (s) return s;
  s = encode_bf16_sw128(&tv, vc, 3, dims, strides, box);
  if (s) return s;
  pre::AArgs A;
  A.q = (const __nv_bfloat16*)q;
  A.bt = bt;
  A.out = (__nv_bfloat16*)out;
  A.S = (int)a.seq_len;
  A.Hq = (int)a.n_heads;
  A.Hkv = (int)a.n_kv_heads;
  A.pps = (int)a.pages_per_seq;
  A.n_qt = (int)((a.seq_len + pre::kAQ - 1) / pre::kAQ);
  A.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)a.head_dim));
  A.epi = c.epi;
  const dim3 grid(A.n_qt, a.n_heads, a.seqs);
  if (getenv("KD_ATTN_DEBUG")) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pre::prefill_attention_kernel<128>, pre::kAThreads,
                                                  pre::attn_smem<128>());
    int occ0 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ0, pre::prefill_attention_kernel<128>, pre::kAThreads, 0);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, pre::prefill_attention_kernel<128>);
    fprintf(stderr, "prefill attention: %d CTAs/SM (smem %zu B, %d threads); %d without smem; regs %d, static smem %zu, max dyn %d, carveout %d\n",
            occ, pre::attn_smem<128>(), pre::kAThreads, occ0, fa.numRegs, fa.sharedSizeBytes,
            fa.maxDynamicSharedSizeBytes, fa.preferredShmemCarveout);
  }
  if (a.head_dim == 128)
    KD_CUDA_CHECK(kd_launch(pre::prefill_attention_kernel<128>, grid, dim3(pre::kAThreads), pre::attn_smem<128>(),
                            c.stream, tk, tv, A),
                  "prefill attention launch");
  else
    KD_CUDA_CHECK(kd_launch(pre::prefill_attention_kernel<64>, grid, dim3(pre::kAThreads), pre::attn_smem<64>(),
                            c.stream, tk, tv, A),
                  "prefill attention launch");
  if (signals) *signals = grid.x * grid.y * grid.z;
  return KD_OK;
}

}  // namespace kd
