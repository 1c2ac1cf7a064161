// gemm.cu — decode GEMM Y[M,N] = X[M,K]·W[N,K]ᵀ on 5th-gen tensor cores
// (SURVEY §8(a) a4 QKV, a7 O, a9 gate_up, a10 down; C1.2).
//
// Decode GEMMs stream bf16 weights once with M (tokens) ≤ 256: arithmetic
// intensity ≈ M flop/B < the B200 ridge (≈255), so the bound is HBM. Design:
//  * swap-AB: the weight tile is the MMA A operand (M_mma = 128 output
//    features), the activations are the B operand (N_mma = M rounded up to
//    16); D lives in TMEM (fp32, 128 lanes × N_mma columns, double-buffered).
//  * TMA (cp.async.bulk.tensor, 128B swizzle, K-major) feeds a deep smem ring;
//    one elected lane issues tcgen05.mma.cta_group::1.kind::f16, tcgen05.commit
//    releases smem stages and hands accumulators to 4 epilogue warps
//    (tcgen05.ld 32x32b).
//  * stream-K: the (tile, k-block) units are split evenly over one persistent
//    CTA per SM, so every SM streams the same number of weight bytes whatever
//    N/128 is. A tile cut between CTAs is finished by the last contributor to
//    arrive, which sums all contributors' fp32 partials in contributor order
//    (bitwise deterministic; the tile counter returns to 0).
#include <dlfcn.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <map>
#include <mutex>
#include <vector>

#include "launch.hpp"
#include "tcgen05.cuh"

namespace kd {
namespace gemm {

constexpr int kThreads = 256;   // w0 TMA, w1 MMA + TMEM alloc, w4..w7 epilogue
constexpr int kBM = 128;        // weight rows per tile (MMA M)
constexpr int kBK = 64;         // K per stage (one 128-byte swizzle row of bf16)
constexpr int kStageA = kBM * kBK * 2;
constexpr int kSmemBudget = 200 * 1024;
constexpr int kMaxStages = 8;
constexpr int kChunk = 16;      // epilogue columns per tcgen05.ld (mma_n is a multiple of 16)

struct Args {
  __nv_bfloat16* Y;
  float* part;       // [tiles][max_contrib][M][128]
  unsigned* counter; // [tiles]
  int M, N, K, mma_n, stages, kblocks, tiles, max_contrib;
  int kbs;           // 64-column boxes per pipeline stage (k-block = 64·kbs columns)
  int silu;          // fused SiLU·mul epilogue: tile t = gate block t (rows 0-63) + up block t
                     // (rows 64-127) → a[j][64t + i] (row stride N/2), bits of a9 then a8
  int split_tiles;   // any tile cut between CTAs
  int fold_grid;     // split tiles folded after a grid barrier by all CTAs (many
                     // contributors per tile) instead of by their last arriver
  long long units;
  Epi epi;
  unsigned long long* trace;  // debug: 32 %globaltimer stamps per CTA (nullable)
  // grouped (MoE expert) mode: groups > 0; tile t → group t / tpg, n-tile t % tpg;
  // meta = int32 count[groups], offset[groups] (rows of X/Y), read on device
  int groups, tpg;
  const int* meta;            // counts of this GEMM's experts (already offset by expert0)
  int moff;                   // offsets are at meta + moff (= meta_experts)
  int dbg;                    // debug A/B knob (KD_GEMM_DBG): 1 skip owner Y stores, 2 skip owner fold
  unsigned* err;              // runtime error word (nullable): set to 2 when the fold barrier times out
  Acq acq;                    // chunk-aware consumer: X (slot 0) acquired per k-block by the TMA warp
  const float* dssq;          // deferred RMSNorm of X (nullable, silu only): gate/up sums × 1/rms(token)
};

#define KD_TRACE(slot) \
  do {                 \
    if (A.trace) A.trace[blockIdx.x * 32 + (slot)] = gtimer(); \
  } while (0)
// cycle-resolution stamps (clock64) into slots 16..31 (csk epilogue sub-phases)
#define KD_CTRACE(slot) \
  do {                 \
    if (A.trace) A.trace[blockIdx.x * 32 + (slot)] = (unsigned long long)clock64(); \
  } while (0)

// a13 consumer side in the TMA producer warp (lane 0): before the activation
// tile of k-block kb is loaded, acquire the chunks of the remote X that hold
// its columns [kb·64·kbs, (kb+1)·64·kbs) (ascending; `held` caches them); the
// proxy fence orders the acquired generic-proxy data before the TMA reads
__device__ __forceinline__ void acquire_x(const Acq& acq, int xi, int kb, int kbs, int K, uint32_t* held) {
  if (xi < 0) return;
  const uint32_t before = *held;
  const uint32_t lo = (uint32_t)kb * kbs * 64u * 2u, hi = (uint32_t)min(K, (kb + 1) * kbs * 64) * 2u;
  acq_range(acq, xi, lo, hi, held);
  if (*held != before) asm volatile("fence.proxy.async.global;" ::: "memory");
}

// unit range of CTA c: [c·U/G, (c+1)·U/G); owner of unit u: ⌈(u+1)·G/U⌉ − 1
__host__ __device__ __forceinline__ long long unit_begin(long long c, long long U, long long G) { return c * U / G; }
__host__ __device__ __forceinline__ long long unit_owner(long long u, long long U, long long G) {
  return ((u + 1) * G + U - 1) / U - 1;
}

// fused a8 on the GEMM output (KD_OP_GEMM_SILU): gate/up sums rounded to bf16
// (the plain GEMM's output) then exactly silu_mul_kernel's fp32 math
__device__ __forceinline__ float rbf(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }
__device__ __forceinline__ uint32_t silu2(float g0, float g1, float u0, float u1) {
  g0 = rbf(g0), g1 = rbf(g1), u0 = rbf(u0), u1 = rbf(u1);
  const float s0 = silu_fast(g0), s1 = silu_fast(g1);
  return pack_bf16(s0 * u0, s1 * u1);
}
// store 4 fused outputs a[row][col..col+3] (row stride ldy) to Y and every peer copy
__device__ __forceinline__ void store_silu4(const Args& A, size_t yo, const float4& g, const float4& u) {
  uint2 o;
  o.x = silu2(g.x, g.y, u.x, u.y);
  o.y = silu2(g.z, g.w, u.z, u.w);
  *reinterpret_cast<uint2*>(A.Y + yo) = o;
  for (int p = 0; p < A.epi.n; ++p) if (epi_row_in(A.epi, p, (uint32_t)(yo / (A.N / 2)))) *reinterpret_cast<uint2*>((__nv_bfloat16*)A.epi.dst[p] + yo) = o;
}

// deferred RMSNorm (KD_NORM_DEFER): 1/rms of token j from the producer's
// per-CTA partial sums of r'² (layout KD_DNORM_*: eps, N, then KD_DNORM_PARTS
// partials per token, unused ones zero), summed in index order
__device__ __forceinline__ float dnorm_inv(const float* d, int j) {
  const float4* p = reinterpret_cast<const float4*>(d + KD_DNORM_HDR + (size_t)j * KD_DNORM_PARTS);
  float4 v[KD_DNORM_PARTS / 4];
#pragma unroll
  for (int c = 0; c < KD_DNORM_PARTS / 4; ++c) v[c] = __ldcg(p + c);  // all in flight
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < KD_DNORM_PARTS / 4; ++c) {
    s += v[c].x;
    s += v[c].y;
    s += v[c].z;
    s += v[c].w;
  }
  return rsqrtf(s / __ldcg(d + 1) + __ldcg(d));
}

// kX: the round-2 handoff protocol (chunk byte counts, in-kernel acquires,
// residency / log words) is compiled in; launches without chunked transfers
// use the kX = false instance, whose code is the plain GEMM + CTA-mode peer
// stores (measured: the extra code cost 0.7-1.5 µs per launch otherwise)
template <bool kX>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmap_w, const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ Args A) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // align by offsetting the __shared__ array itself (a uintptr_t round trip
  // loses the address space: the epilogue's staging stores compiled to
  // generic ST.E with 64-bit address math, measured ≈35 cycles each)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int S = A.stages, kbs = A.kbs;
  const int xbox = A.mma_n * kBK * 2;          // one 64-column X box
  const int wst = kbs * kStageA, xst = kbs * xbox;
  uint8_t* sa = smem;                          // S × kbs × 16 KB (W)
  uint8_t* sb = smem + (size_t)S * wst;        // S × kbs × mma_n·128 B (X)
  uint64_t* full = (uint64_t*)(sb + (size_t)S * xst);
  uint64_t* empty = full + kMaxStages;
  uint64_t* tfull = empty + kMaxStages;        // [2]
  uint64_t* tempty = tfull + 2;                // [2]
  uint64_t* fixbar = tempty + 2;               // last arriver's bulk loads of the partials
  uint32_t* tmem_slot = (uint32_t*)(fixbar + 1);
  volatile unsigned* s_flag = (volatile unsigned*)(tmem_slot + 1);
  __nv_bfloat16* ystage = (__nv_bfloat16*)(fixbar + 2);  // 2 x [16][128] bf16 epilogue transpose
  unsigned* s_cnt = (unsigned*)(ystage + 2 * kChunk * kBM);  // COUNT-mode bytes per (peer, chunk) (this CTA)
  float* s_inv = (float*)(s_cnt + kMaxPeers * kMaxChunks);    // [M] deferred-norm 1/rms per token (dssq)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) KD_TRACE(0);
  pdl_launch_dependents();
  if constexpr (kX) {
    epi_started(A.epi);
    if (threadIdx.x < kMaxPeers * kMaxChunks) s_cnt[threadIdx.x] = 0u;  // (ordered by the __syncthreads below)
  }
  // COUNT mode: tally the bytes this CTA streams into each chunk of the output row
  const int row_elems = A.silu ? A.N / 2 : A.N;
  auto count = [&](size_t yo, unsigned bytes) {  // per peer: only the rows it receives
    if constexpr (kX) {
      if (A.epi.nch) {
        const int c = epi_chunk_of(A.epi, (uint32_t)(yo % (size_t)row_elems) * 2u);
        const uint32_t row = (uint32_t)(yo / (size_t)row_elems);
        for (int p = 0; p < A.epi.n; ++p)
          if (epi_row_in(A.epi, p, row)) atomicAdd(&s_cnt[p * kMaxChunks + c], bytes);
      }
    }
  };
  const long long U = A.units, G = gridDim.x, c = blockIdx.x;
  const long long u0 = unit_begin(c, U, G), u1 = unit_begin(c + 1, U, G);
  const int KB = A.kblocks;
  const uint32_t ncols = (2 * A.mma_n <= 32) ? 32 : (2 * A.mma_n <= 64 ? 64 : (2 * A.mma_n <= 128 ? 128 : (2 * A.mma_n <= 256 ? 256 : 512)));

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    mbar_init(fixbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmap_w) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmap_x) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) KD_TRACE(1);

  auto w_row = [&](int t) { return A.groups ? (t / A.tpg) * A.N + (t % A.tpg) * kBM : t * kBM; };
  if (warp == 0) {
    // ------------------------------------------------ TMA producer (warp-uniform loop, lane 0 issues)
    const uint64_t pw = policy_evict_first(), px = policy_evict_last();
    const unsigned tx = (unsigned)(wst + xst);
    const long long n_pre = std::min<long long>(S, u1 - u0);
    // (tile, k-block) of a unit, advanced incrementally: a 64-bit division per
    // stage (a ~300-cycle subroutine) was measured at ≈600 cycles of issue
    // cost per stage in this warp
    const int t_first = (int)(u0 / KB), kb_first = (int)(u0 - (long long)t_first * KB);
    auto load_w = [&](int t, int kb, int s) {
      for (int b = 0; b < kbs; ++b)
        tma_load_2d(sa + (size_t)s * wst + b * kStageA, &tmap_w, (kb * kbs + b) * kBK, w_row(t), &full[s], pw);
    };
    const int xi = kX ? acq_find(A.acq, 0) : -1;
    uint32_t held = 0;
    auto load_x = [&](int t, int kb, int s) {
      const int xr = A.groups ? __ldg(A.meta + A.moff + t / A.tpg) : 0;
      if constexpr (kX) acquire_x(A.acq, xi, kb, kbs, A.K, &held);
      for (int b = 0; b < kbs; ++b)
        tma_load_2d(sb + (size_t)s * xst + b * xbox, &tmap_x, (kb * kbs + b) * kBK, xr, &full[s], px);
    };
    if (lane == 0) KD_CTRACE(24);
    int t = t_first, kb = kb_first;
    if (lane == 0) {
      // weights never depend on the previous kernel: fill the first ring of W
      // tiles before the grid-dependency wait (overlaps the previous kernel's
      // tail), then the activations of those stages, then steady state
      for (long long i = 0; i < n_pre; ++i) {
        mbar_expect_tx(&full[i], tx);
        load_w(t, kb, (int)i);
        if (i == 0) KD_CTRACE(25);
        if (++kb == KB) kb = 0, ++t;
      }
      KD_CTRACE(26);
      KD_TRACE(2);
      pdl_wait();
      t = t_first, kb = kb_first;
      for (long long i = 0; i < n_pre; ++i) {
        load_x(t, kb, (int)i);
        if (++kb == KB) kb = 0, ++t;
      }
    }
    __syncwarp();
    t = __shfl_sync(0xffffffffu, t, 0);
    kb = __shfl_sync(0xffffffffu, kb, 0);
    long long i = n_pre;
    int s = (int)(n_pre % S), ph = (int)(n_pre / S);
    for (long long u = u0 + n_pre; u < u1; ++u, ++i) {
      mbar_wait(&empty[s], (unsigned)((ph - 1) & 1));
      if (lane == 0) {
        mbar_expect_tx(&full[s], tx);
        load_w(t, kb, s);
        load_x(t, kb, s);
      }
      __syncwarp();
      if (++kb == KB) kb = 0, ++t;
      if (++s == S) s = 0, ++ph;
    }
    if (lane == 0) KD_TRACE(3);
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer (warp-uniform loop, lane 0 issues)
    if (lane == 0) pdl_wait();
    __syncwarp();
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(A.mma_n >> 3) << 17) |
                           ((uint32_t)(kBM >> 4) << 24);
    long long i = 0;
    int seg = 0, st = 0, ph = 0;  // ring slot / phase of unit i, advanced incrementally (no 64-bit division per stage)
    long long u = u0;
    int t = (int)(u0 / KB);
    while (u < u1) {
      const long long seg_end = std::min<long long>(u1, (long long)(t + 1) * KB);
      const int a = seg & 1, use = seg >> 1;
      if (use > 0) mbar_wait(&tempty[a], (unsigned)((use - 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t tmem_d = tmem_base + (uint32_t)(a * A.mma_n);
      bool first = true;
      for (; u < seg_end; ++u, ++i) {
        const int s = st;
        mbar_wait(&full[s], (unsigned)(ph & 1));
        if (++st == S) st = 0, ++ph;
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (KD_MMA_WS) {  // every lane, elect.sync issues (uniform operands)
          if (lane == 0 && i == 0) KD_TRACE(4);
          const uint32_t a_addr = smem_u32(sa + (size_t)s * wst);
          const uint32_t b_addr = smem_u32(sb + (size_t)s * xst);
          for (int b = 0; b < kbs; ++b)
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k)
              mma_bf16_ws(tmem_d, sw128_desc(a_addr + b * kStageA + 32 * k), sw128_desc(b_addr + b * xbox + 32 * k),
                          idesc, (first && b == 0 && k == 0) ? 0u : 1u);
          mma_commit_ws(&empty[s]);
        } else if (lane == 0) {
          if (i == 0) KD_TRACE(4);
          const uint32_t a_addr = smem_u32(sa + (size_t)s * wst);
          const uint32_t b_addr = smem_u32(sb + (size_t)s * xst);
          for (int b = 0; b < kbs; ++b)
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k)
              // advance 16 bf16 = 32 B inside the 128 B swizzle row
              mma_bf16(tmem_d, sw128_desc(a_addr + b * kStageA + 32 * k), sw128_desc(b_addr + b * xbox + 32 * k), idesc,
                       (first && b == 0 && k == 0) ? 0u : 1u);
          mma_commit(&empty[s]);  // smem stage free once these MMAs retire
        }
        __syncwarp();
        first = false;
      }
      if (lane == 0) mma_commit(&tfull[a]);  // accumulator ready for the epilogue
      __syncwarp();
      ++seg;
      ++t;
    }
    if (lane == 0) KD_TRACE(5);
  } else if (warp >= 4) {
    // ------------------------------------------------ epilogue (TMEM → HBM / peers)
    // Whole tiles are stored straight from TMEM. A split tile's contributors
    // each publish their fp32 partial [M][128] (slot = contributor − first
    // contributor); after a grid-wide barrier every CTA folds an equal slice
    // of all split tiles, summing the partials in contributor order (bitwise
    // deterministic). A single CTA folding a whole tile was measured at
    // ≈5 µs (one SM reads ≈40-60 GB/s); spread over the grid the fold is
    // ≈32 KB per CTA. Every CTA releases the consumer flags once, at the end.
    const int q = warp - 4;                 // TMEM lane quarter
    const int row_in_tile = q * 32 + lane;  // output feature within the tile
    const int ep_tid = threadIdx.x - 128;
    const size_t part_elems = (size_t)A.M * kBM;
    pdl_wait();  // scratch and Y may still be in use by the previous kernel
    if (A.dssq) {  // deferred RMSNorm of X: per-token 1/rms while the first tile still streams
      for (int j = ep_tid; j < A.M; j += 128) s_inv[j] = dnorm_inv(A.dssq, j);
      named_bar(1, 128);
    }
    int seg = 0;
    long long u = u0;
    auto out_coords = [&](int t, int* nb0, int* y0, int* mv) {
      const int grp = A.groups ? t / A.tpg : 0;
      *nb0 = (A.groups ? t % A.tpg : t) * kBM;
      *y0 = A.groups ? __ldg(A.meta + A.moff + grp) : 0;
      *mv = A.groups ? min(__ldg(A.meta + grp), A.M) : A.M;
    };
    while (u < u1) {
      const int t = (int)(u / KB);
      const long long t_begin = (long long)t * KB, t_end = t_begin + KB;
      const long long seg_end = std::min<long long>(u1, t_end);
      const bool whole = (u == t_begin && seg_end == t_end);
      const int a = seg & 1;
      mbar_wait_sleep(&tfull[a], (unsigned)((seg >> 1) & 1), 128);
      if (ep_tid == 0 && seg < 3) KD_TRACE(6 + 2 * seg);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(a * A.mma_n);
      int nb0, y0, mv;
      out_coords(t, &nb0, &y0, &mv);
      if (!whole) {
        const long long first = unit_owner(t_begin, U, G);
        float* my_part = A.part + ((size_t)t * A.max_contrib + (c - first)) * part_elems;
        for (int j0 = 0; j0 < A.M; j0 += kChunk) {
          float v[kChunk];
          tmem_ld16(tbase + j0, v);
#pragma unroll
          for (int j = 0; j < kChunk; ++j)
            if (j0 + j < A.M) __stcg(my_part + (size_t)(j0 + j) * kBM + row_in_tile, v[j]);
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[a]);
        if (!A.fold_grid) {
          // few contributors per tile: the LAST to arrive folds the tile alone
          // (contributor order → deterministic) and resets the counter
          const long long lastc = unit_owner(t_end - 1, U, G);
          const int n_contrib = (int)(lastc - first + 1);
          unsigned* arrive = A.counter + 2 + t;
          named_bar(1, 128);
          // the acq_rel add releases the partial (the 128 threads' stores are
          // ordered before it by the named barrier: release is cumulative) and
          // acquires the other contributors' for the last arriver
          if (ep_tid == 0) s_flag[0] = atom_add_acq_rel_gpu(arrive, 1u);
          named_bar(1, 128);
          if (s_flag[0] == (unsigned)(n_contrib - 1)) {
            if (ep_tid == 0) *arrive = 0u;
            const float4* parts = reinterpret_cast<const float4*>(A.part + (size_t)t * A.max_contrib * part_elems);
            const int per = (int)(part_elems / 4);
            if (A.silu) {  // gate float4 (rows r..r+3 < 64) with its up partner 16 float4s on
              // 4 items per round with every (item, contributor) load in flight
              // together: the fold is L2-latency-bound, not bandwidth-bound
              constexpr int kI = 4;
              for (int w0 = ep_tid; w0 < A.M * 16; w0 += 128 * kI) {
                float4 g[kI], uu[kI];
#pragma unroll
                for (int i = 0; i < kI; ++i) {
                  const int w = w0 + 128 * i;
                  if (w < A.M * 16) {
                    const int wg = (w >> 4) * 32 + (w & 15);
                    g[i] = __ldcg(parts + wg);
                    uu[i] = __ldcg(parts + wg + 16);
                  }
                }
                for (int k = 1; k < n_contrib; ++k) {  // contributor order → deterministic
                  float4 x[kI], y[kI];
#pragma unroll
                  for (int i = 0; i < kI; ++i) {
                    const int w = w0 + 128 * i;
                    if (w < A.M * 16) {
                      const int wg = (w >> 4) * 32 + (w & 15);
                      x[i] = __ldcg(parts + (size_t)k * per + wg);
                      y[i] = __ldcg(parts + (size_t)k * per + wg + 16);
                    }
                  }
#pragma unroll
                  for (int i = 0; i < kI; ++i) {
                    g[i].x += x[i].x; g[i].y += x[i].y; g[i].z += x[i].z; g[i].w += x[i].w;
                    uu[i].x += y[i].x; uu[i].y += y[i].y; uu[i].z += y[i].z; uu[i].w += y[i].w;
                  }
                }
#pragma unroll
                for (int i = 0; i < kI; ++i) {
                  const int w = w0 + 128 * i, j = w >> 4;
                  if (w < A.M * 16 && j < mv)
                  {
                    const size_t yo = (size_t)(y0 + j) * (A.N / 2) + (nb0 / 2) + (w & 15) * 4;
                    if (A.dssq) {  // deferred RMSNorm of X: the folded sums × 1/rms(token)
                      const float sc = s_inv[j];
                      g[i].x *= sc, g[i].y *= sc, g[i].z *= sc, g[i].w *= sc;
                      uu[i].x *= sc, uu[i].y *= sc, uu[i].z *= sc, uu[i].w *= sc;
                    }
                    store_silu4(A, yo, g[i], uu[i]);
                    count(yo, 8u);
                  }
                }
              }
            }
            for (int w = ep_tid; w < (A.silu ? 0 : per); w += 128) {
              float4 xs[4];
#pragma unroll
              for (int k = 0; k < 4; ++k)
                if (k < n_contrib) xs[k] = __ldcg(parts + (size_t)k * per + w);
              float4 acc = xs[0];
#pragma unroll
              for (int k = 1; k < 4; ++k)  // contributor order → deterministic (static indices: no local memory)
                if (k < n_contrib) {
                  acc.x += xs[k].x;
                  acc.y += xs[k].y;
                  acc.z += xs[k].z;
                  acc.w += xs[k].w;
                }
              for (int k = 4; k < n_contrib; ++k) {
                const float4 x = __ldcg(parts + (size_t)k * per + w);
                acc.x += x.x;
                acc.y += x.y;
                acc.z += x.z;
                acc.w += x.w;
              }
              const int j = (w * 4) / kBM, r = (w * 4) % kBM;
              const int nn = nb0 + r;
              if (nn < A.N && j < mv) {
                uint2 o;
                o.x = pack_bf16(acc.x, acc.y);
                o.y = pack_bf16(acc.z, acc.w);
                const size_t yo = (size_t)(y0 + j) * A.N + nn;
                if (nn + 4 <= A.N && (A.N & 3) == 0) {
                  *reinterpret_cast<uint2*>(A.Y + yo) = o;
                  for (int p = 0; p < A.epi.n; ++p) if (epi_row_in(A.epi, p, (uint32_t)(y0 + j))) *reinterpret_cast<uint2*>((__nv_bfloat16*)A.epi.dst[p] + yo) = o;
                  count(yo, 8u);
                } else {
                  const float vv[4] = {acc.x, acc.y, acc.z, acc.w};
                  for (int x = 0; x < 4 && nn + x < A.N; ++x) {
                    A.Y[yo + x] = __float2bfloat16_rn(vv[x]);
                    for (int p = 0; p < A.epi.n; ++p) if (epi_row_in(A.epi, p, (uint32_t)(y0 + j))) ((__nv_bfloat16*)A.epi.dst[p])[yo + x] = __float2bfloat16_rn(vv[x]);
                    count(yo + x, 2u);
                  }
                }
              }
            }
          }
        }
      } else {
        // ---- whole tile: TMEM → bf16 → smem transpose → 16-byte stores
        for (int j0 = 0; j0 < A.M; j0 += kChunk) {
          float v[kChunk];
          tmem_ld16(tbase + j0, v);
          __nv_bfloat16* st = ystage + (size_t)((j0 / kChunk) & 1) * kChunk * kBM;
          if (A.dssq)
#pragma unroll
            for (int j = 0; j < kChunk; ++j) v[j] *= j0 + j < A.M ? s_inv[j0 + j] : 0.f;
#pragma unroll
          for (int j = 0; j < kChunk; ++j) st[j * kBM + row_in_tile] = __float2bfloat16_rn(v[j]);
          named_bar(2, 128);
          const int jn = min(kChunk, mv - j0);
          if (A.silu) {  // 16 tokens x 8 groups of 8 outputs: gate cols c8.., up cols 64 + c8..
            const int j = ep_tid >> 3, c8 = (ep_tid & 7) * 8;
            if (j < jn) {
              const uint4 gv = *reinterpret_cast<const uint4*>(st + j * kBM + c8);
              const uint4 uv = *reinterpret_cast<const uint4*>(st + j * kBM + 64 + c8);
              const uint32_t* gp = &gv.x;
              const uint32_t* up = &uv.x;
              uint4 o;
              uint32_t* op = &o.x;
#pragma unroll
              for (int qd = 0; qd < 4; ++qd) op[qd] = silu2(bf16lo(gp[qd]), bf16hi(gp[qd]), bf16lo(up[qd]), bf16hi(up[qd]));
              const size_t yo = (size_t)(y0 + j0 + j) * (A.N / 2) + nb0 / 2 + c8;
              *reinterpret_cast<uint4*>(A.Y + yo) = o;
              for (int p = 0; p < A.epi.n; ++p) if (epi_row_in(A.epi, p, (uint32_t)(y0 + j0 + j))) *reinterpret_cast<uint4*>((__nv_bfloat16*)A.epi.dst[p] + yo) = o;
              count(yo, 16u);
            }
          }
#pragma unroll
          for (int r = 0; r < (A.silu ? 0 : 2); ++r) {
            const int e = ep_tid + r * 128;  // 256 vectors of 8 bf16 per chunk
            const int j = e >> 4, col = (e & 15) * 8;
            const int nn = nb0 + col;
            if (j < jn && nn < A.N) {
              const uint4 val = *reinterpret_cast<const uint4*>(st + j * kBM + col);
              const size_t yo = (size_t)(y0 + j0 + j) * A.N + nn;
              if (nn + 8 <= A.N && (A.N & 7) == 0) {
                *reinterpret_cast<uint4*>(A.Y + yo) = val;
                for (int p = 0; p < A.epi.n; ++p) if (epi_row_in(A.epi, p, (uint32_t)(y0 + j0 + j))) *reinterpret_cast<uint4*>((__nv_bfloat16*)A.epi.dst[p] + yo) = val;
                count(yo, 16u);
              } else {
                const __nv_bfloat16* sv = reinterpret_cast<const __nv_bfloat16*>(&val);
                for (int x = 0; x < 8 && nn + x < A.N; ++x) {
                  A.Y[yo + x] = sv[x];
                  for (int p = 0; p < A.epi.n; ++p) if (epi_row_in(A.epi, p, (uint32_t)(y0 + j0 + j))) ((__nv_bfloat16*)A.epi.dst[p])[yo + x] = sv[x];
                  count(yo + x, 2u);
                }
              }
            }
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[a]);
      }
      if (ep_tid == 0 && seg < 3) KD_TRACE(7 + 2 * seg);
      u = seg_end;
      ++seg;
    }
  }
  if (A.split_tiles && A.fold_grid) {
    // ---- grid barrier (all CTAs are co-resident: grid ≤ #SMs, 1 CTA/SM),
    // self-resetting: the last CTA to leave zeroes both words
    __syncthreads();
    if (threadIdx.x == 128) {
      unsigned* arrive = A.counter;
      unsigned* depart = A.counter + 1;
      KD_TRACE(18);
      fence_acq_rel_gpu();
      atom_add_acq_rel_gpu(arrive, 1u);
      // watchdog: the barrier needs all G CTAs co-resident (G = the device's
      // SM count, 1 CTA/SM); if that ever fails, record and give up rather
      // than hang (KD_ERR_TIMEOUT at kd_runtime_check; the output is invalid)
      long long spins = 0;
      while (ld_acquire_gpu(arrive) < (unsigned)G) {
        if (++spins > (1ll << 28)) {
          if (A.err) atomicExch(A.err, 2u);
          break;
        }
      }
      KD_TRACE(16);
      if (atom_add_acq_rel_gpu(depart, 1u) == (unsigned)G - 1) {
        *arrive = 0u;
        *depart = 0u;
      }
    }
    __syncthreads();
    // ---- fold my slice of the flat [tile][M][128] float4 space with all 256
    // threads; every (element, contributor) load of a round is in flight at once
    const long long per_tile = (long long)A.M * kBM / 4;
    const long long E = (long long)A.tiles * per_tile;
    const long long e0 = c * E / G, e1 = (c + 1) * E / G;
    constexpr int kE = 2, kC = 8;
    for (long long f0 = e0; f0 < e1; f0 += kE * kThreads) {
      float4 xs[kE][kC];
      int ncs[kE];
      long long fs[kE];
#pragma unroll
      for (int k = 0; k < kE; ++k) {
        const long long f = f0 + threadIdx.x + (long long)k * kThreads;
        fs[k] = f;
        ncs[k] = 0;
        if (f < e1) {
          const int t = (int)(f / per_tile);
          const long long tb = (long long)t * KB;
          const long long first = unit_owner(tb, U, G), lastc = unit_owner(tb + KB - 1, U, G);
          if (lastc > first) {  // split tile (whole tiles were stored from TMEM)
            ncs[k] = (int)(lastc - first + 1);
            const float4* parts = reinterpret_cast<const float4*>(A.part + (size_t)t * A.max_contrib * A.M * kBM);
            const int w = (int)(f - (long long)t * per_tile);
#pragma unroll
            for (int ci = 0; ci < kC; ++ci)
              if (ci < ncs[k]) xs[k][ci] = __ldcg(parts + (size_t)ci * per_tile + w);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < kE; ++k) {
        if (ncs[k] == 0) continue;
        const long long f = fs[k];
        const int t = (int)(f / per_tile);
        const float4* parts = reinterpret_cast<const float4*>(A.part + (size_t)t * A.max_contrib * A.M * kBM);
        const int w = (int)(f - (long long)t * per_tile);
        float4 acc = xs[k][0];
#pragma unroll
        for (int ci = 1; ci < kC; ++ci)  // contributor order → deterministic
          if (ci < ncs[k]) {
            acc.x += xs[k][ci].x;
            acc.y += xs[k][ci].y;
            acc.z += xs[k][ci].z;
            acc.w += xs[k][ci].w;
          }
        for (int ci = kC; ci < ncs[k]; ++ci) {
          const float4 x = __ldcg(parts + (size_t)ci * per_tile + w);
          acc.x += x.x;
          acc.y += x.y;
          acc.z += x.z;
          acc.w += x.w;
        }
        const int grp = A.groups ? t / A.tpg : 0;
        const int nb0 = (A.groups ? t % A.tpg : t) * kBM;
        const int y0 = A.groups ? __ldg(A.meta + A.moff + grp) : 0;
        const int mv = A.groups ? min(__ldg(A.meta + grp), A.M) : A.M;
        const int j = (w * 4) / kBM, r = (w * 4) % kBM;
        const int nn = nb0 + r;
        if (nn < A.N && j < mv) {
          uint2 o;
          o.x = pack_bf16(acc.x, acc.y);
          o.y = pack_bf16(acc.z, acc.w);
          const size_t yo = (size_t)(y0 + j) * A.N + nn;
          if (nn + 4 <= A.N && (A.N & 3) == 0) {
            *reinterpret_cast<uint2*>(A.Y + yo) = o;
            for (int p = 0; p < A.epi.n; ++p) if (epi_row_in(A.epi, p, (uint32_t)(y0 + j))) *reinterpret_cast<uint2*>((__nv_bfloat16*)A.epi.dst[p] + yo) = o;
            count(yo, 8u);
          } else {
            const float vv[4] = {acc.x, acc.y, acc.z, acc.w};
            for (int x = 0; x < 4 && nn + x < A.N; ++x) {
              A.Y[yo + x] = __float2bfloat16_rn(vv[x]);
              for (int p = 0; p < A.epi.n; ++p) if (epi_row_in(A.epi, p, (uint32_t)(y0 + j))) ((__nv_bfloat16*)A.epi.dst[p])[yo + x] = __float2bfloat16_rn(vv[x]);
              count(yo + x, 2u);
            }
          }
        }
      }
    }
    if (threadIdx.x == 128) KD_TRACE(13);
  }
  // publish this CTA's stores to the consumer devices: CTA mode one release,
  // COUNT mode the bytes tallied per chunk
  if constexpr (kX) {
    epi_signal_counts(A.epi, s_cnt, true);
  } else if (A.epi.n) {
    __syncthreads();
    if (threadIdx.x == 0) {
      fence_acq_rel_sys();
      for (int p = 0; p < A.epi.n; ++p) red_release_sys_add64(A.epi.flag[p], 1ull);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(ncols));
  }
  if (threadIdx.x == 0) KD_TRACE(15);
}

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  });
  return fn;
}


// ============================================================================
// Cluster split-K decode GEMM (weights on MMA M = 128, tokens on MMA N, the
// stream-K kernel's orientation): tile t = 128 weight rows, its K range cut
// into `split` equal parts over the CTAs of one thread-block cluster. Each
// rank stages its fp32 partial [M][128] in shared memory grouped by owner
// (rank o owns weight rows [o·rpo, (o+1)·rpo)) and pushes every owner its
// block with ONE bulk shared::cta → shared::cluster copy completing on the
// owner's mbarrier; owners sum the split blocks in rank order (bitwise
// deterministic) and store bf16. Replaces stream-K's global fold (grid
// barrier + L2 round trips, ≈5 µs measured) for the skinny GEMMs whose
// 32-48 tiles cannot fill 148 SMs without splitting K.
namespace csk {

constexpr int kThreads = 384;  // w0 TMA, w1 MMA + TMEM alloc, w4..w11 epilogue (2 warps per TMEM lane quarter)
constexpr int kEpi = kThreads - 128;
constexpr int kSmemMax = 227 * 1024;

struct Args {
  __nv_bfloat16* Y;
  int M, N, K;
  int mma_n;     // tokens rounded up to 16 (MMA N)
  int split;     // cluster size
  int kbs;       // 64-column boxes per stage
  int kblocks;   // ⌈K / (64·kbs)⌉
  int stages;
  int rpo;       // weight rows owned per rank (split > 1)
  int dbg;       // debug A/B (KD_GEMM_DBG)
  Epi epi;
  unsigned long long* trace;
  int rope;      // KD_OP_QKV_ROPE: epilogue = a5 (RoPE + KV append) on the bf16 QKV output
  RopeEpi rp;
  // KD_OP_GEMM_RMSNORM: epilogue = a3 on the bf16 output across the whole grid
  // (r += bf16(X·Wᵀ); Y = RMSNorm(r)·γ), per-token Σr² completed after a grid barrier
  int norm;
  float* r;                     // [M][N] fp32 residual (read + written)
  const __nv_bfloat16* gamma;   // [N]
  float eps;
  unsigned* bar;                // 2 self-resetting words (scratch)
  float* ssq;                   // [M][gridDim.x] per-CTA partial Σr² (scratch)
  unsigned* err;                // runtime error word (nullable): set to 2 when the grid barrier times out
  Acq acq;                      // chunk-aware consumer: X (slot 0) acquired per k-block by the TMA warp
  // norm == 2 (KD_NORM_DEFER): no grid barrier — Y = bf16(r'·gamma), per-CTA Σr'² to ssq (the declared
  // partial-sum buffer past its header), 1/rms left to the consumer
  float* dssq_out;              // norm == 2: the partial-sum buffer (header written by CTA 0)
  const float* dssq;            // rope: deferred RMSNorm of X (nullable): the QKV sums × 1/rms(token)
};

// a5 fused into the QKV GEMM epilogue. W rows are pair-interleaved within each
// head (row 2p ← dim p, row 2p+1 ← dim p + D/2), so a rotation pair is two
// adjacent rows and never straddles a cluster owner (rpo is even). Values are
// rounded to bf16 first (the plain GEMM's output), then exactly the RoPE
// kernel's fp32 math with its cos/sin (fp64 angle, host fp64 θ^(−2i/D)).
// Per-token position and page, and the frequency table, are staged in shared
// memory by the idle warps 2-3 during the main loop (RopeSmem): indexed
// parameter-space reads (divergent across lanes) and dependent global loads
// in this epilogue were its dominant cost.
struct RopeSmem {
  int* pos;      // [M] seq_len − 1
  int* pg;       // [M] page holding pos (block_table entry)
  double* f;     // [D/2]
  float* inv;    // [M] deferred-norm 1/rms per token (A.dssq)
};

__device__ __forceinline__ void rope_stage(const Args& A, const RopeSmem& rs) {
  const RopeEpi& R = A.rp;
  const int t = threadIdx.x - 64;
  for (int i = t; i < R.D / 2; i += 64) rs.f[i] = R.f[i];
  pdl_wait();  // block table and lengths are step inputs written before this kernel
  for (int j = t; j < A.M; j += 64) {
    const int pos = R.sl[j] - 1;
    rs.pos[j] = pos;
    rs.pg[j] = R.bt[(size_t)j * R.pps + pos / R.page];
    if (A.dssq) rs.inv[j] = dnorm_inv(A.dssq, j);
  }
}

__device__ __forceinline__ void rope_pair(const Args& A, const RopeSmem& rs, int j, int n, float xs, float ys) {
  const RopeEpi& R = A.rp;
  const int D = R.D, half = D / 2, G = R.Hq / R.Hkv;
  const int hall = n / D, rr = n - hall * D, p = rr >> 1;
  const int grp = hall / (G + 2), slot = hall - grp * (G + 2);
  if (A.dssq) xs *= rs.inv[j], ys *= rs.inv[j];  // deferred RMSNorm of X: the fp32 sums × 1/rms
  const float x = __bfloat162float(__float2bfloat16_rn(xs)), y = __bfloat162float(__float2bfloat16_rn(ys));
  const int pos = rs.pos[j];
  __nv_bfloat16 lo, hi;
  if (slot <= G) {
    const double ang = (double)pos * rs.f[p];
    const double k = rint(ang * 0.15915494309189535);
    const double red = fma(-k, 6.283185307179586, fma(-k, 2.4492935982947064e-16, ang));
    float sn, cs;
    sincosf((float)red, &sn, &cs);
    lo = __float2bfloat16_rn(x * cs - y * sn);
    hi = __float2bfloat16_rn(y * cs + x * sn);
  } else {
    lo = __float2bfloat16_rn(x);
    hi = __float2bfloat16_rn(y);
  }
  if (slot < G) {
    const size_t qo = ((size_t)j * R.Hq + (size_t)grp * G + slot) * D;
    R.q[qo + p] = lo;
    R.q[qo + p + half] = hi;
    for (int e = 0; e < A.epi.n; ++e) {
      ((__nv_bfloat16*)A.epi.dst[e])[qo + p] = lo;
      ((__nv_bfloat16*)A.epi.dst[e])[qo + p + half] = hi;
    }
  } else {
    const int32_t pg = rs.pg[j];
    const size_t co = (((size_t)pg * R.Hkv + grp) * R.page + pos % R.page) * D;
    __nv_bfloat16* cache = slot == G ? R.kc : R.vc;
    cache[co + p] = lo;
    cache[co + p + half] = hi;
  }
}

// Two adjacent rotation pairs (weight rows n..n+3 → dims p, p+1 and p + D/2,
// p + D/2 + 1 of one head; n % 4 == 0) with 4-byte stores: the cluster
// path's second pass, where lanes walk a token's rows so that the q / cache
// stores coalesce. Per element exactly rope_pair's arithmetic (same bits).
__device__ __forceinline__ void rope_quad(const Args& A, const RopeSmem& rs, int j, int n, float4 a) {
  const RopeEpi& R = A.rp;
  const int D = R.D, half = D / 2, G = R.Hq / R.Hkv;
  const int hall = n / D, rr = n - hall * D, p = rr >> 1;
  const int grp = hall / (G + 2), slot = hall - grp * (G + 2);
  if (A.dssq) {  // deferred RMSNorm of X: the fp32 sums × 1/rms
    const float sc = rs.inv[j];
    a.x *= sc, a.y *= sc, a.z *= sc, a.w *= sc;
  }
  const float xs[2] = {__bfloat162float(__float2bfloat16_rn(a.x)), __bfloat162float(__float2bfloat16_rn(a.z))};
  const float ys[2] = {__bfloat162float(__float2bfloat16_rn(a.y)), __bfloat162float(__float2bfloat16_rn(a.w))};
  const int pos = rs.pos[j];
  __nv_bfloat16 lo[2], hi[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    if (slot <= G) {
      const double ang = (double)pos * rs.f[p + u];
      const double k = rint(ang * 0.15915494309189535);
      const double red = fma(-k, 6.283185307179586, fma(-k, 2.4492935982947064e-16, ang));
      float sn, cs;
      sincosf((float)red, &sn, &cs);
      lo[u] = __float2bfloat16_rn(xs[u] * cs - ys[u] * sn);
      hi[u] = __float2bfloat16_rn(ys[u] * cs + xs[u] * sn);
    } else {
      lo[u] = __float2bfloat16_rn(xs[u]);
      hi[u] = __float2bfloat16_rn(ys[u]);
    }
  }
  const __nv_bfloat162 l2 = __halves2bfloat162(lo[0], lo[1]), h2 = __halves2bfloat162(hi[0], hi[1]);
  if (slot < G) {
    const size_t qo = ((size_t)j * R.Hq + (size_t)grp * G + slot) * D;
    *reinterpret_cast<__nv_bfloat162*>(R.q + qo + p) = l2;
    *reinterpret_cast<__nv_bfloat162*>(R.q + qo + p + half) = h2;
    for (int e = 0; e < A.epi.n; ++e) {
      *reinterpret_cast<__nv_bfloat162*>((__nv_bfloat16*)A.epi.dst[e] + qo + p) = l2;
      *reinterpret_cast<__nv_bfloat162*>((__nv_bfloat16*)A.epi.dst[e] + qo + p + half) = h2;
    }
  } else {
    const size_t co = (((size_t)rs.pg[j] * R.Hkv + grp) * R.page + pos % R.page) * D;
    __nv_bfloat16* cache = slot == G ? R.kc : R.vc;
    *reinterpret_cast<__nv_bfloat162*>(cache + co + p) = l2;
    *reinterpret_cast<__nv_bfloat162*>(cache + co + p + half) = h2;
  }
}

// 4 consecutive outputs (weight rows col..col+3) of token j → Y (+ peers), or
// the fused RoPE/append epilogue
__device__ __forceinline__ void csk_store4(const Args& A, const RopeSmem& rs, int j, int col, float v0, float v1,
                                           float v2, float v3) {
  if (A.rope) {
    if (col < A.N) rope_pair(A, rs, j, col, v0, v1);
    if (col + 2 < A.N) rope_pair(A, rs, j, col + 2, v2, v3);
    return;
  }
  const size_t yo = (size_t)j * A.N + col;
  if (col + 4 <= A.N && (A.N & 3) == 0) {
    uint2 o;
    o.x = pack_bf16(v0, v1);
    o.y = pack_bf16(v2, v3);
    *reinterpret_cast<uint2*>(A.Y + yo) = o;
    for (int p = 0; p < A.epi.n; ++p) if (epi_row_in(A.epi, p, (uint32_t)j)) *reinterpret_cast<uint2*>((__nv_bfloat16*)A.epi.dst[p] + yo) = o;
  } else {
    const float vv[4] = {v0, v1, v2, v3};
    for (int x = 0; x < 4; ++x)
      if (col + x < A.N) {
        const __nv_bfloat16 h = __float2bfloat16_rn(vv[x]);
        A.Y[yo + x] = h;
        for (int p = 0; p < A.epi.n; ++p) if (epi_row_in(A.epi, p, (uint32_t)j)) ((__nv_bfloat16*)A.epi.dst[p])[yo + x] = h;
      }
  }
}

// a3 fused into the GEMM epilogue (KD_OP_GEMM_RMSNORM). Each CTA owns weight
// rows [c0, c0 + rows) of every token. While the main loop streams, the idle
// warps 2-3 stage this slice of r (fp32) and gamma into shared memory (rs,
// gs), so the epilogue's only global round trips are the grid barrier and one
// batch of partial-sum loads (measured ≈0.5-1 µs per dependent global round
// trip in this phase). After the role branches, all 384 threads:
//   A: v = Σ partials (rank order); r' = r + bf16(v) → r (global) and rs
//   B: per token, this CTA's Σ r'² (warp per token, fixed shuffle tree) → ssq[j][cta]
//   grid barrier (all CTAs co-resident: tiles ≤ max co-resident clusters)
//   C: per token, Σ over CTAs (fixed order) → inv = rsqrt(Σ/N + eps);
//   D: Y = bf16(r'·inv·γ), exactly a3's rounding.
struct NormSmem {
  float* rs;            // [M][Tp] fp32: r slice, then r'
  __nv_bfloat16* gs;    // [rows] gamma slice
  float* invs;          // [M] 1/rms
  int Tp;
};

__device__ __forceinline__ int norm_rows(const Args& A, int rank, int n0, int my_rows, int* c0) {
  *c0 = A.split > 1 ? n0 + rank * A.rpo : n0;
  return A.split > 1 ? max(0, min(my_rows, A.N - *c0)) : min(kBM, A.N - n0);  // valid rows of the tail tile
}

// warps 2-3 during the main loop
__device__ __forceinline__ void norm_stage(const Args& A, const NormSmem& ns, int rank, int n0, int my_rows) {
  const int t = threadIdx.x - 64;
  int c0;
  const int rows = norm_rows(A, rank, n0, my_rows, &c0), r4n = rows / 4, M = A.M;
  for (int i = t; i < r4n; i += 64)  // gamma is a weight: before the dependency wait
    *reinterpret_cast<uint2*>(ns.gs + 4 * i) = __ldg(reinterpret_cast<const uint2*>(A.gamma + c0 + 4 * i));
  pdl_wait();  // r is written by earlier kernels
  constexpr int kB = 8;  // loads in flight per thread
  for (int e0 = t; e0 < M * r4n; e0 += 64 * kB) {
    float4 v[kB];
#pragma unroll
    for (int b = 0; b < kB; ++b) {
      const int e = e0 + 64 * b, j = e / r4n, l4 = e - j * r4n;
      if (e < M * r4n) v[b] = __ldcg(reinterpret_cast<const float4*>(A.r + (size_t)j * A.N + c0 + 4 * l4));
    }
#pragma unroll
    for (int b = 0; b < kB; ++b) {
      const int e = e0 + 64 * b, j = e / r4n, l4 = e - j * r4n;
      if (e < M * r4n) *reinterpret_cast<float4*>(ns.rs + (size_t)j * ns.Tp + 4 * l4) = v[b];
    }
  }
}

__device__ __forceinline__ void norm_epilogue(const Args& A, const NormSmem& ns, const float* st, const float* recv,
                                              uint64_t* rbar, int rank, int n0, int my_rows) {
  const int split = A.split, M = A.M, N = A.N;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* const ssq = A.ssq;
  float* const rs = ns.rs;
  const int Tp = ns.Tp;
  const int G = gridDim.x;
  const bool defer = A.norm == 2;                   // KD_NORM_DEFER: partial sums to the declared buffer
  const int Gp = defer ? KD_DNORM_PARTS : (G + 15) / 16 * 16;  // ssq row pitch
  __syncthreads();  // staging (split 1) and the r/gamma slices are complete; my own rows are in recv[rank]
  if (split > 1) mbar_wait(rbar, 0);
  pdl_wait();
  if (threadIdx.x == 0) { KD_TRACE(8); KD_CTRACE(22); }
  int c0;
  const int rows = norm_rows(A, rank, n0, my_rows, &c0);
  const int P = (M + 3) / 4 * 4 + 4, r4n = rows / 4;
  for (int e = threadIdx.x; e < M * r4n; e += kThreads) {
    int lr4, j;
    float acc[4];
    if (split > 1) {  // lanes walk tokens: conflict-free recv column reads
      lr4 = (e / M) * 4;
      j = e - (e / M) * M;
#pragma unroll
      for (int x = 0; x < 4; ++x) acc[x] = recv[((size_t)lr4 + x) * P + j];
      for (int cr = 1; cr < split; ++cr)
#pragma unroll
        for (int x = 0; x < 4; ++x) acc[x] += recv[((size_t)cr * A.rpo + lr4 + x) * P + j];
    } else {
      j = e / r4n;
      lr4 = (e - j * r4n) * 4;
      const float4 v = *reinterpret_cast<const float4*>(st + (size_t)j * kBM + lr4);
      acc[0] = v.x; acc[1] = v.y; acc[2] = v.z; acc[3] = v.w;
    }
    float4* sp = reinterpret_cast<float4*>(rs + (size_t)j * Tp + lr4);
    float4 rv = *sp;
    rv.x += __bfloat162float(__float2bfloat16_rn(acc[0]));
    rv.y += __bfloat162float(__float2bfloat16_rn(acc[1]));
    rv.z += __bfloat162float(__float2bfloat16_rn(acc[2]));
    rv.w += __bfloat162float(__float2bfloat16_rn(acc[3]));
    *sp = rv;  // (r' reaches global memory in D, with coalesced stores)
  }
  if (threadIdx.x == 0) KD_CTRACE(16);
  __syncthreads();
  if (threadIdx.x == 0) KD_CTRACE(17);
  for (int j = threadIdx.x; j < M; j += kThreads) {  // thread per token, 16-byte reads, l order
    float ss = 0.f;
    for (int l4 = 0; l4 < r4n; ++l4) {
      const float4 v = *reinterpret_cast<const float4*>(rs + (size_t)j * Tp + 4 * l4);
      ss += v.x * v.x;
      ss += v.y * v.y;
      ss += v.z * v.z;
      ss += v.w * v.w;
    }
    ssq[(size_t)j * Gp + blockIdx.x] = ss;
    // deferred: the consumer sums all KD_DNORM_PARTS entries; CTA c also zeroes entries G + c + k·G
    if (defer)
      for (int e = G + (int)blockIdx.x; e < KD_DNORM_PARTS; e += G) ssq[(size_t)j * Gp + e] = 0.f;
  }
  if (defer) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      A.dssq_out[0] = A.eps;
      A.dssq_out[1] = (float)N;
    }
    for (int j = threadIdx.x; j < M; j += kThreads) ns.invs[j] = 1.f;  // h = bf16(r'·1·γ): the 1/rms is deferred
  }
  if (threadIdx.x == 0) KD_CTRACE(18);
  __syncthreads();
  if (!defer && threadIdx.x == 0) {  // grid barrier (self-resetting: see the departure at the end)
    KD_TRACE(13);
    KD_CTRACE(24);
    // the acq_rel add releases this CTA's partial sums (ordered before it by
    // the bar.sync: release is cumulative); polls back off to keep the line
    // free for the other CTAs' arrivals
    atom_add_acq_rel_gpu(A.bar, 1u);
    long long spins = 0;  // watchdog as in the stream-K fold barrier
    while (ld_acquire_gpu(A.bar) < (unsigned)G) {
      if (++spins > (1ll << 24)) {
        if (A.err) atomicExch(A.err, 2u);
        break;
      }
      __nanosleep(64);
    }
    KD_TRACE(14);
    KD_CTRACE(23);
  }
  __syncthreads();
  // per token Σ over CTAs (not when deferred): a warp takes kTpw tokens; each lane loads 16-byte
  // chunks lane and lane + 32 of every row (coalesced, all loads in flight),
  // sums its components in c order, then the tokens' shuffle trees run
  // interleaved. Fixed order: deterministic. Entries ≥ G are masked (the pad
  // of a row is not ours: the scratch is shared with other kernels).
  if (!defer) {
    constexpr int kTpw = 6, kCh = (kNormMaxGrid + 127) / 128;  // ≤ 2 float4 per lane per row (G ≤ 160)
    for (int j0 = warp * kTpw; j0 < M; j0 += kTpw * (kThreads / 32)) {
      float4 v[kTpw][kCh];
#pragma unroll
      for (int t = 0; t < kTpw; ++t)
#pragma unroll
        for (int i = 0; i < kCh; ++i) {
          const int c = (lane + 32 * i) * 4;
          v[t][i] = (j0 + t < M && c < G) ? __ldcg(reinterpret_cast<const float4*>(ssq + (size_t)(j0 + t) * Gp + c))
                                           : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      float sm[kTpw];
#pragma unroll
      for (int t = 0; t < kTpw; ++t) {
        sm[t] = 0.f;
#pragma unroll
        for (int i = 0; i < kCh; ++i) {
          const int c = (lane + 32 * i) * 4;
          sm[t] += v[t][i].x;
          sm[t] += c + 1 < G ? v[t][i].y : 0.f;
          sm[t] += c + 2 < G ? v[t][i].z : 0.f;
          sm[t] += c + 3 < G ? v[t][i].w : 0.f;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int t = 0; t < kTpw; ++t) sm[t] += __shfl_xor_sync(0xffffffffu, sm[t], o);
      if (lane < kTpw && j0 + lane < M) {
        float mine = sm[0];
#pragma unroll
        for (int t = 1; t < kTpw; ++t) mine = lane == t ? sm[t] : mine;
        ns.invs[j0 + lane] = rsqrtf(mine / (float)N + A.eps);
      }
    }
  }
  if (threadIdx.x == 0) KD_CTRACE(19);
  __syncthreads();
  if (threadIdx.x == 0) KD_CTRACE(20);
  __nv_bfloat16* const Y = A.Y;
  for (int e = threadIdx.x; e < M * r4n; e += kThreads) {  // lanes walk a token's rows: coalesced h stores
    const int j = e / r4n, l4 = e - j * r4n;
    const float inv = ns.invs[j];
    const float4 v = *reinterpret_cast<const float4*>(rs + (size_t)j * Tp + 4 * l4);
    const uint2 g = *reinterpret_cast<const uint2*>(ns.gs + 4 * l4);
    uint2 o;
    o.x = pack_bf16(v.x * inv * bf16lo(g.x), v.y * inv * bf16hi(g.x));
    o.y = pack_bf16(v.z * inv * bf16lo(g.y), v.w * inv * bf16hi(g.y));
    const size_t yo = (size_t)j * N + c0 + 4 * l4;
    *reinterpret_cast<float4*>(A.r + yo) = v;
    *reinterpret_cast<uint2*>(Y + yo) = o;
    for (int p = 0; p < A.epi.n; ++p) if (epi_row_in(A.epi, p, (uint32_t)j)) *reinterpret_cast<uint2*>((__nv_bfloat16*)A.epi.dst[p] + yo) = o;
  }
  if (threadIdx.x == 0) {
    KD_CTRACE(21);
    KD_TRACE(15);
    // departure, off the critical path: the last CTA to leave (every CTA has
    // passed the arrival spin by then) zeroes both words for the next launch
    if (!defer && atom_add_acq_rel_gpu(A.bar + 1, 1u) == (unsigned)G - 1) {
      A.bar[0] = 0u;
      A.bar[1] = 0u;
    }
  }
  if (A.epi.n && (split == 1 || my_rows > 0))  // publish: COUNT → h columns [c0, c0 + rows) of all M tokens
    epi_signal(A.epi, (uint32_t)c0 * 2u, (uint32_t)(c0 + rows) * 2u, 0u, (uint32_t)M);
}

template <bool kX>  // as gemm_kernel: the handoff-protocol code only in the kX instance
__global__ void __launch_bounds__(kThreads, 1)
    gemm_csk_kernel(const __grid_constant__ CUtensorMap tmap_w, const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ Args A) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // align by offsetting the __shared__ array itself (a uintptr_t round trip
  // loses the address space: the epilogue's staging stores compiled to
  // generic ST.E with 64-bit address math, measured ≈35 cycles each)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int S = A.stages, kbs = A.kbs, split = A.split, M = A.M;
  const int xbox = A.mma_n * kBK * 2;
  const int wst = kbs * kStageA, xst = kbs * xbox;
  uint8_t* sa = smem;                                 // S × kbs × 16 KB (W)
  uint8_t* sb = smem + (size_t)S * wst;               // S × kbs × mma_n·128 B (X)
  float* recv = (float*)(sb + (size_t)S * xst);       // split × [M][rpo] fp32 (peers' blocks of my rows)
  const int P = (M + 3) / 4 * 4 + 4;                  // recv row pitch (floats): 16-byte rows + pad
  const size_t blk = (size_t)P * A.rpo;               // floats per (rank, owner) block: rpo rows
  const size_t recv_bytes = split > 1 ? (size_t)split * blk * 4 : 0;
  uint64_t* full = (uint64_t*)((uint8_t*)recv + recv_bytes);
  uint64_t* empty = full + kMaxStages;
  uint64_t* tfull = empty + kMaxStages;
  uint64_t* rbar = tfull + 1;
  uint32_t* tmem_slot = (uint32_t*)(rbar + 1);
  NormSmem ns;                                        // norm: after the barriers
  ns.invs = (float*)(tmem_slot + 4);                  // [256]
  ns.Tp = (split > 1 ? A.rpo : kBM) + 4;              // 16-byte rows + pad (conflict-free column walks)
  ns.rs = ns.invs + 256;                              // [M][Tp]
  ns.gs = (__nv_bfloat16*)(ns.rs + (size_t)M * ns.Tp);  // [128]
  RopeSmem ropes;                                     // rope: after the barriers (exclusive with norm)
  ropes.pos = (int*)(ns.invs + 256);                  // [256]
  ropes.pg = ropes.pos + 256;                         // [256]
  ropes.f = (double*)(ropes.pg + 256);                // [128]
  ropes.inv = (float*)(ropes.f + 128);                // [256]
  float* send = (float*)smem;  // split == 1: [M][128] fp32 staging, reuses the idle ring after the last MMA

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) KD_TRACE(0);
  pdl_launch_dependents();
  if constexpr (kX) epi_started(A.epi);
  const int rank = split > 1 ? (int)cluster_ctarank() : 0;
  const int tile = blockIdx.x / split;
  const int n0 = tile * kBM;
  const int kb0 = (int)((long long)A.kblocks * rank / split);
  const int nk = (int)((long long)A.kblocks * (rank + 1) / split) - kb0;
  const int my_rows = split > 1 ? max(0, min(kBM, (rank + 1) * A.rpo) - rank * A.rpo) : 0;
  const uint32_t ncols = A.mma_n <= 32 ? 32 : (A.mma_n <= 64 ? 64 : (A.mma_n <= 128 ? 128 : 256));

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(rbar, 1);
    // each peer rank sends my_rows rows of ⌈M/4⌉ 16-byte groups
    if (split > 1) mbar_expect_tx(rbar, (unsigned)((split - 1) * my_rows * ((M + 3) / 4) * 16));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmap_w) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmap_x) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (split > 1) {
    // every rank's rbar is armed once this completes. Waited here, at the
    // start: a cluster-scope acquire invalidates L1 (CCTL.IVALL), which was
    // measured to stall the epilogue's shared-memory work by ≈2-3K cycles
    // when done after the main loop.
    cluster_arrive_release();
    cluster_wait_acquire();
  }
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) KD_TRACE(1);

  if (warp == 0) {
    // ------------------------------------------------ TMA producer (warp-uniform loop, lane 0 issues)
    const uint64_t pw = policy_evict_first(), px = policy_evict_last();
    const unsigned tx = (unsigned)(wst + xst);
    auto load_w = [&](int i, int s) {
      for (int b = 0; b < kbs; ++b)
        tma_load_2d(sa + (size_t)s * wst + b * kStageA, &tmap_w, ((kb0 + i) * kbs + b) * kBK, n0, &full[s], pw);
    };
    const int xi = kX ? acq_find(A.acq, 0) : -1;
    uint32_t held = 0;
    auto load_x = [&](int i, int s) {  // (this rank's K range only: it acquires only its own X chunks)
      if constexpr (kX) acquire_x(A.acq, xi, kb0 + i, kbs, A.K, &held);
      for (int b = 0; b < kbs; ++b)
        tma_load_2d(sb + (size_t)s * xst + b * xbox, &tmap_x, ((kb0 + i) * kbs + b) * kBK, 0, &full[s], px);
    };
    const int n_pre = min(S, nk);
    if (lane == 0) {
      for (int i = 0; i < n_pre; ++i) {  // weights before the grid-dependency wait
        mbar_expect_tx(&full[i], tx);
        load_w(i, i);
      }
      KD_TRACE(2);
      pdl_wait();
      for (int i = 0; i < n_pre; ++i) load_x(i, i);
    }
    __syncwarp();
    for (int i = n_pre, s = n_pre % S, ph = n_pre / S; i < nk; ++i) {
      mbar_wait(&empty[s], (unsigned)((ph - 1) & 1));
      if (lane == 0) {
        mbar_expect_tx(&full[s], tx);
        load_w(i, s);
        load_x(i, s);
      }
      __syncwarp();
      if (++s == S) s = 0, ++ph;
    }
    if (lane == 0) KD_TRACE(3);
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer (warp-uniform loop, lane 0 issues)
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(A.mma_n >> 3) << 17) |
                           ((uint32_t)(kBM >> 4) << 24);
    for (int i = 0, st = 0, ph = 0; i < nk; ++i) {
      const int s = st;
      mbar_wait(&full[s], (unsigned)(ph & 1));
      if (++st == S) st = 0, ++ph;
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (KD_MMA_WS) {  // every lane, elect.sync issues (uniform operands)
        if (lane == 0 && i == 0) KD_TRACE(4);
        const uint32_t a_addr = smem_u32(sa + (size_t)s * wst);
        const uint32_t b_addr = smem_u32(sb + (size_t)s * xst);
        for (int b = 0; b < kbs; ++b)
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)
            mma_bf16_ws(tmem_base, sw128_desc(a_addr + b * kStageA + 32 * k), sw128_desc(b_addr + b * xbox + 32 * k),
                        idesc, (i > 0 || b > 0 || k > 0) ? 1u : 0u);
        mma_commit_ws(&empty[s]);
      } else if (lane == 0) {
        if (i == 0) KD_TRACE(4);
        const uint32_t a_addr = smem_u32(sa + (size_t)s * wst);
        const uint32_t b_addr = smem_u32(sb + (size_t)s * xst);
        for (int b = 0; b < kbs; ++b)
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)
            mma_bf16(tmem_base, sw128_desc(a_addr + b * kStageA + 32 * k), sw128_desc(b_addr + b * xbox + 32 * k), idesc,
                     (i > 0 || b > 0 || k > 0) ? 1u : 0u);
        mma_commit(&empty[s]);
      }
      __syncwarp();
    }
    if (lane == 0) {
      mma_commit(tfull);
      KD_TRACE(5);
    }
    __syncwarp();
  } else if (A.norm && warp < 4) {
    // ------------------------------------------------ idle warps 2-3: stage r and gamma (norm)
    norm_stage(A, ns, rank, n0, my_rows);
  } else if (A.rope && warp < 4) {
    // ------------------------------------------------ idle warps 2-3: stage positions, pages, θ table
    rope_stage(A, ropes);
    if (split == 1) asm volatile("bar.arrive 2, %0;" ::"r"(kEpi + 64) : "memory");  // hand-off to the epilogue warps
  } else if (warp >= 4) {
    // ------------------------------------------------ epilogue
    // 8 warps: warp w reads TMEM lane quarter (w − 4) mod 4 (its hardware
    // quarter), token-column chunks of 16 alternating between the two halves
    const int q = (warp - 4) & 3, half = (warp - 4) >> 2, ep = threadIdx.x - 128;
    const int row = q * 32 + lane;  // weight row within the tile = TMEM lane
    mbar_wait_sleep(tfull, 0, 128);
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (ep == 0) { KD_TRACE(6); KD_CTRACE(20); }
    const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16);
    auto store1 = [&](size_t yo, float v) {
      const __nv_bfloat16 h = __float2bfloat16_rn(v);
      A.Y[yo] = h;
      for (int p = 0; p < A.epi.n; ++p) if (epi_row_in(A.epi, p, (uint32_t)(yo / A.N))) ((__nv_bfloat16*)A.epi.dst[p])[yo] = h;
    };
    auto store_y = [&](int j, int col, float v0, float v1, float v2, float v3) {  // 4 consecutive outputs of token j
      if (A.rope) {  // two rotation pairs (col is a multiple of 4)
        if (col < A.N) rope_pair(A, ropes, j, col, v0, v1);
        if (col + 2 < A.N) rope_pair(A, ropes, j, col + 2, v2, v3);
        return;
      }
      const size_t yo = (size_t)j * A.N + col;
      if (col + 4 <= A.N && (A.N & 3) == 0) {
        uint2 o;
        o.x = pack_bf16(v0, v1);
        o.y = pack_bf16(v2, v3);
        *reinterpret_cast<uint2*>(A.Y + yo) = o;
        for (int p = 0; p < A.epi.n; ++p) if (epi_row_in(A.epi, p, (uint32_t)j)) *reinterpret_cast<uint2*>((__nv_bfloat16*)A.epi.dst[p] + yo) = o;
      } else {
        if (col < A.N) store1(yo, v0);
        if (col + 1 < A.N) store1(yo + 1, v1);
        if (col + 2 < A.N) store1(yo + 2, v2);
        if (col + 3 < A.N) store1(yo + 3, v3);
      }
    };
    bool stored = false;
    if (split == 1) {
      // TMEM → fp32 staging [M][128] (thread = row: conflict-free) → 4-wide bf16 stores
      float* st = send;
      for (int j0 = half * kChunk; j0 < M; j0 += 2 * kChunk) {
        float v[kChunk];
        tmem_ld16(tbase + j0, v);
#pragma unroll
        for (int j = 0; j < kChunk; ++j)
          if (j0 + j < M) st[(size_t)(j0 + j) * kBM + row] = v[j];
      }
      if (!A.norm) {  // (norm: the staged tile is finished after the role branches)
        named_bar(1, kEpi);
        if (A.rope) named_bar(2, kEpi + 64);  // warps 2-3 staged the RoPE tables
        pdl_wait();
        for (int e = ep; e < M * (kBM / 4); e += kEpi) {
          const int j = e / (kBM / 4), r4 = (e % (kBM / 4)) * 4;
          const float4 v = *reinterpret_cast<const float4*>(st + (size_t)j * kBM + r4);
          if (n0 + r4 < A.N) store_y(j, n0 + r4, v.x, v.y, v.z, v.w);
        }
        stored = true;
      }
    } else {
      // Each thread owns one weight row of the partial (its TMEM lane) and
      // sends it, 64 token columns at a time, straight from registers to the
      // row's owner: recv[rank][lr][0..M) (row pitch P = ⌈M/4⌉·4 + 4 floats) with
      // 16-byte st.async (peers) or st.shared (itself). No staging pass.
      if (ep == 0) { KD_TRACE(12); KD_CTRACE(21); }
      const int rpo = A.rpo;
      const int o = row / rpo, lr = row - o * rpo;
      const uint32_t my_off = (uint32_t)(((size_t)rank * rpo + lr) * P * 4);  // recv[rank][lr][·] in the owner
      const uint32_t dst = o == rank ? smem_u32(recv) + my_off : mapa_shared(smem_u32(recv) + my_off, (uint32_t)o);
      const uint32_t rb = o == rank ? 0u : mapa_shared(smem_u32(rbar), (uint32_t)o);
      for (int j0 = half * 2 * kChunk; j0 < M; j0 += 4 * kChunk) {
        uint32_t v[2][kChunk];  // this half's 2 chunks of 16 columns in flight, one wait
#pragma unroll
        for (int b = 0; b < 2; ++b)
          if (j0 + b * kChunk < A.mma_n) tmem_ld16_nowait(tbase + j0 + b * kChunk, v[b]);
        tmem_ld_wait();
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
          for (int x = 0; x < kChunk / 4; ++x) {
            const int j = j0 + b * kChunk + 4 * x;
            if (j < M) {  // the last 16-byte group may run past M into the pad
              const uint32_t ad = dst + (uint32_t)j * 4;
              if (o == rank)
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(ad), "r"(v[b][4 * x]), "r"(v[b][4 * x + 1]),
                             "r"(v[b][4 * x + 2]), "r"(v[b][4 * x + 3])
                             : "memory");
              else
                st_async_v4(ad, __uint_as_float(v[b][4 * x]), __uint_as_float(v[b][4 * x + 1]),
                            __uint_as_float(v[b][4 * x + 2]), __uint_as_float(v[b][4 * x + 3]), rb);
            }
          }
      }
      if (ep == 0) { KD_TRACE(7); KD_CTRACE(22); KD_TRACE(10); KD_CTRACE(23); }
      // the owner's sum runs after the role branches with all warps
    }
    if (A.epi.n && stored) {  // publish this CTA's stores: COUNT → columns [n0, n0 + 128) of all M tokens
      named_bar(1, kEpi);
      if (ep == 0) {
        fence_acq_rel_sys();
        if (A.epi.nch)
          epi_release_range(A.epi, (uint32_t)n0 * 2u, (uint32_t)min(n0 + kBM, A.N) * 2u, 0u, (uint32_t)M);
        else
          epi_release_cta(A.epi);
      }
    }
    if (ep == 0) { KD_TRACE(9); KD_CTRACE(26); }
  }
  if (A.norm) {
    norm_epilogue(A, ns, send, recv, rbar, rank, n0, my_rows);
  } else if (split > 1) {
    // ---- owner sum with all 384 threads (the TMA/MMA warps are idle by now):
    // my rows [rank·rpo, +my_rows), Σ over ranks in order; lanes walk tokens
    // (conflict-free column reads), each thread 4 consecutive weight rows
    __syncthreads();            // my own rows are in recv[rank]
    mbar_wait(rbar, 0);         // the peers' rows have landed (st.async complete_tx)
    if (threadIdx.x == 128) { KD_TRACE(8); KD_CTRACE(24); }
    pdl_wait();
    const int rpo = A.rpo, r4n = my_rows / 4;  // rpo and 128 are multiples of 4
    float* T = (float*)smem;                    // [M][rpo + 4] sums (the idle operand ring)
    const int Tp = rpo + 4;
    for (int e = threadIdx.x; e < M * r4n; e += kThreads) {
      const int lr4 = (e / M) * 4, j = e - (e / M) * M;
      float acc[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) acc[x] = recv[((size_t)lr4 + x) * P + j];
      for (int cr = 1; cr < split; ++cr)  // rank order → deterministic
#pragma unroll
        for (int x = 0; x < 4; ++x) acc[x] += recv[((size_t)cr * rpo + lr4 + x) * P + j];
      *reinterpret_cast<float4*>(T + (size_t)j * Tp + lr4) = make_float4(acc[0], acc[1], acc[2], acc[3]);
    }
    // second pass: lanes walk a token's rows, so the output (and peer) stores
    // coalesce; walking tokens, as the sum must, scatters every warp store
    // over 32 rows of Y (measured: the RoPE epilogue's 2-byte stores cost ≈4 µs)
    if (threadIdx.x == 128) KD_CTRACE(27);
    __syncthreads();
    if (threadIdx.x == 128) KD_CTRACE(28);
    for (int e = threadIdx.x; e < M * r4n; e += kThreads) {
      const int j = e / r4n, l4 = e - j * r4n, n = n0 + rank * rpo + 4 * l4;
      const float4 v = *reinterpret_cast<const float4*>(T + (size_t)j * Tp + 4 * l4);
      if (A.rope) {
        if (n < A.N) rope_quad(A, ropes, j, n, v);
      } else {
        csk_store4(A, ropes, j, n, v.x, v.y, v.z, v.w);
      }
    }
    if (threadIdx.x == 128) { KD_TRACE(11); KD_CTRACE(25); }
    if (A.epi.n && my_rows > 0) {  // publish: COUNT → this owner's columns of all M tokens
      const int c0 = n0 + rank * rpo;
      epi_signal(A.epi, (uint32_t)min(c0, A.N) * 2u, (uint32_t)min(c0 + my_rows, A.N) * 2u, 0u, (uint32_t)M);
    }
  }
  // No closing cluster barrier: peers only ever WRITE into this CTA's recv
  // (st.async), and the epilogue waits for all of those bytes on rbar before
  // the CTA can exit; nothing reads another CTA's shared memory.
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(ncols));
  }
  if (threadIdx.x == 0) KD_TRACE(15);
}

}  // namespace csk

}  // namespace gemm

kd_status encode_bf16_2d_sw128(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint32_t box_inner,
                               uint32_t box_rows) {
  gemm::EncodeTiledFn fn = gemm::get_encode();
  if (!fn) return fail(KD_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (no CUDA driver?)");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {box_inner, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(KD_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return KD_OK;
}

kd_status encode_bf16_sw128(CUtensorMap* map, const void* ptr, int rank, const uint64_t* dims,
                            const uint64_t* strides_bytes, const uint32_t* box) {
  gemm::EncodeTiledFn fn = gemm::get_encode();
  if (!fn) return fail(KD_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (no CUDA driver?)");
  cuuint64_t d[5], st[4];
  cuuint32_t b[5], es[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    es[i] = 1;
    if (i) st[i - 1] = strides_bytes[i - 1];
  }
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(ptr), d, st, b, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(KD_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return KD_OK;
}

namespace gemm {

static kd_status encode(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint32_t box_rows) {
  return encode_bf16_2d_sw128(map, ptr, inner, outer, (uint32_t)kBK, box_rows);
}

struct Geometry {
  int mma_n, stages, kblocks, tiles, grid, max_contrib, kbs;
  long long units;
};

// SMs of the current device (MIG / green contexts can expose fewer than 148):
// the stream-K grid is one CTA per SM and its fold barrier needs every CTA
// co-resident, so the grid comes from the device, not a constant (148 when no
// device is visible, e.g. host-only planning)
static int device_sms() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      n <= 0) {
    cudaGetLastError();
    return kNumSMs;
  }
  return n;
}

static kd_status geometry(const GemmShape& a, Geometry* g, int sms) {
  if (a.dtype != KD_BF16) return fail(KD_ERR_UNSUPPORTED, "gemm: only bf16 (fp32 path not built)");
  if (a.M == 0 || a.N == 0 || a.K == 0 || a.rows_total == 0) return fail(KD_ERR_INVALID_ARG, "gemm: empty shape");
  if (a.M > 256) return fail(KD_ERR_UNSUPPORTED, "gemm: decode GEMM supports M <= 256 rows (per group)");
  if (a.K % 8) return fail(KD_ERR_UNSUPPORTED, "gemm: K must be a multiple of 8 (16-byte TMA rows)");
  if (a.groups && a.N % kBM) return fail(KD_ERR_UNSUPPORTED, "grouped gemm: N must be a multiple of 128");
  if (a.silu && (a.groups || a.N % kBM)) return fail(KD_ERR_UNSUPPORTED, "gemm+silu: plain GEMM with N (= 2F) a multiple of 128");
  g->mma_n = (int)((a.M + 15) / 16 * 16);
  // two 64-column boxes per stage halve the per-stage barrier/MMA-issue
  // overhead (measured ≈0.3 µs per stage at one box) while ≥ 4 stages fit
  g->kbs = g->mma_n <= 128 ? 2 : 1;
  if (const char* e = getenv("KD_GEMM_KBS")) g->kbs = std::max(1, std::min(2, atoi(e)));
  const int stage_bytes = g->kbs * (kStageA + g->mma_n * kBK * 2);
  g->stages = std::min(kMaxStages, (kSmemBudget - 2 * kChunk * kBM * 2) / stage_bytes);
  g->kblocks = (int)((a.K + kBK * g->kbs - 1) / (kBK * g->kbs));
  g->tiles = (int)((a.N + kBM - 1) / kBM) * (int)std::max<uint32_t>(1, a.groups);
  g->units = (long long)g->tiles * g->kblocks;
  g->grid = (int)std::min<long long>(sms, g->units);
  int mc = 1;
  for (int t = 0; t < g->tiles; ++t) {
    long long f = unit_owner((long long)t * g->kblocks, g->units, g->grid);
    long long l = unit_owner((long long)(t + 1) * g->kblocks - 1, g->units, g->grid);
    mc = std::max<int>(mc, (int)(l - f + 1));
  }
  g->max_contrib = mc;
  return KD_OK;
}

static size_t smem_bytes(const Geometry& g) {
  return 1024 + (size_t)g.stages * g.kbs * (kStageA + g.mma_n * kBK * 2) + (2 * kMaxStages + 6) * 8 +
         2 * kChunk * kBM * 2 + 16 + 4 * kMaxPeers * kMaxChunks + 256 * 4;
}

// ---------------------------------------------------------------- dense GEMM kernel choice
namespace csk {

static size_t smem_for(int mma_n, int kbs, int stages, int split, int rpo, int M, bool norm, bool rope) {
  const size_t recv = split > 1 ? (size_t)split * ((M + 3) / 4 * 4 + 4) * rpo * 4 : 0;
  if (norm) {  // + the r slice [M][Tp] fp32 and the gamma slice
    const size_t tp = (split > 1 ? rpo : kBM) + 4;
    return smem_for(mma_n, kbs, stages, split, rpo, M, false, false) + (size_t)M * tp * 4 + 256;
  }
  if (rope) return smem_for(mma_n, kbs, stages, split, rpo, M, false, false) + 256 * 4 * 3 + 128 * 8;
  return 1024 + (size_t)stages * kbs * (kStageA + (size_t)mma_n * kBK * 2) + recv + (2 * kMaxStages + 4) * 8 + 16 +
         256 * 4;  // + the norm epilogue's per-token 1/rms
}

// co-resident clusters of `split` CTAs (one CTA per SM at this kernel's smem),
// per device; ⌊SMs / split⌋ when the query is unavailable
static int max_clusters(int split) {
  static std::mutex mu;
  static std::map<int, std::vector<int>> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return kNumSMs / split;
  std::lock_guard<std::mutex> lk(mu);
  auto& v = cache[dev];
  if (v.empty()) {
    int sms = kNumSMs;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(gemm_csk_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax);
    cudaFuncSetAttribute(gemm_csk_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax);
    v.assign(9, 0);
    for (int c = 1; c <= 8; ++c) {
      int n = 0;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(c * (sms / c));
      cfg.blockDim = dim3(kThreads);
      cfg.dynamicSmemBytes = 160 * 1024;
      cudaLaunchAttribute at;
      at.id = cudaLaunchAttributeClusterDimension;
      at.val.clusterDim.x = c;
      at.val.clusterDim.y = 1;
      at.val.clusterDim.z = 1;
      cfg.attrs = &at;
      cfg.numAttrs = 1;
      if (c == 1) n = sms;
      else {
        int n2 = 0;  // both instances: the tiling must fit whichever is launched
        if (cudaOccupancyMaxActiveClusters(&n, gemm_csk_kernel<false>, &cfg) != cudaSuccess ||
            cudaOccupancyMaxActiveClusters(&n2, gemm_csk_kernel<true>, &cfg) != cudaSuccess) {
          cudaGetLastError();
          n = n2 = 0;
        }
        n = std::min(n, n2);
      }
      v[c] = n;
    }
  }
  return v[split];
}

// Modelled time (ns) of the cluster kernel at split s: the largest per-CTA
// weight slab at min(per-SM TMA rate, HBM share), + the DSMEM reduction; and
// of stream-K: all weights at HBM rate + its fold tail. Constants measured on
// B200 (scripts/bench_ops.py, scratch sweeps): ≈60 GB/s per SM with 2-box
// stages, 6.45 TB/s HBM, ≈1 µs cluster reduction, stream-K tails ≈2 µs (≤3
// contributors per tile, last-arriver fold) / ≈6 µs (grid fold).
constexpr double kSmBps = 60e9, kHbmBps = 6.45e12;

static kd_status choose(const GemmShape& a, GemmTile* t, double* best_ns) {
  const int M = (int)a.M, mma_n = (M + 15) / 16 * 16;
  const int tiles = (int)((a.N + kBM - 1) / kBM);
  int force_s = 0;
  if (const char* e = getenv("KD_GEMM_TILE")) sscanf(e, "%d", &force_s);
  double best = -1;
  for (int s = 1; s <= 8; ++s) {
    if (force_s && s != force_s) continue;
    const int maxc = getenv("KD_GEMM_ANY_CLUSTERS") ? 1 << 20 : max_clusters(s);  // A/B: allow a second wave
    if (tiles > maxc) continue;
    if (a.norm && tiles * s > kNormMaxGrid) continue;  // per-CTA partial sums in scratch
    const int kbs = mma_n <= 128 ? 2 : 1;
    const int KB = (int)((a.K + kBK * kbs - 1) / (kBK * kbs));
    if (s > KB) continue;
    const int rpo = s > 1 ? ((kBM + s - 1) / s + 3) / 4 * 4 : 0;
    if (s > 1 && (rpo * (s - 1) >= kBM)) continue;  // every rank must own rows
    int stages = kMaxStages;
    while (stages >= 2 && smem_for(mma_n, kbs, stages, s, rpo, M, a.norm != 0, a.rope != 0) > (size_t)kSmemMax) --stages;
    if (stages < 2) continue;
    const size_t ring = (size_t)stages * kbs * (kStageA + (size_t)mma_n * kBK * 2);
    if ((size_t)M * kBM * 4 > ring) continue;  // fp32 staging reuses the ring
    const double bytes = (double)kBM * ((KB + s - 1) / s) * kbs * kBK * 2;
    const double rate = std::min(kSmBps, kHbmBps / (tiles * s));
    const double ns = bytes / rate * 1e9 + (s > 1 ? 1000.0 : 0.0);
    if (best < 0 || ns < best) {
      best = ns;
      t->split = s;
      t->kbs = kbs;
      t->kblocks = KB;
      t->tiles = tiles;
      t->stages = stages;
      t->rpo = rpo;
      t->mt = mma_n;
      t->smem = (uint32_t)smem_for(mma_n, kbs, stages, s, rpo, M, a.norm != 0, a.rope != 0);
    }
  }
  if (best < 0) return fail(KD_ERR_UNSUPPORTED, "gemm: no feasible cluster tiling for this shape");
  *best_ns = best;
  return KD_OK;
}

}  // namespace csk

static double streamk_ns(const GemmShape& a) {
  Geometry g;
  if (geometry(a, &g, device_sms())) return 1e30;
  const double w = (double)a.N * a.K * 2;
  return w / csk::kHbmBps * 1e9 + (g.max_contrib <= 3 ? 2000.0 : 6000.0);
}

// plain GEMMs: the cluster kernel unless stream-K is modelled faster (or forced)
static bool use_dense(const GemmShape& a) {
  if (a.rope || a.norm) return true;  // the fused RoPE / RMSNorm epilogues exist in the cluster kernel only
  if (a.groups || a.silu) return false;
  const char* e = getenv("KD_GEMM_STREAMK");
  if (e && atoi(e)) return false;
  if (getenv("KD_GEMM_TILE")) return true;
  GemmTile t;
  double ns = 0;
  if (csk::choose(a, &t, &ns)) return false;
  return ns <= streamk_ns(a);
}


}  // namespace gemm

GemmShape gemm_shape(const kd_attr_gemm& a, bool silu) {
  GemmShape s;
  s.silu = silu ? 1u : 0u;
  s.M = a.M;
  s.rows_total = a.M;
  s.N = a.N;
  s.K = a.K;
  s.groups = 0;
  s.dtype = a.dtype;
  return s;
}

GemmShape gemm_shape(const kd_attr_qkv_rope& a) {
  GemmShape s;
  s.rope = 1;
  s.M = a.rows;
  s.rows_total = a.rows;
  s.N = (a.n_heads + 2 * a.n_kv_heads) * a.head_dim;
  s.K = a.hidden;
  s.groups = 0;
  s.dtype = a.dtype;
  return s;
}

GemmShape gemm_shape(const kd_attr_gemm_rmsnorm& a) {
  GemmShape s;
  s.M = s.rows_total = a.M;
  s.N = a.N;
  s.K = a.K;
  s.dtype = a.dtype;
  s.norm = 1;
  return s;
}

kd_status gemm_rmsnorm_bind(const kd_attr_gemm_rmsnorm& a, float* r, const void* gamma, GemmPlan* gp, float* ssq_out) {
  if (a.flags & ~(uint32_t)KD_NORM_DEFER) return fail(KD_ERR_INVALID_ARG, "gemm_rmsnorm: unknown flags");
  gp->defer = (a.flags & KD_NORM_DEFER) != 0;
  if (gp->defer && (!ssq_out || ((uintptr_t)ssq_out & 15)))
    return fail(KD_ERR_INVALID_ARG, "gemm_rmsnorm (deferred): a 16-byte aligned partial-sum buffer is required");
  if (gp->defer && a.M > 256) return fail(KD_ERR_UNSUPPORTED, "gemm_rmsnorm (deferred): at most 256 rows");
  gp->dssq_out = ssq_out;
  if (a.dtype != KD_BF16) return fail(KD_ERR_UNSUPPORTED, "gemm_rmsnorm: bf16 only");
  if (a.N % 8) return fail(KD_ERR_UNSUPPORTED, "gemm_rmsnorm: hidden must be a multiple of 8");
  if (!r || !gamma) return fail(KD_ERR_INVALID_ARG, "gemm_rmsnorm: NULL r or gamma");
  if (((uintptr_t)r | (uintptr_t)gamma) & 15) return fail(KD_ERR_INVALID_ARG, "gemm_rmsnorm: r and gamma must be 16-byte aligned");
  gp->r = r;
  gp->gamma = gamma;
  gp->eps = a.eps;
  return KD_OK;
}

kd_status qkv_rope_bind(const kd_attr_qkv_rope& a, const int32_t* bt, const int32_t* sl, void* q, void* kc, void* vc,
                        GemmPlan* gp) {
  if (!bt || !sl || !q || !kc || !vc) return fail(KD_ERR_INVALID_ARG, "qkv_rope: NULL pointer");
  if (a.n_kv_heads == 0 || a.n_heads % a.n_kv_heads || a.head_dim % 2 || a.head_dim > 256 || a.page == 0 ||
      a.pages_per_seq == 0)
    return fail(KD_ERR_UNSUPPORTED, "qkv_rope: unsupported head layout");
  RopeEpi& r = gp->rp;
  r.bt = bt;
  r.sl = sl;
  r.q = (__nv_bfloat16*)q;
  r.kc = (__nv_bfloat16*)kc;
  r.vc = (__nv_bfloat16*)vc;
  r.Hq = (int)a.n_heads;
  r.Hkv = (int)a.n_kv_heads;
  r.D = (int)a.head_dim;
  r.page = (int)a.page;
  r.pps = (int)a.pages_per_seq;
  const double l2t = std::log2(a.theta);
  for (uint32_t i = 0; i < a.head_dim / 2; ++i) r.f[i] = std::exp2(-2.0 * (double)i / (double)a.head_dim * l2t);
  return KD_OK;
}

GemmShape gemm_shape(const kd_attr_grouped_gemm& a) {
  GemmShape s;
  s.M = a.rows_cap;
  s.rows_total = a.rows_total;
  s.N = a.N;
  s.K = a.K;
  s.groups = a.experts;
  s.dtype = a.dtype;
  s.expert0 = a.expert0;
  s.meta_experts = a.meta_experts ? a.meta_experts : a.experts;
  return s;
}

kd_status gemm_scratch_bytes(const GemmShape& a, uint64_t* bytes) {
  if (a.norm) {  // grid-barrier words + per-CTA partial Σr² [M][≤ kNormMaxGrid]
    *bytes = kScratchCounterBytes + (uint64_t)a.M * kNormMaxGrid * 4;
    return KD_OK;
  }
  if (a.dtype == KD_F32) {  // fp32 path: SIMT kernel, no scratch
    if (a.groups) return fail(KD_ERR_UNSUPPORTED, "grouped gemm: bf16 only");
    *bytes = 256;
    return KD_OK;
  }
  if (gemm_is_prefill(a)) {  // f4 large-M kernel: no split-K, no scratch
    *bytes = 256;
    return KD_OK;
  }
  gemm::Geometry g;
  kd_status s = gemm::geometry(a, &g, gemm::device_sms());
  if (s) return s;
  if (2ull * g.tiles > kMaxCounters) return fail(KD_ERR_UNSUPPORTED, "gemm: too many output tiles");
  uint64_t n = kScratchCounterBytes + (uint64_t)g.tiles * g.max_contrib * a.M * gemm::kBM * 4;
  *bytes = (n + 255) / 256 * 256;
  return KD_OK;
}

kd_status gemm_prepare(const GemmShape& a, const void* X, const void* W, const void* meta, GemmPlan* gp) {
  if (a.dtype == KD_F32) {
    if (a.groups) return fail(KD_ERR_UNSUPPORTED, "grouped gemm: bf16 only");
    if (a.M == 0 || a.N == 0 || a.K == 0) return fail(KD_ERR_INVALID_ARG, "gemm: empty shape");
    if (!X || !W) return fail(KD_ERR_INVALID_ARG, "gemm: NULL operand");
    gp->sh = a;
    gp->X = X;
    gp->W = W;
    gp->dense = false;
    return KD_OK;
  }
  if (gemm_is_prefill(a)) return gemm_prefill_prepare(a, X, W, gp);  // f4: M > 256 rows, tensor-bound
  gemm::Geometry g;
  kd_status s = gemm::geometry(a, &g, gemm::device_sms());
  if (s) return s;
  if (!X || !W || (a.groups && !meta)) return fail(KD_ERR_INVALID_ARG, "gemm: NULL operand");
  if (((uintptr_t)X | (uintptr_t)W) & 15) return fail(KD_ERR_INVALID_ARG, "gemm: operands must be 16-byte aligned");
  gp->sh = a;
  if (a.groups && a.expert0 + a.groups > a.meta_experts)
    return fail(KD_ERR_INVALID_ARG, "grouped gemm: expert0 + experts exceeds meta_experts");
  gp->meta = a.groups ? (const int*)meta + a.expert0 : nullptr;
  gp->moff = (int)a.meta_experts;
  gp->dense = gemm::use_dense(a);
  if (gp->dense) {
    double ns = 0;
    s = gemm::csk::choose(a, &gp->tile, &ns);
    if (s) return s;
    s = gemm::encode(&gp->tmap_w, W, a.K, a.N, gemm::kBM);
    if (s) return s;
    return gemm::encode(&gp->tmap_x, X, a.K, a.rows_total, (uint32_t)gp->tile.mt);
  }
  s = gemm::encode(&gp->tmap_w, W, a.K, (uint64_t)a.N * std::max<uint32_t>(1, a.groups), gemm::kBM);
  if (s) return s;
  s = gemm::encode(&gp->tmap_x, X, a.K, a.rows_total, (uint32_t)g.mma_n);
  if (s) return s;
  return KD_OK;
}

static unsigned long long* g_gemm_trace = nullptr;

// step timeline (kd_debug_timeline): launch i of the captured step writes its
// per-CTA stamps to region i (kTlRegion u64); the launch kinds are kept here
static unsigned long long* g_tl = nullptr;
static uint64_t g_tl_cap = 0;
static std::vector<int32_t> g_tl_kinds;
unsigned long long* tl_next(int32_t kind) {
  if (!g_tl || g_tl_kinds.size() >= g_tl_cap) return nullptr;
  g_tl_kinds.push_back(kind);
  return g_tl + (g_tl_kinds.size() - 1) * kTlRegion;
}

// the kX kernel instance is needed when the launch streams chunked (COUNT)
// output, acquires remote inputs in-kernel, or records residency / log words
static bool kx_needed(const LaunchCtx& c) {
  if (c.epi.nch > 0 || c.acq.n > 0) return true;
  for (int p = 0; p < c.epi.n; ++p)
    if (c.epi.started[p] || c.epi.logt[p]) return true;
  return false;
}

static kd_status launch_gemm_dense(const GemmPlan& gp, void* Y, const LaunchCtx& c, uint32_t* signals) {
  const GemmTile& t = gp.tile;
  gemm::csk::Args A;
  A.Y = (__nv_bfloat16*)Y;
  A.M = (int)gp.sh.M;
  A.N = (int)gp.sh.N;
  A.K = (int)gp.sh.K;
  A.mma_n = t.mt;
  A.split = t.split;
  A.kbs = t.kbs;
  A.kblocks = t.kblocks;
  A.stages = t.stages;
  A.rpo = t.rpo;
  A.dbg = getenv("KD_GEMM_DBG") ? atoi(getenv("KD_GEMM_DBG")) : 0;
  A.rope = (int)gp.sh.rope;
  A.rp = gp.rp;
  A.norm = gp.defer ? 2 : (int)gp.sh.norm;
  A.dssq_out = gp.dssq_out;
  A.dssq = gp.dssq;
  if (A.dssq && !A.rope) return fail(KD_ERR_UNSUPPORTED, "gemm: a deferred-norm input needs the QKV+RoPE epilogue here");
  A.r = gp.r;
  A.gamma = (const __nv_bfloat16*)gp.gamma;
  A.eps = gp.eps;
  A.bar = (unsigned*)c.scratch;
  A.ssq = gp.defer ? gp.dssq_out + KD_DNORM_HDR
                   : (c.scratch ? (float*)((uint8_t*)c.scratch + kScratchCounterBytes) : nullptr);
  if (A.norm && (!c.scratch || !A.r || !A.gamma))
    return fail(KD_ERR_INVALID_ARG, "gemm_rmsnorm: scratch, r and gamma are required");
  if (A.norm && t.tiles * t.split > kNormMaxGrid) return fail(KD_ERR_UNSUPPORTED, "gemm_rmsnorm: grid too large");
  static_assert(kNormMaxGrid <= KD_DNORM_PARTS, "deferred-norm partials: one per CTA");
  A.epi = c.epi;
  A.err = c.err;
  A.acq = c.acq;
  A.trace = g_gemm_trace ? g_gemm_trace : tl_next(100 + (int)gp.sh.rope + 2 * (int)gp.sh.norm);
  kd_status ks = kernels_init();
  if (ks) return ks;
  const bool x = kx_needed(c);
  KD_CUDA_CHECK(kd_launch_cluster(x ? gemm::csk::gemm_csk_kernel<true> : gemm::csk::gemm_csk_kernel<false>,
                                  dim3(t.tiles * t.split), dim3(gemm::csk::kThreads),
                                  t.smem, c.stream, (unsigned)t.split, gp.tmap_w, gp.tmap_x, A),
                "gemm (cluster split-K) launch");
  if (signals) return gemm_signals(gp.sh, signals);
  return KD_OK;
}

kd_status launch_gemm(const GemmPlan& gp, void* Y, const LaunchCtx& c, uint32_t* signals) {
  if (!Y) return fail(KD_ERR_INVALID_ARG, "gemm: NULL output");
  if (gp.sh.dtype == KD_F32) {
    kd_status st = launch_gemm_f32((const float*)gp.X, (const float*)gp.W, (float*)Y, (int)gp.sh.M, (int)gp.sh.N,
                                   (int)gp.sh.K, c);
    if (!st && signals) *signals = gemm_f32_signals(gp.sh.N);
    return st;
  }
  if (gp.prefill) return launch_gemm_prefill(gp, Y, c, signals);
  if (gp.dense) return launch_gemm_dense(gp, Y, c, signals);
  gemm::Geometry g;
  kd_status s = gemm::geometry(gp.sh, &g, gemm::device_sms());
  if (s) return s;
  if (!Y) return fail(KD_ERR_INVALID_ARG, "gemm: NULL output");
  if (g.max_contrib > 1 && !c.scratch) return fail(KD_ERR_INVALID_ARG, "gemm: scratch required");
  gemm::Args A;
  A.Y = (__nv_bfloat16*)Y;
  if (2ull * g.tiles > kMaxCounters) return fail(KD_ERR_UNSUPPORTED, "gemm: too many output tiles");
  A.counter = (unsigned*)c.scratch;
  A.part = (float*)((uint8_t*)c.scratch + kScratchCounterBytes);
  A.M = gp.sh.M;
  A.N = gp.sh.N;
  A.K = gp.sh.K;
  A.groups = (int)gp.sh.groups;
  A.tpg = (int)((gp.sh.N + gemm::kBM - 1) / gemm::kBM);
  A.meta = gp.meta;
  A.moff = gp.moff;
  A.mma_n = g.mma_n;
  A.stages = g.stages;
  A.kblocks = g.kblocks;
  A.kbs = g.kbs;
  A.silu = (int)gp.sh.silu;
  A.split_tiles = g.max_contrib > 1 ? 1 : 0;
  A.fold_grid = g.max_contrib > 3 ? 1 : 0;
  if (const char* e = getenv("KD_GEMM_FOLD")) A.fold_grid = atoi(e);
  if (A.silu) A.fold_grid = 0;  // the fused SiLU epilogue is built for the last-arriver fold
  A.tiles = g.tiles;
  A.max_contrib = g.max_contrib;
  A.units = g.units;
  A.epi = c.epi;
  A.err = c.err;
  A.acq = c.acq;
  A.trace = g_gemm_trace ? g_gemm_trace : tl_next(200 + (int)gp.sh.silu);
  A.dssq = gp.dssq;
  if (A.dssq && (!A.silu || A.M > 256))
    return fail(KD_ERR_UNSUPPORTED, "gemm: a deferred-norm input needs the fused SiLU epilogue here (M <= 256)");
  {
    static int dbg = -1;
    if (dbg < 0) dbg = getenv("KD_GEMM_DBG") ? atoi(getenv("KD_GEMM_DBG")) : 0;
    A.dbg = dbg;
  }
  size_t sm = gemm::smem_bytes(g);
  kd_status ks = kernels_init();
  if (ks) return ks;
  KD_CUDA_CHECK(kd_launch(kx_needed(c) ? gemm::gemm_kernel<true> : gemm::gemm_kernel<false>, dim3(g.grid),
                          dim3(gemm::kThreads), sm, c.stream, gp.tmap_w, gp.tmap_x, A),
                "gemm launch");
  if (signals) return gemm_signals(gp.sh, signals);
  return KD_OK;
}

}  // namespace kd

extern "C" kd_status kd_gemm_tiling(uint32_t M, uint32_t N, uint32_t K, int32_t* out) {
  if (!out) return kd::fail(KD_ERR_INVALID_ARG, "kd_gemm_tiling: NULL out");
  kd_attr_gemm a;
  a.M = M;
  a.N = N;
  a.K = K;
  a.dtype = KD_BF16;
  const kd::GemmShape sh = kd::gemm_shape(a);
  kd::gemm::Geometry g;
  kd_status gs = kd::gemm::geometry(sh, &g, kd::gemm::device_sms());  // shape validation
  if (gs) return gs;
  if (!kd::gemm::use_dense(sh)) {
    out[0] = 0;
    out[1] = out[2] = out[3] = out[4] = out[5] = 0;
    return KD_OK;
  }
  kd::GemmTile t;
  double ns = 0;
  kd_status s = kd::gemm::csk::choose(sh, &t, &ns);
  if (s) return s;
  out[0] = 1;
  out[1] = t.split;
  out[2] = kd::gemm::kBM;
  out[3] = t.tiles;
  out[4] = t.stages;
  out[5] = (int32_t)t.smem;
  return KD_OK;
}

extern "C" kd_status kd_debug_gemm_trace(void* dev_buf) {  // 32 u64 stamps per CTA
  kd::g_gemm_trace = (unsigned long long*)dev_buf;
  return KD_OK;
}

extern "C" kd_status kd_debug_timeline(void* dev_buf, uint64_t bytes) {
  kd::g_tl = (unsigned long long*)dev_buf;
  kd::g_tl_cap = dev_buf ? bytes / (kd::kTlRegion * 8) : 0;
  kd::g_tl_kinds.clear();
  return KD_OK;
}

extern "C" kd_status kd_debug_timeline_kinds(int32_t* out, uint32_t cap, uint32_t* n) {
  if (!n) return kd::fail(KD_ERR_INVALID_ARG, "kd_debug_timeline_kinds: NULL n");
  *n = (uint32_t)kd::g_tl_kinds.size();
  if (out)
    for (uint32_t i = 0; i < *n && i < cap; ++i) out[i] = kd::g_tl_kinds[i];
  return KD_OK;
}

namespace kd {

kd_status gemm_signals(const GemmShape& a, uint32_t* s) {
  if (a.dtype == KD_F32) {
    *s = gemm_f32_signals(a.N);
    return KD_OK;
  }
  if (gemm_is_prefill(a)) {
    *s = gemm_prefill_signals(a);
    return KD_OK;
  }
  if (gemm::use_dense(a)) {
    // one release per storing CTA: every tile once (split 1), else every
    // cluster rank that owns weight rows
    GemmTile t;
    double ns = 0;
    kd_status st = gemm::csk::choose(a, &t, &ns);
    if (st) return st;
    const int owners = t.split == 1 ? 1 : (gemm::kBM + t.rpo - 1) / t.rpo;
    *s = (uint32_t)(t.tiles * owners);
    return KD_OK;
  }
  gemm::Geometry g;
  kd_status st = gemm::geometry(a, &g, gemm::device_sms());
  if (st) return st;
  // one flag increment per CTA, after its whole tiles and its fold slice
  *s = (uint32_t)g.grid;
  return KD_OK;
}

kd_status gemm_grid(const GemmShape& a, uint32_t* grid) {
  if (a.dtype == KD_F32) return fail(KD_ERR_UNSUPPORTED, "gemm_grid: bf16 only");
  if (gemm_is_prefill(a)) {
    *grid = gemm_prefill_signals(a);
    return KD_OK;
  }
  if (gemm::use_dense(a)) {
    GemmTile t;
    double ns = 0;
    kd_status st = gemm::csk::choose(a, &t, &ns);
    if (st) return st;
    *grid = (uint32_t)(t.tiles * t.split);
    return KD_OK;
  }
  gemm::Geometry g;
  kd_status st = gemm::geometry(a, &g, gemm::device_sms());
  if (st) return st;
  *grid = (uint32_t)g.grid;
  return KD_OK;
}

kd_status gemm_init_attrs() {
  for (auto f : {gemm::gemm_kernel<false>, gemm::gemm_kernel<true>}) {
    KD_CUDA_CHECK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024), "gemm smem attr");
    KD_CUDA_CHECK(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100), "gemm carveout");
  }
  for (auto f : {gemm::csk::gemm_csk_kernel<false>, gemm::csk::gemm_csk_kernel<true>}) {
    KD_CUDA_CHECK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, gemm::csk::kSmemMax),
                  "gemm dense smem attr");
    KD_CUDA_CHECK(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100), "gemm dense carveout");
  }
  return KD_OK;
}

kd_status attention_init_attrs();    // attention.cu
kd_status elementwise_init_attrs();  // elementwise.cu

kd_status kernels_init() {
  static std::mutex mu;
  static std::vector<int> done;
  int dev = 0;
  KD_CUDA_CHECK(cudaGetDevice(&dev), "cudaGetDevice");
  std::lock_guard<std::mutex> lk(mu);
  for (int d : done)
    if (d == dev) return KD_OK;
  kd_status s = gemm_init_attrs();
  if (s) return s;
  s = attention_init_attrs();
  if (s) return s;
  s = elementwise_init_attrs();
  if (s) return s;
  done.push_back(dev);
  return KD_OK;
}

}  // namespace kd
