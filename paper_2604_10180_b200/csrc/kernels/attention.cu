// attention.cu — paged GQA decode attention (C1.5).
//
// For sequence b, kv head g and the G = Hq/Hkv query heads sharing it:
//   s_t = q_h·k_t/√D (t < seq_len[b]); p = softmax(s); out_h = Σ_t p_t v_t.
//
// B200 design (HBM-bound: 4 FLOP/B at G=4, 8 at G=8):
//  * persistent, warp-specialised CTAs (2 per SM) with dynamically fetched
//    work items (sequence, kv head, split); each item streams the KV pages of
//    its split exactly once for all G heads (GQA reuse).
//  * HND cache [page][Hkv][16][D]: one page's K (or V) slab for one kv head is
//    a 16 × D tile → TMA tensor copies (box 16 tokens × 64 dims, 128-byte
//    swizzle) into an S-stage mbarrier ring; stage s always feeds consumer
//    warp s % 4.
//  * tokens are the MMA rows: Sᵀ = K·Qᵀ (m16 tokens × n8 heads × k16 dims)
//    and Oᵀ = Vᵀ·Pᵀ (m16 dims × n8 heads × k16 tokens) with mma.sync
//    m16n8k16 bf16 → fp32 — 2·D/16 MMAs per page, no padding rows for G ≥ 8.
//    K and Vᵀ fragments come from ldmatrix (.trans for V) on the swizzled
//    tiles (conflict-free); Pᵀ goes from the C to the B fragment layout with
//    two movmatrix.trans; Qᵀ is register-resident per item.
//  * online softmax in fp32 with exp2; per-warp states merged in fixed warp
//    order by an epilogue warp; splits merged in fixed split order by whichever
//    item of the (b, g) unit finishes last → bitwise deterministic.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "launch.hpp"
#include "mmasync.cuh"

namespace kd {
namespace attn {
using mmas::tma_3d;
using mmas::ldsm_x4;
using mmas::ldsm_x4_t;
using mmas::movm_t;
using mmas::mma16816;
using mmas::tile_off;

constexpr int kWarps = 4;           // consumer warps
constexpr int kThreads = (kWarps + 2) * 32;  // + producer + epilogue warp
// Page j lives in stage j % S and is consumed by warp j % kWarps. With
// S % kWarps == 0 every stage is always consumed by the SAME warp, in round
// order, so no waiter can run two mbarrier phases ahead (parity waits alias
// after two phases).
constexpr int kPage = 16;
constexpr int kMaxG = 8;
constexpr int kMaxPagesPerSplit = 512;
// split merge fast path (all of a unit's partial loads in one batch) when
// splits·G ≤ this and splits ≤ kFastSplits
constexpr int kFastSplitLse = 128, kFastSplits = 4;

struct Params {
  const __nv_bfloat16* q;
  const __nv_bfloat16* kc;
  const __nv_bfloat16* vc;
  const int32_t* bt;
  const int32_t* sl;
  __nv_bfloat16* out;
  float* lse;         // KD_ATTN_LSE: [rows][Hq] base-2 LSE after the [rows][Hq][D] bf16 out (nullable)
  size_t lse_off;     // byte offset of lse inside the output buffer (for the peer copies)
  float* part_o;      // [rows][Hkv][splits][G][D]
  float* part_lse;    // [rows][Hkv][splits][G]
  unsigned* counter;  // [rows][Hkv]
  unsigned* work;     // item ticket counter (last word of the counter region)
  unsigned long long* tl;    // kd_debug_timeline region (nullable): per CTA [0] entry, [1] producer past
                             // its dependency wait, [2] producer done, [3] epilogue done, [4] consumers done,
                             // [5..8] epilogue slot acquired / done of its last two items, [9] last split atomic
  unsigned long long* prof;  // KD_ATTN_PROF experiments: [0] producer empty-wait cycles, [1] consumer full-wait, [2] consumer busy, [3] pages
  int Hq, Hkv, G, pps, splits, pages_per_split;
  int rows;           // sequences; items are kv-head-major: it = (g·rows + b)·splits + split
  int prefetch;       // stream the first item's safe pages before griddepcontrol.wait (KD_ATTN_PREFETCH=0 disables)
  int l2pf;           // pages of the first item past the smem ring the idle epilogue warp warms L2 with (KD_ATTN_L2PF)
  float scale_log2;   // log2(e)/sqrt(D)
  Epi epi;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void st_f4_keep(float* p, float4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void st_f1_keep(float* p, float v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}
// L2 load issued at this point of the program (asm volatile: the compiler
// cannot sink it to the first use, so a batch of them is in flight together)
__device__ __forceinline__ float4 ldcg_f4_now(const float* p) {
  float4 v;
  asm volatile("ld.global.cg.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
// L2 prefetch of one 3-D K/V slab box (no shared memory, no completion)
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global [%0, {%1, %2, %3}];" ::"l"((uint64_t)map), "r"(c0), "r"(c1),
               "r"(c2)
               : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_gpu_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

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

__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// 4 consecutive output dims as bf16 (8-byte store), mirrored to the peers.
__device__ __forceinline__ void store_out4(const Params& P, size_t oi, float4 v) {
  uint2 pk;
  pk.x = pack_bf16(v.x, v.y);
  pk.y = pack_bf16(v.z, v.w);
  *reinterpret_cast<uint2*>(P.out + oi) = pk;
  for (int pp = 0; pp < P.epi.n; ++pp) *reinterpret_cast<uint2*>((__nv_bfloat16*)P.epi.dst[pp] + oi) = pk;
}

// one (row, head) base-2 LSE of a KD_ATTN_LSE partial, mirrored to the peers
__device__ __forceinline__ void store_lse(const Params& P, size_t li, float v) {
  P.lse[li] = v;
  for (int pp = 0; pp < P.epi.n; ++pp) reinterpret_cast<float*>((uint8_t*)P.epi.dst[pp] + P.lse_off)[li] = v;
}

// Persistent, warp-specialised, dynamically scheduled: the producer takes
// item tickets from a global counter (item = (sequence, kv head, split),
// split fastest) and publishes them to the other warps through a 4-slot smem
// ring, so SMs that get more HBM bandwidth simply process more items. Which
// CTA processes an item never changes the result: split bounds and every
// merge order are fixed (bitwise deterministic). The CTA drawing the very
// last ticket (n_items + gridDim.x − 1: every CTA draws exactly one failing
// ticket) resets the counter for the next launch.
//  * producer warp (lane 0 issues): per item a bulk copy of its G query rows
//    into a 2-slot Q ring, then the K/V tiles of all its items back to back
//    through one S-stage ring (block-table ids fetched one 32-page chunk
//    ahead, lanes in parallel). CTA-global page counter gj: stage gj % S,
//    consumer warp gj % kWarps.
//  * 4 consumer warps: online softmax over their pages; per-warp (O, m, l) to
//    a double-buffered combine slot; straight on to the next item.
//  * epilogue warp: merges the 4 warp states (fixed order), writes the output
//    (1 split) or the split partial + counter; the last-arriving split merges
//    all splits (fixed order) and signals the consumers of this unit.
template <int D, int S>
__global__ void __launch_bounds__(kThreads) decode_attention_kernel(const __grid_constant__ CUtensorMap tk,
                                                                    const __grid_constant__ CUtensorMap tv, Params P,
                                                                    int n_items) {
  static_assert(S % kWarps == 0, "each stage must belong to one consumer warp");
  static_assert(D % 64 == 0, "head_dim must be a multiple of 64");
  constexpr int KS = D / 16;          // k-steps of Sᵀ = K·Qᵀ, m-blocks of Oᵀ = Vᵀ·Pᵀ
  constexpr int SLAB = kPage * D;     // elements per page slab
  constexpr int SLAB_B = SLAB * 2;    // bytes
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // swizzle atoms: 1024-B aligned
  const int G = P.G, Hkv = P.Hkv;
  uint8_t* ks = smem;                                                   // [S] K tiles
  uint8_t* vs = ks + S * SLAB_B;                                        // [S] V tiles
  __nv_bfloat16* qsm = reinterpret_cast<__nv_bfloat16*>(vs + S * SLAB_B);  // [2][G][D]
  float* comb = reinterpret_cast<float*>(qsm + 2 * G * D);                // [2][kWarps][G][D]
  float* comb_ml = comb + 2 * kWarps * G * D;                             // [2][kWarps][G][2]
  uint64_t* full = reinterpret_cast<uint64_t*>(comb_ml + 2 * kWarps * G * 2);
  uint64_t* empty = full + S;
  uint64_t* qfull = empty + S;   // [2]
  uint64_t* qempty = qfull + 2;  // [2]
  uint64_t* cfull = qempty + 2;  // [2]
  uint64_t* cempty = cfull + 2;  // [2]
  uint64_t* ifull = cempty + 2;  // [4] item ring
  uint64_t* iempty = ifull + 4;  // [4]
  __shared__ int s_item[4];
  __shared__ float s_w[kWarps * kMaxG], s_M[kMaxG], s_L[kMaxG];  // epilogue merge weights
  __shared__ float s_lse[kFastSplitLse];                           // split merge: every (split, head) LSE

  pdl_launch_dependents();
  epi_started(P.epi);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto tl_stamp = [&](int slot) {
    unsigned long long gt;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(gt));
    atomicMax(&P.tl[blockIdx.x * 32 + slot], gt);
  };
  if (P.tl && threadIdx.x == 0) tl_stamp(0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&qfull[s], 1);
      mbar_init(&qempty[s], kWarps);
      mbar_init(&cfull[s], kWarps);
      mbar_init(&cempty[s], 1);
    }
    for (int s = 0; s < 4; ++s) {
      mbar_init(&ifull[s], 1);
      mbar_init(&iempty[s], kWarps + 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // every warp but the producer waits for the previous grid here; the
  // producer first streams the K/V pages of its statically assigned first
  // item that the previous kernels cannot be writing (see the producer)
  if (warp != kWarps) pdl_wait();
  const bool single = (P.splits == 1);
  auto next_item = [&](int k) -> int {  // consumer / epilogue side of the item ring
    const int is = k & 3;
    mbar_wait(&ifull[is], (k >> 2) & 1);
    const int it = s_item[is];
    __syncwarp();
    if (lane == 0) mbar_arrive(&iempty[is]);
    return it;
  };

  if (warp == kWarps) {
    // ================= producer
    auto ids_of = [&](int it, int j0) -> int {  // this lane's page id of chunk j0 of item it
      if (it < 0) return 0;
      const int split = it % P.splits, b = (it / P.splits) % P.rows;
      const int j = j0 + lane, pg = split * P.pages_per_split + j;
      return (j < P.pages_per_split && pg < P.pps) ? __ldg(P.bt + (size_t)b * P.pps + pg) : 0;
    };
    // CTA c's first item is c (static); tickets t ≥ 0 hand out items
    // gridDim.x + t. Every CTA draws exactly one failing ticket, so the last
    // ticket value is max(0, n_items − grid) + grid − 1: its drawer resets the
    // counter for the next launch.
    const unsigned n_dyn = n_items > (int)gridDim.x ? (unsigned)(n_items - (int)gridDim.x) : 0u;
    auto fetch = [&]() -> int {
      unsigned t = 0;
      if (lane == 0) {
        t = atomicAdd(P.work, 1u);
        if (t == n_dyn + gridDim.x - 1) atomicExch(P.work, 0u);  // last ticket: reset
      }
      t = __shfl_sync(0xffffffffu, t, 0);
      return t < n_dyn ? (int)(gridDim.x + t) : -1;
    };
    uint64_t pol = 0;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    uint32_t gj = 0;
    long long pw = 0, p_item = 0, p_issue = 0;
    const long long p_start = P.prof ? clock64() : 0;
    unsigned long long p_gt0 = 0;
    if (P.prof) asm volatile("mov.u64 %0, %globaltimer;" : "=l"(p_gt0));
    // ---- before the grid-dependency wait: the first item (static) and its
    // first min(S, pages) K/V slabs, all strictly before the page holding
    // position len−1 — the only page of a sequence this step's RoPE/append
    // writes. The block table and lengths are step inputs (not written by
    // the previous kernels). The ticket counter is only touched after the wait.
    const int it0 = (int)blockIdx.x < n_items ? (int)blockIdx.x : -2;  // −2: draw after the wait
    int n_pre = 0;
    int mine = ids_of(it0 < 0 ? -1 : it0, 0);
    if (it0 >= 0 && P.prefetch) {
      const int split = it0 % P.splits, unit = it0 / P.splits;
      const int g = unit / P.rows, b = unit % P.rows;
      const int len = __ldg(P.sl + b);
      const int p0 = split * P.pages_per_split;
      const int np = max(0, min((len + kPage - 1) / kPage, p0 + P.pages_per_split) - p0);
      const int safe = max(0, min(np, (len - 1) / kPage - p0));  // pages before the appended one
      n_pre = min(min(S, 32), safe);
      for (int t = 0; t < n_pre; ++t) {
        const int pid = __shfl_sync(0xffffffffu, mine, t);
        if (lane == 0) {
          const int row = (pid * Hkv + g) * kPage;
          mbar_expect_tx(&full[t], 2u * SLAB_B);
          tma_3d(ks + t * SLAB_B, &tk, 0, 0, row, &full[t], pol);
          tma_3d(vs + t * SLAB_B, &tv, 0, 0, row, &full[t], pol);
        }
      }
      gj = (uint32_t)n_pre;
    }
    pdl_wait();
    if (P.tl && lane == 0) tl_stamp(1);
    int it = it0 == -2 ? fetch() : it0;
    if (it0 == -2) mine = ids_of(it, 0);
    for (int k = 0;; ++k) {
      if (lane == 0) {  // publish the item (or the end marker -1)
        const int is = k & 3;
        if (k >= 4) mbar_wait(&iempty[is], ((k >> 2) - 1) & 1);
        s_item[is] = it;
        mbar_arrive(&ifull[is]);
      }
      if (it < 0) break;
      const long long ti0 = P.prof ? clock64() : 0;
      const int it_next = fetch();
      const int split = it % P.splits, unit = it / P.splits;
      const int g = unit / P.rows, b = unit % P.rows;
      const int len = P.sl[b];
      const int p0 = split * P.pages_per_split;
      const int np = max(0, min((len + kPage - 1) / kPage, p0 + P.pages_per_split) - p0);
      if (P.prof) p_item += clock64() - ti0;
      if (lane == 0) {
        const int qs = k & 1;
        if (k >= 2) mbar_wait(&qempty[qs], ((k >> 1) - 1) & 1);
        mbar_expect_tx(&qfull[qs], (unsigned)(G * D * 2));
        bulk_g2s(qsm + qs * G * D, P.q + (size_t)b * P.Hq * D + (size_t)g * G * D, (unsigned)(G * D * 2), &qfull[qs]);
      }
      for (int j0 = 0;; j0 += 32) {
        const bool more = j0 + 32 < np;
        const int nxt = more ? ids_of(it, j0 + 32) : ids_of(it_next, 0);
        const int cnt = min(32, np - j0);
        for (int t = (k == 0 && j0 == 0) ? n_pre : 0; t < cnt; ++t, ++gj) {  // slabs already in flight skipped
          const int pid = __shfl_sync(0xffffffffu, mine, t);
          const long long tq = P.prof ? clock64() : 0;
          if (lane == 0) {
            const uint32_t st = gj % S, round = gj / S;
            if (round > 0) {
              const long long t0 = P.prof ? clock64() : 0;
              mbar_wait(&empty[st], (round - 1) & 1);
              if (P.prof) pw += clock64() - t0;
            }
            const int row = (pid * Hkv + g) * kPage;
            mbar_expect_tx(&full[st], 2u * SLAB_B);
            tma_3d(ks + st * SLAB_B, &tk, 0, 0, row, &full[st], pol);
            tma_3d(vs + st * SLAB_B, &tv, 0, 0, row, &full[st], pol);
            if (P.prof) p_issue += clock64() - tq;
          }
        }
        mine = nxt;
        if (!more) break;
      }
      it = it_next;
    }
    if (P.tl && lane == 0) tl_stamp(2);
    if (P.prof && lane == 0) {
      unsigned long long gt;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(gt));
      atomicAdd(&P.prof[7], gt - p_gt0);  // producer lifetime, ns
      unsigned smid;
      asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
      P.prof[8 + blockIdx.x * 5 + 0] = smid;
      P.prof[8 + blockIdx.x * 5 + 1] = p_gt0;
      P.prof[8 + blockIdx.x * 5 + 2] = gt;
      atomicAdd(&P.prof[0], (unsigned long long)pw);
      atomicAdd(&P.prof[4], (unsigned long long)(clock64() - p_start));
      atomicAdd(&P.prof[5], (unsigned long long)p_item);
      atomicAdd(&P.prof[6], (unsigned long long)p_issue);
    }
    return;
  }

  if (warp == kWarps + 1) {
    // ================= epilogue: merge warps (fixed order), then splits (fixed order)
    // Idle until the first item's pages are consumed: warm L2 with that
    // item's pages past the producer's smem prefill (step inputs and earlier
    // steps' cache only — the appended page is excluded), so a CTA resident
    // before its dependency resolves (on SMs the previous kernel leaves free)
    // turns its wait into HBM traffic the first item then finds in L2
    if (P.l2pf > 0 && (int)blockIdx.x < n_items) {
      const int it0 = (int)blockIdx.x, split = it0 % P.splits, unit = it0 / P.splits;
      const int g = unit / P.rows, b = unit % P.rows;
      const int len = __ldg(P.sl + b);
      const int p0 = split * P.pages_per_split;
      const int np = max(0, min((len + kPage - 1) / kPage, p0 + P.pages_per_split) - p0);
      const int safe = max(0, min(np, (len - 1) / kPage - p0));
      const int t0 = P.prefetch ? min(min(S, 32), safe) : 0, t1 = min(safe, t0 + P.l2pf);
      for (int t = t0 + lane; t < t1; t += 32) {
        const int pid = __ldg(P.bt + (size_t)b * P.pps + p0 + t);
        const int row = (pid * Hkv + g) * kPage;
        tma_prefetch_3d(&tk, 0, 0, row);
        tma_prefetch_3d(&tv, 0, 0, row);
      }
    }
    // timeline (P.tl): combine slot acquired / item done of the last two items, last split atomic
    unsigned long long e_c[2] = {0, 0}, e_d[2] = {0, 0}, e_a = 0;
    uint64_t pkeep = 0;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pkeep));
    auto gnow = [] {
      unsigned long long t;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      return t;
    };
    for (int k = 0;; ++k) {
      if (P.tl && k > 0) e_d[1] = gnow();
      const int it = next_item(k);
      if (it < 0) break;
      const int split = it % P.splits, unit = it / P.splits;
      const int g = unit / P.rows, b = unit % P.rows;
      const int cs = k & 1;
      mbar_wait(&cfull[cs], (k >> 1) & 1);
      if (P.tl) e_c[0] = e_c[1], e_d[0] = e_d[1], e_c[1] = gnow();
      const float* cb = comb + (size_t)cs * kWarps * G * D;
      const float* cml = comb_ml + cs * kWarps * G * 2;
      // per-head warp weights: lane (w, h) → s_w[w][h] = 2^(m_w − M_h); s_M, s_L
      if (lane < kWarps * G) {
        const int w = lane / G, h = lane % G;
        float M = -INFINITY;
#pragma unroll
        for (int x = 0; x < kWarps; ++x) M = fmaxf(M, cml[(x * G + h) * 2]);
        const float Mu = (M == -INFINITY) ? 0.f : M;
        float L = 0.f;
#pragma unroll
        for (int x = 0; x < kWarps; ++x) L += exp2f(cml[(x * G + h) * 2] - Mu) * cml[(x * G + h) * 2 + 1];
        s_w[w * kMaxG + h] = exp2f(cml[(w * G + h) * 2] - Mu);
        if (w == 0) s_M[h] = M, s_L[h] = L;
      }
      __syncwarp();
      for (int e4 = lane; e4 < G * D / 4; e4 += 32) {
        const int h = (e4 * 4) / D, d0 = (e4 * 4) % D;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
          const float sc = s_w[w * kMaxG + h];
          const float4 v = *reinterpret_cast<const float4*>(cb + ((size_t)w * G + h) * D + d0);
          acc.x += sc * v.x, acc.y += sc * v.y, acc.z += sc * v.z, acc.w += sc * v.w;
        }
        const float L = s_L[h];
        const float inv = L > 0.f ? 1.f / L : 0.f;
        acc.x *= inv, acc.y *= inv, acc.z *= inv, acc.w *= inv;
        if (single) {
          store_out4(P, (size_t)b * P.Hq * D + (size_t)(g * G + h) * D + d0, acc);
          if (P.lse && d0 == 0) store_lse(P, (size_t)b * P.Hq + g * G + h, L > 0.f ? s_M[h] + log2f(L) : -INFINITY);
        } else {
          const size_t pi = (((size_t)unit * P.splits + split) * G + h);
          // evict_last: the unit's last split merges these up to a whole
          // launch later, after ~1 GB of KV pages streamed through L2
          st_f4_keep(P.part_o + pi * D + d0, acc, pkeep);
          if (d0 == 0) st_f1_keep(P.part_lse + pi, L > 0.f ? s_M[h] + log2f(L) : -INFINITY, pkeep);
        }
      }
      // every lane fences its own partial stores at gpu scope before lane 0's
      // release-add publishes them (PTX memory model: a bar.warp.sync is not a
      // documented morally-strong barrier, so cumulativity through it is not
      // relied on)
      if (!single) __threadfence();
      __syncwarp();
      if (lane == 0) mbar_arrive(&cempty[cs]);
      bool done = true;
      if (!single) {
        unsigned prev = 0;
        // the acq_rel add releases this warp's (fenced) partial and acquires
        // the other splits' partials for the last arriver
        if (lane == 0) prev = atom_add_acq_rel_gpu(&P.counter[unit], 1u);
        done = __shfl_sync(0xffffffffu, prev, 0) == (unsigned)P.splits - 1;
        if (P.tl) e_a = gnow();
        if (done) {
          __syncwarp();
          // each lane acquires the counter itself until it reads every split's
          // arrival (lane 0's add above made it P.splits), so its partial loads
          // below are ordered after all splits' releases (one L2 round trip;
          // was a fence.acq_rel.gpu after the warp sync, ≈1.7 µs at the tail)
          // (lane 0's add already made the count P.splits: the first read
          // normally succeeds; the bound only guards against a broken invariant)
          for (int spins = 0; ld_acquire_gpu_u32(&P.counter[unit]) < (unsigned)P.splits && spins < (1 << 20); ++spins) {
          }
          const float* lse = P.part_lse + (size_t)unit * P.splits * G;  // [split][G]
          const float* po = P.part_o + (size_t)unit * P.splits * G * D;  // [split][G][D]
          const int nl = P.splits * G, n_e4 = G * D / 4;
          if (nl <= kFastSplitLse && P.splits <= kFastSplits && n_e4 <= 32 * 4) {
            // fast path: every partial this lane combines and every LSE in one
            // batch, then per head max / normaliser in split order from shared
            // memory (a dependent L2 round trip costs ~1 µs here, and the last
            // units' merges are the kernel's tail)
            float4 v[4][kFastSplits];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int e4 = lane + 32 * k, h = (e4 * 4) / D, d0 = (e4 * 4) % D;
#pragma unroll
              for (int sp = 0; sp < kFastSplits; ++sp)
                if (e4 < n_e4 && sp < P.splits)
                  v[k][sp] = ldcg_f4_now(po + ((size_t)sp * G + h) * D + d0);
            }
            for (int i = lane; i < nl; i += 32) s_lse[i] = __ldcg(lse + i);  // (both batches in flight)
            __syncwarp();
            if (lane < G) {
              float M = -INFINITY;
              for (int sp = 0; sp < P.splits; ++sp) M = fmaxf(M, s_lse[sp * G + lane]);
              const float Mu = (M == -INFINITY) ? 0.f : M;
              float L = 0.f;
              for (int sp = 0; sp < P.splits; ++sp) L += exp2f(s_lse[sp * G + lane] - Mu);
              s_M[lane] = Mu, s_L[lane] = L;
            }
            __syncwarp();
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int e4 = lane + 32 * k, h = (e4 * 4) / D, d0 = (e4 * 4) % D;
              if (e4 >= n_e4) continue;
              const float Mu = s_M[h];
              float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
              for (int sp = 0; sp < kFastSplits; ++sp)
                if (sp < P.splits) {
                  const float sc = exp2f(s_lse[sp * G + h] - Mu);
                  acc.x += sc * v[k][sp].x, acc.y += sc * v[k][sp].y, acc.z += sc * v[k][sp].z, acc.w += sc * v[k][sp].w;
                }
              const float L = s_L[h];
              const float inv = L > 0.f ? 1.f / L : 0.f;
              acc.x *= inv, acc.y *= inv, acc.z *= inv, acc.w *= inv;
              store_out4(P, (size_t)b * P.Hq * D + (size_t)(g * G + h) * D + d0, acc);
              if (P.lse && d0 == 0) store_lse(P, (size_t)b * P.Hq + g * G + h, L > 0.f ? Mu + log2f(L) : -INFINITY);
            }
          } else {
            // per-head max / normaliser over the splits (lanes over splits)
            for (int h = 0; h < G; ++h) {
              float M = -INFINITY;
              for (int sp = lane; sp < P.splits; sp += 32) M = fmaxf(M, __ldcg(lse + sp * G + h));
  #pragma unroll
              for (int x = 16; x; x >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, x));
              const float Mu = (M == -INFINITY) ? 0.f : M;
              float L = 0.f;
              for (int sp = lane; sp < P.splits; sp += 32) L += exp2f(__ldcg(lse + sp * G + h) - Mu);
  #pragma unroll
              for (int x = 16; x; x >>= 1) L += __shfl_xor_sync(0xffffffffu, L, x);
              if (lane == 0) s_M[h] = Mu, s_L[h] = L;
            }
            __syncwarp();
            for (int e4 = lane; e4 < G * D / 4; e4 += 32) {
              const int h = (e4 * 4) / D, d0 = (e4 * 4) % D;
              const float Mu = s_M[h];
              float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
              int sp = 0;
              for (; sp + 4 <= P.splits; sp += 4) {  // 4 independent L2 round trips in flight
                float wv[4];
                float4 v[4];
  #pragma unroll
                for (int u = 0; u < 4; ++u) {
                  wv[u] = __ldcg(lse + (sp + u) * G + h);
                  v[u] = __ldcg(reinterpret_cast<const float4*>(po + ((size_t)(sp + u) * G + h) * D + d0));
                }
  #pragma unroll
                for (int u = 0; u < 4; ++u) {
                  const float sc = exp2f(wv[u] - Mu);
                  acc.x += sc * v[u].x, acc.y += sc * v[u].y, acc.z += sc * v[u].z, acc.w += sc * v[u].w;
                }
              }
              for (; sp < P.splits; ++sp) {
                const float sc = exp2f(__ldcg(lse + sp * G + h) - Mu);
                const float4 v = __ldcg(reinterpret_cast<const float4*>(po + ((size_t)sp * G + h) * D + d0));
                acc.x += sc * v.x, acc.y += sc * v.y, acc.z += sc * v.z, acc.w += sc * v.w;
              }
              const float L = s_L[h];
              const float inv = L > 0.f ? 1.f / L : 0.f;
              acc.x *= inv, acc.y *= inv, acc.z *= inv, acc.w *= inv;
              store_out4(P, (size_t)b * P.Hq * D + (size_t)(g * G + h) * D + d0, acc);
              if (P.lse && d0 == 0) store_lse(P, (size_t)b * P.Hq + g * G + h, L > 0.f ? Mu + log2f(L) : -INFINITY);
            }
          }
          if (lane == 0) P.counter[unit] = 0u;  // ready for the next launch
        }
      }
      if (done && P.epi.n) {
        // every lane fences its own peer stores at system scope, then lane 0
        // releases: COUNT mode → the unit's G·D output columns of row b go to
        // the chunk(s) they fall in (units are drawn kv-head-major, so the
        // low-column chunks complete first and the consumer starts on them
        // while later kv heads are still computed); CTA mode → one increment
        fence_acq_rel_sys();
        __syncwarp();
        if (lane == 0) {
          if (P.epi.nch)
            epi_release_range(P.epi, (uint32_t)(g * G * D) * 2u, (uint32_t)((g + 1) * G * D) * 2u, (uint32_t)b,
                              (uint32_t)b + 1u);
          else
            epi_release_cta(P.epi);
        }
      }
    }
    if (P.tl && lane == 0) {
      tl_stamp(3);
      P.tl[blockIdx.x * 32 + 5] = e_c[0];
      P.tl[blockIdx.x * 32 + 6] = e_d[0];
      P.tl[blockIdx.x * 32 + 7] = e_c[1];
      P.tl[blockIdx.x * 32 + 8] = e_d[1];
      P.tl[blockIdx.x * 32 + 9] = e_a;
    }
    if (P.prof && lane == 0) {
      unsigned long long gt;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(gt));
      P.prof[8 + blockIdx.x * 5 + 4] = gt;
    }
    return;
  }

  // ================= consumers
  const int gid = lane >> 2, c = lane & 3;
  // ldmatrix row addresses of this lane (matrix mi = lane/8, row r = lane%8):
  //  K (A of Sᵀ = K·Qᵀ, non-trans): token (mi&1)*8 + r, chunk +(mi>>1)
  //  V (A of Oᵀ = Vᵀ·Pᵀ, trans):    token (mi>>1)*8 + r, chunk +(mi&1)
  const int mi = lane >> 3, r8 = lane & 7;
  const int k_tok = ((mi & 1) << 3) + r8, k_dc = mi >> 1;
  const int v_tok = ((mi >> 1) << 3) + r8, v_dc = mi & 1;
  const uint32_t ks_u = smem_u32(ks), vs_u = smem_u32(vs);
  uint32_t gbase = 0;
  long long fw = 0, busy = 0, npg = 0;
  for (int k = 0;; ++k) {
    const int it = next_item(k);
    if (it < 0) break;
    const int split = it % P.splits, b = (it / P.splits) % P.rows;
    const int len = P.sl[b];
    const int p0 = split * P.pages_per_split;
    const int np = max(0, min((len + kPage - 1) / kPage, p0 + P.pages_per_split) - p0);
    // Qᵀ as the B operand: qb[ks] = {Q[gid][16ks+2c..], Q[gid][16ks+8+2c..]}; heads ≥ G are zero
    uint32_t qb[KS][2];
    {
      const int qs = k & 1;
      mbar_wait(&qfull[qs], (k >> 1) & 1);
      const uint32_t* qh = reinterpret_cast<const uint32_t*>(qsm + qs * G * D + gid * D);
#pragma unroll
      for (int s = 0; s < KS; ++s) {
        qb[s][0] = gid < G ? qh[8 * s + c] : 0u;
        qb[s][1] = gid < G ? qh[8 * s + 4 + c] : 0u;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&qempty[qs]);
    }
    // Oᵀ accumulators: o[mb] = {(dim 16mb+gid, head 2c), (.., 2c+1), (dim 16mb+gid+8, 2c), (.., 2c+1)}
    float o[KS][4];
#pragma unroll
    for (int j = 0; j < KS; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
    float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};  // heads 2c, 2c+1 (l: this lane's tokens)

    for (int j = (int)((warp - gbase % kWarps + kWarps) % kWarps); j < np; j += kWarps) {
      const uint32_t gj = gbase + j;
      const int st = gj % S;
      const long long t0 = P.prof ? clock64() : 0;
      mbar_wait(&full[st], (gj / S) & 1);
      const long long t1 = P.prof ? clock64() : 0;
      if (P.prof) fw += t1 - t0;
      const uint32_t kt = ks_u + st * SLAB_B, vt = vs_u + st * SLAB_B;
      const int tok0 = (p0 + j) * kPage;
      const int valid = min(kPage, len - tok0);
      if (valid < kPage) {  // zero the V rows past the end (0·garbage must not be NaN)
        uint4* vrow = reinterpret_cast<uint4*>(vs + st * SLAB_B + valid * D * 2);  // token rows are contiguous
        for (int e = lane; e < (kPage - valid) * D / 8; e += 32) vrow[e] = make_uint4(0, 0, 0, 0);
        __syncwarp();
      }
      // ---- Sᵀ = K Qᵀ : 16 tokens × 8 heads, two accumulation chains
      float sa[4] = {0.f, 0.f, 0.f, 0.f}, sb[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int s = 0; s < KS; ++s) {
        uint32_t a0, a1, a2, a3;
        ldsm_x4(kt + tile_off<D>(s >> 2, k_tok, ((s & 3) << 1) + k_dc), a0, a1, a2, a3);
        if (s & 1)
          mma16816(sb, a0, a1, a2, a3, qb[s][0], qb[s][1]);
        else
          mma16816(sa, a0, a1, a2, a3, qb[s][0], qb[s][1]);
      }
      // lane holds tokens gid, gid+8 × heads 2c, 2c+1
      float sv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) sv[i] = (sa[i] + sb[i]) * P.scale_log2;
      if (gid >= valid) sv[0] = sv[1] = -INFINITY;
      if (gid + 8 >= valid) sv[2] = sv[3] = -INFINITY;
      float mx0 = fmaxf(sv[0], sv[2]), mx1 = fmaxf(sv[1], sv[3]);
#pragma unroll
      for (int x = 4; x < 32; x <<= 1) {
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, x));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, x));
      }
      const float mn0 = fmaxf(m_run[0], mx0), mn1 = fmaxf(m_run[1], mx1);
      const float mu0 = (mn0 == -INFINITY) ? 0.f : mn0, mu1 = (mn1 == -INFINITY) ? 0.f : mn1;
      const float al0 = exp2f(m_run[0] - mu0), al1 = exp2f(m_run[1] - mu1);
      const float p0v = exp2f(sv[0] - mu0), p1v = exp2f(sv[1] - mu1);
      const float p2v = exp2f(sv[2] - mu0), p3v = exp2f(sv[3] - mu1);
      l_run[0] = l_run[0] * al0 + (p0v + p2v);
      l_run[1] = l_run[1] * al1 + (p1v + p3v);
      m_run[0] = mn0;
      m_run[1] = mn1;
#pragma unroll
      for (int mb = 0; mb < KS; ++mb) {
        o[mb][0] *= al0;
        o[mb][1] *= al1;
        o[mb][2] *= al0;
        o[mb][3] *= al1;
      }
      // Pᵀ as the B operand (k = tokens, n = heads): transpose the C fragment
      const uint32_t pb0 = movm_t(pack_bf16(p0v, p1v));  // tokens 0..7
      const uint32_t pb1 = movm_t(pack_bf16(p2v, p3v));  // tokens 8..15
      // ---- Oᵀ += Vᵀ Pᵀ : per 16-dim block
#pragma unroll
      for (int mb = 0; mb < KS; ++mb) {
        uint32_t a0, a1, a2, a3;
        ldsm_x4_t(vt + tile_off<D>(mb >> 2, v_tok, ((mb & 3) << 1) + v_dc), a0, a1, a2, a3);
        mma16816(o[mb], a0, a1, a2, a3, pb0, pb1);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      if (P.prof) busy += clock64() - t1, ++npg;
    }
    gbase += np;
    // per-warp state → combine slot (unnormalised O, m, l) for the epilogue warp
#pragma unroll
    for (int x = 4; x < 32; x <<= 1) {
      l_run[0] += __shfl_xor_sync(0xffffffffu, l_run[0], x);
      l_run[1] += __shfl_xor_sync(0xffffffffu, l_run[1], x);
    }
    const int cs = k & 1;
    if (k >= 2) mbar_wait(&cempty[cs], ((k >> 1) - 1) & 1);
    float* cw = comb + ((size_t)cs * kWarps + warp) * G * D;
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int h = 2 * c + hh;
      if (h < G) {
#pragma unroll
        for (int mb = 0; mb < KS; ++mb) {
          cw[h * D + 16 * mb + gid] = o[mb][hh];
          cw[h * D + 16 * mb + gid + 8] = o[mb][2 + hh];
        }
        if (gid == 0) {
          comb_ml[((cs * kWarps + warp) * G + h) * 2 + 0] = m_run[hh];
          comb_ml[((cs * kWarps + warp) * G + h) * 2 + 1] = l_run[hh];
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&cfull[cs]);
  }
  if (P.tl && lane == 0) tl_stamp(4);
  if (P.prof && lane == 0) {
    unsigned long long gt;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(gt));
    atomicMax(&P.prof[8 + blockIdx.x * 5 + 3], gt);
    atomicAdd(&P.prof[1], (unsigned long long)fw);
    atomicAdd(&P.prof[2], (unsigned long long)busy);
    atomicAdd(&P.prof[3], (unsigned long long)npg);
  }
}

template <int D, int S>
size_t smem_bytes(int G) {
  return 1024 + (size_t)2 * S * kPage * D * 2 + (size_t)2 * G * D * 2 + (size_t)2 * kWarps * G * D * 4 +
         2 * kWarps * G * 2 * 4 + (2 * S + 16) * 8;
}

using KernelFn = void (*)(CUtensorMap, CUtensorMap, Params, int);
struct Variant {
  int D, S;
  KernelFn fn;
  size_t (*smem)(int);
};
static Variant g_variants[] = {
    {128, 8, decode_attention_kernel<128, 8>, smem_bytes<128, 8>},
    {128, 12, decode_attention_kernel<128, 12>, smem_bytes<128, 12>},
    {128, 16, decode_attention_kernel<128, 16>, smem_bytes<128, 16>},
    {64, 8, decode_attention_kernel<64, 8>, smem_bytes<64, 8>},
    {64, 16, decode_attention_kernel<64, 16>, smem_bytes<64, 16>},
};
static int occupancy(const Variant& v, int G) {
  int n = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, v.fn, kThreads, v.smem(G));
  if (e != cudaSuccess) {
    if (getenv("KD_ATTN_DEBUG")) fprintf(stderr, "attention occupancy S=%d: %s\n", v.S, cudaGetErrorString(e));
    (void)cudaGetLastError();
    return 0;
  }
  return n;
}

// Stage count: the deepest ring that still keeps 2 CTAs resident per SM at
// this G (2·S·4·D bytes of KV in flight per SM); KD_ATTN_STAGES caps it
// (experiments). Returns the variant and its residency.
static const Variant& pick(int D, int G, int* ctas_per_sm) {
  static int cap = [] {
    const char* e = getenv("KD_ATTN_STAGES");
    return e ? atoi(e) : 64;
  }();
  const Variant* best = nullptr;
  int best_occ = 0;
  for (const Variant& v : g_variants) {
    if (v.D != D || v.S > cap) continue;
    const int occ = occupancy(v, G);
    if (occ < 1) continue;
    const bool better = !best || (std::min(occ, 2) > std::min(best_occ, 2)) ||
                        (std::min(occ, 2) == std::min(best_occ, 2) && v.S > best->S);
    if (better) best = &v, best_occ = occ;
  }
  if (!best) best = &g_variants[D == 128 ? 0 : 3], best_occ = 1;
  *ctas_per_sm = best_occ;
  return *best;
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
  if (const char* e = getenv("KD_ATTN_SPLITS")) splits = std::max(1, atoi(e));  // A/B knob
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
  if (a.flags & ~(uint32_t)KD_ATTN_LSE) return fail(KD_ERR_INVALID_ARG, "attention: unknown flags");
  return KD_OK;
}

}  // namespace attn

kd_status attention_scratch_bytes(const kd_attr_attention& a, uint64_t* bytes) {
  if (a.dtype == KD_F32) {  // fp32 parity kernel: no scratch
    *bytes = 256;
    return KD_OK;
  }
  kd_status s = attn::validate(a);
  if (s) return s;
  attn::Shape sh = attn::choose(a);
  const uint64_t units = (uint64_t)a.rows * a.n_kv_heads, G = a.n_heads / a.n_kv_heads;
  if (units >= kMaxCounters) return fail(KD_ERR_UNSUPPORTED, "attention: too many (sequence, kv head) units");
  uint64_t n = kScratchCounterBytes;  // per-unit split counters + the item ticket counter
  if (sh.splits > 1) n += units * sh.splits * G * (a.head_dim + 1) * 4;
  *bytes = (n + 255) / 256 * 256;
  return KD_OK;
}

kd_status launch_attention(const kd_attr_attention& a, const void* q, const void* kc, const void* vc,
                           const int32_t* bt, const int32_t* sl, void* out, const LaunchCtx& c, uint32_t* signals) {
  if (a.dtype == KD_F32) {
    if (!q || !kc || !vc || !bt || !sl || !out) return fail(KD_ERR_INVALID_ARG, "attention: NULL pointer");
    if (a.flags) return fail(KD_ERR_UNSUPPORTED, "attention (fp32): KD_ATTN_LSE partials are bf16-path only");
    if (a.rows == 0 || a.n_kv_heads == 0 || a.n_heads % a.n_kv_heads || a.head_dim == 0 || a.page == 0)
      return fail(KD_ERR_UNSUPPORTED, "attention (fp32): unsupported shape");
    kd_status st = launch_attention_f32(a, (const float*)q, (const float*)kc, (const float*)vc, bt, sl, (float*)out, c);
    if (!st && signals) *signals = attention_f32_signals(a);
    return st;
  }
  kd_status s = attn::validate(a);
  if (s) return s;
  if (!q || !kc || !vc || !bt || !sl || !out) return fail(KD_ERR_INVALID_ARG, "attention: NULL pointer");
  attn::Shape sh = attn::choose(a);
  const int G = a.n_heads / a.n_kv_heads;
  if (!c.scratch) return fail(KD_ERR_INVALID_ARG, "attention: scratch required");
  attn::Params P;
  P.q = (const __nv_bfloat16*)q;
  P.kc = (const __nv_bfloat16*)kc;
  P.vc = (const __nv_bfloat16*)vc;
  P.bt = bt;
  P.sl = sl;
  P.out = (__nv_bfloat16*)out;
  P.lse_off = (size_t)a.rows * a.n_heads * a.head_dim * 2;
  {
    const char* e = getenv("KD_ATTN_PREFETCH");
    P.prefetch = e ? atoi(e) : 1;
    const char* e2 = getenv("KD_ATTN_L2PF");
    P.l2pf = e2 ? atoi(e2) : 8;  // (same box, 3 rounds: 0 / 8 / 16 / 24 pages → 8.75 / 8.71 / 8.71 / 8.74 ms per step)
  }
  P.lse = (a.flags & KD_ATTN_LSE) ? (float*)((uint8_t*)out + P.lse_off) : nullptr;
  const uint64_t units = (uint64_t)a.rows * a.n_kv_heads;
  if (units >= kMaxCounters) return fail(KD_ERR_UNSUPPORTED, "attention: too many (sequence, kv head) units");
  P.counter = (unsigned*)c.scratch;
  P.work = P.counter + (kMaxCounters - 1);
  P.part_o = (float*)((uint8_t*)c.scratch + kScratchCounterBytes);
  P.part_lse = P.part_o + units * sh.splits * G * a.head_dim;
  P.Hq = a.n_heads;
  P.Hkv = a.n_kv_heads;
  P.rows = (int)a.rows;
  P.G = G;
  P.pps = a.pages_per_seq;
  P.splits = sh.splits;
  P.pages_per_split = sh.pages_per_split;
  P.scale_log2 = (float)(1.4426950408889634 / sqrt((double)a.head_dim));
  P.epi = c.epi;
  kd_status ks = kernels_init();
  if (ks) return ks;
  int per_sm = 1;
  const attn::Variant& v = attn::pick(a.head_dim, G, &per_sm);
  const int n_items = (int)(units * sh.splits);
  const int grid = std::min(n_items, per_sm * kNumSMs);
  if (getenv("KD_ATTN_DEBUG"))
    fprintf(stderr, "attention: D=%d S=%d G=%d per_sm=%d grid=%d items=%d splits=%d smem=%zu\n", v.D, v.S, G, per_sm,
            grid, n_items, sh.splits, v.smem(G));
  static unsigned long long* prof = nullptr;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(c.stream, &cap);
  const bool do_prof = getenv("KD_ATTN_PROF") && cap == cudaStreamCaptureStatusNone;
  if (do_prof && !prof) cudaMalloc(&prof, 64 + 8 * 5 * 4096);
  P.prof = do_prof ? prof : nullptr;
  P.tl = tl_next(300);
  static cudaEvent_t pe0 = nullptr, pe1 = nullptr;
  if (do_prof) {
    cudaMemsetAsync(prof, 0, 64 + 8 * 5 * 4096, c.stream);
    if (!pe0) cudaEventCreate(&pe0), cudaEventCreate(&pe1);
    cudaEventRecord(pe0, c.stream);
  }
  // K/V caches as 2-D [pages·Hkv·16 token rows][D] tensors (the pool size is
  // not part of the attributes: the row extent is set to 2^30, addresses come
  // from the block table)
  // viewed as 3-D (64 dims, D/64 halves, token rows) so one TMA moves a slab
  CUtensorMap tk, tv;
  const uint64_t dims[3] = {64, a.head_dim / 64u, 1ull << 30};
  const uint64_t strides[2] = {128, a.head_dim * 2u};
  const uint32_t box[3] = {64, a.head_dim / 64u, (uint32_t)attn::kPage};
  ks = encode_bf16_sw128(&tk, kc, 3, dims, strides, box);
  if (ks) return ks;
  ks = encode_bf16_sw128(&tv, vc, 3, dims, strides, box);
  if (ks) return ks;
  KD_CUDA_CHECK(kd_launch(v.fn, dim3(grid), dim3(attn::kThreads), v.smem(G), c.stream, tk, tv, P, n_items),
                "attention launch");
  if (do_prof) cudaEventRecord(pe1, c.stream);
  if (do_prof) {
    unsigned long long h[8];
    cudaMemcpyAsync(h, prof, 64, cudaMemcpyDeviceToHost, c.stream);
    cudaStreamSynchronize(c.stream);
    fprintf(stderr, "attn prof: grid %d producer-empty-wait %.3g cyc/CTA; consumer full-wait %.3g busy %.3g cyc/warp; pages %llu (%.0f busy cyc/page)\n",
            grid, (double)h[0] / grid, (double)h[1] / (grid * attn::kWarps), (double)h[2] / (grid * attn::kWarps), h[3],
            (double)h[2] / (double)(h[3] ? h[3] : 1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, pe0, pe1);
    if (grid <= 4096) {
      std::vector<unsigned long long> cta(5 * grid);
      cudaMemcpy(cta.data(), prof + 8, 8 * 5 * grid, cudaMemcpyDeviceToHost);
      unsigned long long ce = 0, ee = 0;
      for (int i = 0; i < grid; ++i) ce = std::max(ce, cta[5 * i + 3]), ee = std::max(ee, cta[5 * i + 4]);
      unsigned long long t0 = ~0ull, t1 = 0;
      for (int i = 0; i < grid; ++i) t0 = std::min(t0, cta[5 * i + 1]), t1 = std::max(t1, cta[5 * i + 2]);
      int late = 0;
      double max_life = 0;
      for (int i = 0; i < grid; ++i) {
        if (cta[5 * i + 1] - t0 > 5000) ++late;
        max_life = std::max(max_life, (double)(cta[5 * i + 2] - cta[5 * i + 1]));
      }
      fprintf(stderr, "attn prof: last consumer end %.1f us, last epilogue end %.1f us\n", (ce - t0) / 1e3, (ee - t0) / 1e3);
      fprintf(stderr, "attn prof: span %.1f us, CTAs starting >5us late: %d, max lifetime %.1f us\n", (t1 - t0) / 1e3,
              late, max_life / 1e3);
      for (int i = 0; i < 6; ++i)
        fprintf(stderr, "  cta %d sm %llu start %.1f end %.1f\n", i, cta[5 * i], (cta[5 * i + 1] - t0) / 1e3,
                (cta[5 * i + 2] - t0) / 1e3);
      for (int i = grid - 3; i < grid; ++i)
        fprintf(stderr, "  cta %d sm %llu start %.1f end %.1f\n", i, cta[5 * i], (cta[5 * i + 1] - t0) / 1e3,
                (cta[5 * i + 2] - t0) / 1e3);
    }
    fprintf(stderr, "attn prof: eager launch %.1f us; producer lifetime %.1f us/CTA -> clock %.0f MHz\n", ms * 1e3,
            (double)h[7] / grid / 1e3, (double)h[4] / (double)h[7] * 1e3);
    fprintf(stderr, "attn prof: producer total %.3g cyc/CTA, item-start %.3g, issue(lane0 incl. empty wait) %.3g\n",
            (double)h[4] / grid, (double)h[5] / grid, (double)h[6] / grid);
  }
  if (signals) return attention_signals(a, signals);
  return KD_OK;
}

kd_status attention_grid(const kd_attr_attention& a, uint32_t* grid) {
  kd_status st = attn::validate(a);
  if (st) return st;
  st = kernels_init();
  if (st) return st;
  const attn::Shape sh = attn::choose(a);
  int per_sm = 1;
  attn::pick(a.head_dim, a.n_heads / a.n_kv_heads, &per_sm);
  const int n_items = (int)((uint64_t)a.rows * a.n_kv_heads * sh.splits);
  *grid = (uint32_t)std::min(n_items, per_sm * kNumSMs);
  return KD_OK;
}

kd_status attention_signals(const kd_attr_attention& a, uint32_t* s) {
  if (a.dtype == KD_F32) {
    *s = attention_f32_signals(a);
    return KD_OK;
  }
  kd_status st = attn::validate(a);
  if (st) return st;
  *s = (uint32_t)a.rows * a.n_kv_heads;  // one finishing CTA per (sequence, kv head)
  return KD_OK;
}

kd_status attention_init_attrs() {
  for (attn::Variant& v : attn::g_variants) {
    const size_t smem = v.smem(attn::kMaxG);
    KD_CUDA_CHECK(cudaFuncSetAttribute(v.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                  "attention smem attr");
    // one carveout (max shared memory) for every kernel of the step: the SM never
    // has to drain and re-split L1/shared memory between consecutive launches
    KD_CUDA_CHECK(cudaFuncSetAttribute(v.fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100), "attention carveout");
  }
  return KD_OK;
}

}  // namespace kd
