// mega.cu — f1: a persistent per-device megakernel that executes a device's
// whole static schedule (the launch-overhead motive is
// PAPER.md §3.3 P:281 "kernel launch overhead" and P:398 "CUDA Graph ... to
// reduce launch overheads"). One launch per step replaces the per-kernel CUDA
// graph: every op of the schedule becomes a task, every task is cut into
// units, and each CTA (one per SM, co-resident by cooperative launch) walks the
// task list in schedule order with warp-specialised roles that persist across
// tasks:
//  * warp 0, loader: all global→shared traffic through one 8 KB-slot arena —
//    GEMM stages (weight boxes + activation boxes, TMA) and attention page
//    slabs (K/V, TMA) — plus the query rows (bulk copy). It runs ahead of the
//    consumers across task boundaries: a GEMM's weight boxes and an
//    attention's KV pages do not depend on the previous task, so they are
//    requested while the previous task's epilogue, fold or norm still runs;
//    only the activation boxes / query rows / the one page this step appends
//    to wait for the task's dependencies (in-kernel flag waits, below).
//  * warp 1, MMA issuer (tcgen05.mma, fp32 accumulators double-buffered in TMEM).
//  * warp 2, attention merge (per-item warp states, split LSE merge).
//  * warps 4-11, workers: attention consumers (mma.sync online softmax, one
//    warp per page slot class), the GEMM epilogue (TMEM → bf16 output or fp32
//    split partial + fold), and the element-wise tasks (add+RMSNorm, RoPE +
//    KV append, SiLU·mul, residual add) with the same per-element arithmetic
//    as the standalone kernels (bitwise identical for those ops).
// Dependencies: a task waits (ld.acquire.gpu on the producer tasks' completion
// counters) for exactly the tasks whose declared spans conflict with its own
// (RAW, WAR, WAW over the plan's buffers — the DAG of P:276 plus the
// anti-dependences a concurrent executor must also respect), transitively
// reduced. Counters are monotonic across steps: a task is complete in step e
// (0-based) at (e + 1) · units, so nothing is ever reset.
// The schedule is a topological order and every wait points to an earlier
// task, so with all CTAs resident the kernel cannot deadlock.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "launch.hpp"
#include "mmasync.cuh"
#include "tcgen05.cuh"

namespace kd {
namespace mega {

using gemm::bulk_g2s;
using gemm::mbar_arrive;
using gemm::mbar_expect_tx;
using gemm::mbar_init;
using gemm::mma_bf16;
using gemm::mma_bf16_ws;
using gemm::mma_commit_ws;
using gemm::mma_commit;
using gemm::named_bar;
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
using mmas::movm_t;
using mmas::tile_off;
using mmas::tma_3d;

constexpr int kWarps = 12, kThreads = kWarps * 32;
constexpr int kLoader = 0, kMma = 1, kMerge = 2, kLoader2 = 3, kW0 = 4;  // workers: warps 4..11
constexpr int kWorkers = 8, kWorkerThreads = kWorkers * 32;
constexpr int kSlot = 8192;   // arena slot: one attention page (K + V slab, D ≤ 128) or 1/SPS GEMM stage
constexpr int kMaxSlots = 28;
constexpr int kMaxStages = 8;
constexpr int kMaxDep = 8;
constexpr int kMaxG = 8;
constexpr int kPage = 16;
constexpr int kAccCols = 128;  // TMEM columns per accumulator (mma_n ≤ 128), two accumulators
constexpr int kBarW = 1, kBarHalf0 = 2;  // named barriers: all workers; worker halves (2, 3)
constexpr int kFastSplits = 4, kFastSplitLse = 128;

enum Kind : int { MK_NORM = 1, MK_GEMM = 2, MK_ROPE = 3, MK_ATTN = 4, MK_SILU = 5, MK_RESID = 6 };

struct alignas(64) Task {
  CUtensorMap tm0;  // GEMM: W [N][K]; ATTN: K cache slabs
  CUtensorMap tm1;  // GEMM: X [M][K]; ATTN: V cache slabs
  int kind;
  int epi;              // GEMM epilogue: 0 plain bf16 Y, 1 RoPE + KV append (KD_OP_QKV_ROPE), 2 SiLU·mul (KD_OP_GEMM_SILU)
  unsigned done_units;  // completion increments per step
  int n_dep;
  int dep[kMaxDep];
  unsigned dep_units[kMaxDep];
  int rot;      // element-wise: unit u runs on CTA (u + rot) % grid
  int n_units;  // element-wise units; GEMM: tiles·KB k-block units; ATTN: items
  const void* a0;
  const void* a1;
  const void* a2;
  void* o0;
  void* o1;
  void* o2;
  const void* dl[kMaxDeltas];
  int n_delta;
  int M, N, K;                         // GEMM / NORM (M rows, N = hidden) / SILU (N = F) / RESID (K = n8)
  int KB, tiles, kbs, mma_n, maxc, gg;  // GEMM: k-blocks per tile, tiles, 64-col boxes per stage, MMA N, contributors bound, CTAs
  unsigned* ctr;                       // GEMM tile arrivals / ATTN unit (split) arrivals
  unsigned* ticket;                    // ATTN item tickets
  const void* ctr2;                    // GEMM RoPE epilogue: block table
  float* part;                         // GEMM partials [tiles][maxc][M][128] / ATTN part_o
  float* part_lse;                     // ATTN
  int Hq, Hkv, D, G, pps, splits, pps_split, page, n_dyn, rows, slot_offset;
  float scale_log2, eps;
  const double* freq;                  // ROPE θ^(−2i/D)
  const float2* rtab;                  // GEMM RoPE epilogue: (cos, sin)[row][D/2] of this step
};

struct Geo {
  int NS, NG, SPS, A;  // arena slots, GEMM stages, slots per stage, attention slots (multiple of 8)
  int n_tasks;
  int Gm;              // comb buffers sized for Gm query heads per kv head
  uint32_t off_q, off_comb, off_ml, off_bar, off_misc;  // dynamic smem offsets
  unsigned long long* trace;  // debug (nullable): [task][CTA][role 4][start, deps, end] %globaltimer
  int pf;                     // prefetch each task's tensor maps at its start (A/B knob KD_MEGA_PF)
  int dbg;                    // experiments (KD_MEGA_DBG): 1 consumers skip the math, 2 + loader skips the TMA
  int l2pf;                   // GEMM weight stages prefetched into L2 during the dependency wait (KD_MEGA_L2PF)
  // RoPE (cos, sin) tables, one per distinct (seq_len buffer, rows, D/2, θ):
  // every CTA computes a slice at kernel start (the step's positions are
  // fixed for the whole step), tab_ready counts the CTAs that finished
  int n_tab;
  const int32_t* tab_sl[4];
  const double* tab_freq[4];
  float2* tab[4];
  int tab_rows[4], tab_half[4];
  unsigned* tab_ready;
};
enum Role : int { R_LOAD = 0, R_MMA = 1, R_MERGE = 2, R_WORK = 3 };
// trace layout: [task][CTA][role 5][4 stamps]; role R_EPI = the GEMM epilogue
// of the CTA's last piece: tfull seen, partial stored + arrived, all partials
// present, fold done
constexpr int kRoles = 5, kStamps = 4;
enum { R_EPI = 4 };
__device__ __forceinline__ void stamp(const Geo& g, int t, int role, int k) {
  if (g.trace) {
    unsigned long long v;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
    g.trace[(((size_t)t * gridDim.x + blockIdx.x) * kRoles + role) * kStamps + k] = v;
  }
}

// ------------------------------------------------------------------ waits with watchdogs
// A broken protocol must not hang the box: every spin is bounded (≈ 4 s of
// clock). The first thread to time out records where (code, CTA, warp, task,
// two wait-specific words) in the control block, sets the runtime error word
// and raises a grid-wide abort flag; every other wait polls the flag and
// returns, so the launch drains (with garbage) and kd_runtime_check reports it.
constexpr long long kTimeout = 1ll << 33;
struct Sm;
__device__ void report(const Sm& S, unsigned* err, unsigned code, unsigned a, unsigned b);
__device__ __forceinline__ bool aborted(const Sm& S);
__device__ __forceinline__ bool mbar_try(uint64_t* b, unsigned parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mwait(uint64_t* b, unsigned parity, unsigned* err, const Sm& S) {
  if (mbar_try(b, parity)) return;
  const long long t0 = clock64();
  for (unsigned n = 0;; ++n) {
    if (mbar_try(b, parity)) return;
    if ((n & 1023u) == 1023u) {
      if (aborted(S)) return;
      if (clock64() - t0 > kTimeout) {
        report(S, err, 5u, smem_u32(b), parity);
        return;
      }
    }
  }
}
__device__ __forceinline__ void mwait_sleep(uint64_t* b, unsigned parity, unsigned* err, const Sm& S) {
  const long long t0 = clock64();
  for (unsigned n = 0; !mbar_try(b, parity); ++n) {
    __nanosleep(128);
    if ((n & 255u) == 255u) {
      if (aborted(S)) return;
      if (clock64() - t0 > kTimeout) {
        report(S, err, 5u, smem_u32(b), parity);
        return;
      }
    }
  }
}
__device__ __forceinline__ unsigned ld_acq_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_rel_gpu(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// publish one completed unit of task t: caller ordered the unit's stores
// before this thread (bar.sync); the release covers them (cumulativity)
__device__ __forceinline__ void signal_done(unsigned* done, int t, unsigned units = 1u) {
  fence_acq_rel_gpu();
  red_rel_gpu(done + t, units);
}

__host__ __device__ __forceinline__ long long ubeg(long long c, long long U, long long G) { return c * U / G; }
__host__ __device__ __forceinline__ long long uowner(long long u, long long U, long long G) {
  return ((u + 1) * G + U - 1) / U - 1;
}

struct Sm {
  uint8_t* arena;
  uint64_t *gfull, *gempty, *afull, *aempty, *tfull, *tempty, *qfull, *qempty, *ifull, *iempty, *cfull, *cempty;
  __nv_bfloat16* qsm;  // [2][Gm·D]
  float* comb;         // [8][Gm][D]
  float* comb_ml;      // [8][Gm][2]
  int* s_item;         // [4]
  int* s_len;          // [4] item ring: context length of the item
  int *rpos, *rpg;     // [128] fused-RoPE fold staging
  uint64_t *xg, *xa;   // arena hand-over between the loaders: GEMM stages drained / odd attention slots drained
  float* red;          // [8] norm partial sums
  unsigned* bcast;     // [4]
  float *s_w, *s_M, *s_L, *s_lse;
  uint32_t* tmem_slot;
  int* cur;            // [12] task index per warp (diagnostics)
  unsigned* abortp;    // control block: grid-wide abort flag
  unsigned* rec;       // control block: first timeout record [8]
};

__device__ __forceinline__ bool aborted(const Sm& S) { return *(volatile unsigned*)S.abortp != 0u; }
__device__ void report(const Sm& S, unsigned* err, unsigned code, unsigned a, unsigned b) {
  if (atomicCAS(S.abortp, 0u, 1u) == 0u) {
    const int warp = threadIdx.x >> 5;
    S.rec[0] = code;
    S.rec[1] = blockIdx.x;
    S.rec[2] = warp;
    S.rec[3] = threadIdx.x & 31;
    S.rec[4] = (unsigned)S.cur[warp];
    S.rec[5] = a;
    S.rec[6] = b;
    S.rec[7] = 1u;
    __threadfence();
    if (err) atomicExch(err, code);
  }
}
// the calling thread waits until every dependency of T completed this step
__device__ void deps_wait(const Task& T, const unsigned* done, unsigned ep, unsigned* err, const Sm& S) {
  for (int i = 0; i < T.n_dep; ++i) {
    const unsigned target = (ep + 1u) * T.dep_units[i];
    const unsigned* p = done + T.dep[i];
    if (ld_acq_gpu(p) >= target) continue;
    const long long t0 = clock64();
    for (unsigned n = 0; ld_acq_gpu(p) < target; ++n) {
      __nanosleep(64);
      if ((n & 255u) == 255u) {
        if (aborted(S)) return;
        if (clock64() - t0 > kTimeout) {
          report(S, err, 4u, (unsigned)T.dep[i], ld_acq_gpu(p));
          return;
        }
      }
    }
  }
  fence_acq_rel_gpu();
}

// Loader state, all in registers (lane 0 of the loader warp). The arena's
// slots are used either as GEMM stages (stage q = slots [q·SPS, (q+1)·SPS),
// round robin) or as attention page slots (round robin, items start on a
// multiple of 8). Before a slot is refilled, the release of its previous use
// must have been waited for: masks of the uses whose release is still owed,
// and the mbarrier parity of that release.
struct Ld {
  unsigned gs = 0;         // GEMM stage fills so far (the MMA warp counts the same)
  int gq = 0;              // next stage
  unsigned gph = 0;        // use parity of the next fill of stage gq (= (gs / NG) & 1)
  uint32_t gpend = 0;      // stages whose release is owed
  uint32_t gpar = 0;       // their release parity
  uint32_t gslots = 0;     // slots covered by owed stages
  uint32_t apend = 0;      // attention slots whose release is owed
  uint32_t apar = 0;       // their release parity
  uint32_t afill = 0;      // per slot: use parity of its next attention fill
  int apos = 0;            // next attention slot
};
__device__ __forceinline__ uint32_t stage_mask(int q, int SPS) { return ((1u << SPS) - 1u) << (q * SPS); }
// wait for the owed release of GEMM stage q (if any)
__device__ __forceinline__ void free_stage(Ld& L, const Sm& S, int q, int SPS, unsigned* err) {
  if ((L.gpend >> q) & 1u) {
    mwait(&S.gempty[q], (L.gpar >> q) & 1u, err, S);
    L.gpend &= ~(1u << q);
    L.gslots &= ~stage_mask(q, SPS);
  }
}
// wait for every owed attention release among the slots of mask m
__device__ __forceinline__ void free_attn(Ld& L, const Sm& S, uint32_t m, unsigned* err) {
  m &= L.apend;
  L.apend &= ~m;
  while (m) {
    const int s = __ffs(m) - 1;
    mwait(&S.aempty[s], (L.apar >> s) & 1u, err, S);
    m &= m - 1u;
  }
}

// ================================================================== loader
__device__ void load_gemm(const Task& T, int t, const Sm& S, const Geo& g, const unsigned* done, unsigned ep, unsigned* err,
                          Ld& L, unsigned nattn, unsigned& xa_seen) {
  const int lane = threadIdx.x & 31;
  // the secondary loader's odd attention slots are all released (every xa
  // phase is consumed in order, before the primary re-arms xg: no aliasing)
  if (lane == 0)
    for (; xa_seen != nattn; ++xa_seen) mwait(S.xa, xa_seen & 1u, err, S);
  const int KB = T.KB, gg = T.gg, NG = g.NG, SPS = g.SPS;
  const long long U = (long long)T.tiles * KB;
  const int c = blockIdx.x;
  if (c >= gg) return;
  const long long u0 = ubeg(c, U, gg), u1 = ubeg(c + 1, U, gg);
  const int n = (int)(u1 - u0);
  if (lane != 0 || n <= 0) return;
  const uint64_t pw = policy_evict_first(), px = policy_evict_last();
  const int kbs = T.kbs, xbox = T.mma_n * 128;
  const unsigned tx = (unsigned)(kbs * (16384 + xbox));
  const int npre = min(NG, n);
  const CUtensorMap* mw = &T.tm0;
  const CUtensorMap* mx = &T.tm1;
  uint8_t* const arena = S.arena;
  // (tile, k-block) and the ring position advance incrementally: a 64-bit
  // division is a ~300-cycle subroutine, per stage
  int tile = (int)(u0 / KB), kb = (int)(u0 % KB);
  const int kb0 = kb, q0 = L.gq;
  auto load_x = [&](int qq, int kk) {
    uint8_t* base = arena + (size_t)qq * SPS * kSlot + kbs * 16384;
    for (int b = 0; b < kbs; ++b) tma_load_2d(base + b * xbox, mx, (kk * kbs + b) * 64, 0, &S.gfull[qq], px);
  };
  for (int i = 0; i < n; ++i) {
    const int q = L.gq;
    free_attn(L, S, stage_mask(q, SPS), err);  // (slots last used by attention pages)
    free_stage(L, S, q, SPS, err);
    mbar_expect_tx(&S.gfull[q], tx);
    uint8_t* base = arena + (size_t)q * SPS * kSlot;
    for (int b = 0; b < kbs; ++b) tma_load_2d(base + b * 16384, mw, (kb * kbs + b) * 64, tile * 128, &S.gfull[q], pw);
    L.gpend |= 1u << q;
    L.gpar = (L.gpar & ~(1u << q)) | (L.gph << q);
    L.gslots |= stage_mask(q, SPS);
    if (i >= npre) {
      load_x(q, kb);
    } else if (i == npre - 1) {
      // weights of the first npre stages are in flight; the HBM would idle
      // while X's producers finish (their fold / norm chain outlasts the
      // ring), so the next l2pf stages' weights go to L2 (bulk prefetch),
      // then wait for the producers of X and issue the held-back X boxes
      {
        int tt = tile, kk = kb;
        const int pf = min(n - npre, g.l2pf);
        for (int j = 0; j < pf; ++j) {
          if (++kk == KB) kk = 0, ++tt;
          for (int b = 0; b < kbs; ++b) gemm::tma_prefetch_2d(mw, (kk * kbs + b) * 64, tt * 128);
        }
      }
      deps_wait(T, done, ep, err, S);
      stamp(g, t, R_LOAD, 1);
      asm volatile("fence.proxy.async.global;" ::: "memory");
      int qq = q0, kk = kb0;
      for (int j = 0; j < npre; ++j) {
        load_x(qq, kk);
        if (++qq == NG) qq = 0;
        if (++kk == KB) kk = 0;
      }
    }
    ++L.gs;
    if (++L.gq == NG) L.gq = 0, L.gph ^= 1u;
    if (++kb == KB) kb = 0, ++tile;
  }
}

// Attention pages are requested by TWO loader warps (a single warp's
// ~300-cycle dependent issue path per page cannot keep up with HBM): page t
// of an item goes to slot (base + t) mod A, base and A even, so loader warp 0
// (the primary: tickets, item ring, query rows, GEMM stages) fills the even
// slots and warp 3 (the secondary, attention only) the odd ones. The arena
// changes hands at task-kind boundaries: before an attention task the primary
// waits for every owed GEMM-stage release and arrives on xg (the secondary
// waits xg before its first page); after one the secondary waits for every
// owed odd-slot release and arrives on xa (the primary waits xa before its
// next GEMM stage).
template <bool kPrimary>
__device__ void load_attn(const Task& T, int t, const Sm& S, const Geo& g, const unsigned* done, unsigned ep, unsigned* err,
                          unsigned& ak, unsigned& ci, Ld& L, unsigned& nattn, unsigned* xa_seen) {
  const int lane = threadIdx.x & 31;
  const int G = (int)gridDim.x, c = blockIdx.x;
  const int D = T.D, Hkv = T.Hkv, Gq = T.G, A = g.A, splits = T.splits, rows = T.rows, ppsp = T.pps_split;
  const int pps = T.pps, Hq = T.Hq, n_dyn = T.n_dyn, n_items = T.n_units, Gm = g.Gm, NG = g.NG;
  const int soff = T.slot_offset;
  const unsigned slab = (unsigned)(kPage * D * 2);
  const unsigned per_step = (unsigned)(n_dyn + G);
  unsigned* const ticket = T.ticket;
  const CUtensorMap* mk = &T.tm0;
  const CUtensorMap* mv = &T.tm1;
  const __nv_bfloat16* qg = (const __nv_bfloat16*)T.a0;
  uint8_t* const arena = S.arena;
  const uint64_t pol = policy_evict_first();
  const int32_t* bt = (const int32_t*)T.a1;
  const int32_t* sl = (const int32_t*)T.a2;
  const int par = kPrimary ? 0 : 1;
  // ---- arena hand-over (GEMM stages → attention slots)
  if (kPrimary) {
    if (lane == 0) {
      for (; *xa_seen != nattn; ++*xa_seen) mwait(S.xa, *xa_seen & 1u, err, S);
      for (int q = 0; q < NG; ++q) free_stage(L, S, q, g.SPS, err);
      mbar_arrive(S.xg);
    }
  } else {
    if (lane == 0) mwait(S.xg, nattn & 1u, err, S);
  }
  __syncwarp();
  auto publish = [&](int it, int len) {
    if (lane == 0) {
      const int is = (int)(ak & 3u);
      if (ak >= 4) mwait(&S.iempty[is], ((ak >> 2) - 1u) & 1u, err, S);
      S.s_item[is] = it;
      S.s_len[is] = len;
      mbar_arrive(&S.ifull[is]);
    }
    __syncwarp();
    ++ak;
  };
  auto take = [&](int& len) -> int {  // the secondary reads the item ring
    const int is = (int)(ak & 3u);
    mwait(&S.ifull[is], (ak >> 2) & 1u, err, S);
    const int it = S.s_item[is];
    len = S.s_len[is];
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.iempty[is]);
    ++ak;
    return it;
  };
  // ticket of the next item: the atomic is issued early and resolved later
  // (its ~1 µs round trip overlaps the current item's page requests)
  auto draw = [&]() -> unsigned { return lane == 0 ? atomicAdd(ticket, 1u) : 0u; };
  auto resolve = [&](unsigned raw) -> int {
    const unsigned tk = __shfl_sync(0xffffffffu, raw, 0) - ep * per_step;
    return tk < (unsigned)n_dyn ? G + (int)tk : -1;
  };
  int it = -1, len = 0;
  if (kPrimary) {
    it = c < n_items ? c : resolve(draw());
    len = it >= 0 ? __ldg(sl + (it / splits) % rows) - soff : 0;
  }
  bool first = true;
  for (;;) {
    unsigned raw_next = 0;
    if (kPrimary) {
      publish(it, len);
      if (it < 0) break;
      raw_next = draw();
    } else {
      it = take(len);
      if (it < 0) break;
    }
    const int split = it % splits, unit = it / splits;
    const int gh = unit / rows, b = unit % rows;
    const int p0 = split * ppsp;
    const int np = max(0, min((len + kPage - 1) / kPage, p0 + ppsp) - p0);
    int base = (L.apos + 7) / 8 * 8;
    if (base >= A) base -= A;
    // pages strictly before the one holding the appended position may be
    // requested before the dependencies (RoPE/append writes only that page)
    const int safe = first ? max(0, min(np, (len - 1) / kPage - p0)) : 0;
    const int npre = min(safe, A);
    // the primary sends the query rows (RoPE output) right after its
    // dependency wait — before any page beyond the ring, whose slot only
    // frees once the consumers (which need q) release it
    bool qdone = !kPrimary;
    auto gate = [&]() {
      if (first) {
        if (lane == 0) {
          deps_wait(T, done, ep, err, S);
          if (kPrimary) stamp(g, t, R_LOAD, 1);
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        first = false;
      }
      if (kPrimary && !qdone) {
        if (lane == 0) {
          const int qs = (int)(ci & 1u);
          if (ci >= 2) mwait(&S.qempty[qs], ((ci >> 1) - 1u) & 1u, err, S);
          mbar_expect_tx(&S.qfull[qs], (unsigned)(Gq * D * 2));
          bulk_g2s(S.qsm + (size_t)qs * Gm * D, qg + (size_t)b * Hq * D + (size_t)gh * Gq * D, (unsigned)(Gq * D * 2),
                   &S.qfull[qs]);
        }
        qdone = true;
      }
      __syncwarp();
    };
    const int32_t* btr = bt + (size_t)b * pps + p0;
    int ids = lane < np ? __ldg(btr + lane) : 0;  // this lane's page id, 32-page chunks, one chunk ahead
    int it_next = -2, len_next = 0;
    int s = base + par;
    for (int j0 = 0; j0 < np; j0 += 32) {
      const int cur = ids;
      if (j0 + 32 < np) ids = j0 + 32 + lane < np ? __ldg(btr + j0 + 32 + lane) : 0;
      const int cnt = min(32, np - j0);
      for (int x = par; x < cnt; x += 2) {
        if (first ? (j0 + x >= npre) : !qdone) gate();
        const int pid = __shfl_sync(0xffffffffu, cur, x);
        if (lane == 0) {
          const uint32_t bit = 1u << s;
          if (L.apend & bit) mwait(&S.aempty[s], (L.apar >> s) & 1u, err, S);
          const uint32_t p = (L.afill >> s) & 1u;
          L.apend |= bit;
          L.apar = (L.apar & ~bit) | (p << s);
          L.afill ^= bit;
          const int row = (pid * Hkv + gh) * kPage;
          uint8_t* dst = arena + (size_t)s * kSlot;
          if (g.dbg >= 2) {
            mbar_arrive(&S.afull[s]);
          } else {
            mbar_expect_tx(&S.afull[s], 2u * slab);
            tma_3d(dst, mk, 0, 0, row, &S.afull[s], pol);
            tma_3d(dst + slab, mv, 0, 0, row, &S.afull[s], pol);
          }
        }
        s += 2;
        if (s >= A) s -= A;
      }
      if (kPrimary && j0 == 0) {  // next item's ticket and length, well before they are needed
        it_next = resolve(raw_next);
        len_next = it_next >= 0 ? __ldg(sl + (it_next / splits) % rows) - soff : 0;
      }
    }
    if (first || !qdone) gate();
    if (kPrimary) {
      if (it_next == -2) {
        it_next = resolve(raw_next);
        len_next = it_next >= 0 ? __ldg(sl + (it_next / splits) % rows) - soff : 0;
      }
      ++ci;
      it = it_next;
      len = len_next;
    }
    L.apos = base + np;
    while (L.apos >= A) L.apos -= A;
  }
  // ---- arena hand-over (odd attention slots → the primary's next GEMM stages)
  if (!kPrimary && lane == 0) {
    const uint32_t m = L.apend;
    L.apend = 0;
    for (uint32_t x = m; x; x &= x - 1u) {
      const int s2 = __ffs(x) - 1;
      mwait(&S.aempty[s2], (L.apar >> s2) & 1u, err, S);
    }
    mbar_arrive(S.xa);
  }
  __syncwarp();
  ++nattn;
}

// ================================================================== MMA issuer
__device__ void mma_gemm(const Task& T, int tmark, const Sm& S, const Geo& g, uint32_t tmem, unsigned* err, unsigned& gs,
                         unsigned& pc) {
  const int lane = threadIdx.x & 31;
  const int KB = T.KB, gg = T.gg, NG = g.NG, SPS = g.SPS;
  const long long U = (long long)T.tiles * KB;
  const int c = blockIdx.x;
  if (c >= gg) return;
  const long long u0 = ubeg(c, U, gg), u1 = ubeg(c + 1, U, gg);
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(T.mma_n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const int kbs = T.kbs, xbox = T.mma_n * 128;
  const uint32_t arena = smem_u32(S.arena);
  int q = (int)(gs % (unsigned)NG);
  unsigned ph = (gs / (unsigned)NG) & 1u;
  int kb = (int)(u0 % KB);
  const int n = (int)(u1 - u0);
  for (int i = 0; i < n;) {
    const int len = min(n - i, KB - kb);  // piece: the rest of this tile within my range
    const unsigned acc = pc & 1u;
    if (pc >= 2) mwait(&S.tempty[acc], ((pc >> 1) - 1u) & 1u, err, S);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t td = tmem + acc * kAccCols;
    for (int v = 0; v < len; ++v) {
      mwait(&S.gfull[q], ph, err, S);
      if (g.trace && lane == 0 && i + v == n - 1) stamp(g, tmark, R_MMA, 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      {  // warp-uniform issue (elect.sync inside the asm: uniform descriptors, no waterfall)
        const uint32_t a = arena + (uint32_t)(q * SPS * kSlot);
        const uint32_t bx = a + kbs * 16384;
        const uint64_t ad0 = sw128_desc(a), bd0 = sw128_desc(bx);
        for (int b = 0; b < kbs; ++b)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            mma_bf16_ws(td, ad0 + (uint64_t)(b * 1024 + 2 * k), bd0 + (uint64_t)(b * (xbox >> 4) + 2 * k), idesc,
                        (v > 0 || b > 0 || k > 0) ? 1u : 0u);
        mma_commit_ws(&S.gempty[q]);
      }
      __syncwarp();
      ++gs;
      if (++q == NG) q = 0, ph ^= 1u;
    }
    if (lane == 0) mma_commit(&S.tfull[acc]);
    __syncwarp();
    ++pc;
    i += len;
    kb = 0;
  }
}

// fused a5 on the folded QKV tile (KD_OP_QKV_ROPE, weight rows pair-interleaved
// inside each head: rows n..n+3 = dims p, p + D/2, p + 1, p + 1 + D/2): the
// per-element arithmetic of rope_append_kernel on the bf16-rounded GEMM output
__device__ __forceinline__ float rbf(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }
__device__ __forceinline__ void rope_quad_m(const Task& T, const Sm& S, int j, int n, float4 a) {
  const int D = T.D, half = D / 2, G = T.Hq / T.Hkv;
  const int hall = n / D, rr = n - hall * D, p = rr >> 1;
  const int grp = hall / (G + 2), slot = hall - grp * (G + 2);
  const float xs[2] = {rbf(a.x), rbf(a.z)};
  const float ys[2] = {rbf(a.y), rbf(a.w)};
  const int pos = S.rpos[j];
  __nv_bfloat16 lo[2], hi[2];
  const float4 csn = __ldcg(reinterpret_cast<const float4*>(T.rtab + (size_t)j * half + p));  // pairs p, p + 1
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    if (slot <= G) {
      const float cs = u ? csn.z : csn.x, sn = u ? csn.w : csn.y;
      lo[u] = __float2bfloat16_rn(xs[u] * cs - ys[u] * sn);
      hi[u] = __float2bfloat16_rn(ys[u] * cs + xs[u] * sn);
    } else {
      lo[u] = __float2bfloat16_rn(xs[u]);
      hi[u] = __float2bfloat16_rn(ys[u]);
    }
  }
  const __nv_bfloat162 l2 = __halves2bfloat162(lo[0], lo[1]), h2 = __halves2bfloat162(hi[0], hi[1]);
  __nv_bfloat16* dst;
  if (slot < G) {
    dst = (__nv_bfloat16*)T.o0 + ((size_t)j * T.Hq + (size_t)grp * G + slot) * D;
  } else {
    dst = (__nv_bfloat16*)(slot == G ? T.o1 : T.o2) + (((size_t)S.rpg[j] * T.Hkv + grp) * T.page + pos % T.page) * D;
  }
  *reinterpret_cast<__nv_bfloat162*>(dst + p) = l2;
  *reinterpret_cast<__nv_bfloat162*>(dst + p + half) = h2;
}

// ================================================================== workers
// GEMM epilogue: TMEM → bf16 output (a whole tile) or fp32 partial, and the
// last contributor of a split tile folds every contributor's partial in
// contributor order (deterministic) into the bf16 output
__device__ void epi_gemm(const Task& T, int t, const Sm& S, const Geo& g, unsigned* done, unsigned ep, uint32_t tmem,
                         unsigned* err, unsigned& pc, const unsigned* g_tab_ready) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, wt = threadIdx.x - kW0 * 32;
  const long long U = (long long)T.tiles * T.KB;
  const int c = blockIdx.x;
  if (c >= T.gg) return;
  const long long u0 = ubeg(c, U, T.gg), u1 = ubeg(c + 1, U, T.gg);
  const int q = warp & 3, h = (warp - kW0) >> 2;
  const int row = q * 32 + lane;
  const int M = T.M, N = T.N;
  __nv_bfloat16* Y = (__nv_bfloat16*)T.o0;
  if (T.epi == 1) {
    // fused RoPE: each token's position and page of the appended slot, and the
    // step's (cos, sin) tables (every CTA computed a slice at kernel start) —
    // staged while the first piece still streams, off the fold's tail
    const int32_t* sl = (const int32_t*)T.a2;
    const int32_t* btp = (const int32_t*)T.ctr2;
    for (int j = wt; j < M; j += kWorkerThreads) {
      const int pos = __ldg(sl + j) - 1;
      S.rpos[j] = pos;
      S.rpg[j] = __ldg(btp + (size_t)j * T.pps + pos / T.page);
    }
    if (wt == 0) {
      const unsigned target = (ep + 1u) * gridDim.x;
      for (long long n2 = 0; ld_acq_gpu(g_tab_ready) < target; ++n2) {
        __nanosleep(32);
        if (n2 > (1ll << 26)) { report(S, err, 4u, 0xFFFFu, 0u); break; }
      }
      fence_acq_rel_gpu();
    }
    named_bar(kBarW, kWorkerThreads);
  }
  for (long long u = u0; u < u1;) {
    const int tile = (int)(u / T.KB);
    const long long tb = (long long)tile * T.KB, te = tb + T.KB;
    const long long pe = min(u1, te);
    const bool whole = (u == tb && pe == te) && T.epi == 0;  // (fused epilogues always go through the fold)
    const unsigned acc = pc & 1u;
    mwait_sleep(&S.tfull[acc], (pc >> 1) & 1u, err, S);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const bool lastp = pe == u1;
    if (lastp && wt == 0) stamp(g, t, R_EPI, 0);
    const uint32_t ta = tmem + acc * kAccCols + ((uint32_t)(q * 32) << 16);
    const int n = tile * 128 + row;
    const int f = (int)uowner(tb, U, T.gg);
    const int nc = (int)uowner(te - 1, U, T.gg) - f + 1, cidx = c - f;
    // partial layout [tile][contributor][weight row][Mp] (Mp = mma_n): a thread
    // owns one weight row, so its 16-token chunk goes out as 4 × 16-byte stores
    const int Mp = T.mma_n;
    float* part = T.part + ((size_t)tile * T.maxc + cidx) * (size_t)Mp * 128 + (size_t)row * Mp;
    for (int cc0 = h; cc0 * 16 < Mp; cc0 += 2) {
      uint32_t v[1][16];
#pragma unroll
      for (int b = 0; b < 1; ++b)
        if ((cc0 + 2 * b) * 16 < Mp) tmem_ld16_nowait(ta + (cc0 + 2 * b) * 16, v[b]);
      tmem_ld_wait();
#pragma unroll
      for (int b = 0; b < 1; ++b) {
        const int cc = cc0 + 2 * b;
        if (cc * 16 >= Mp) continue;
        if (whole) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int tok = cc * 16 + j;
            if (tok < M && n < N) Y[(size_t)tok * N + n] = __float2bfloat16_rn(__uint_as_float(v[b][j]));
          }
        } else {
#pragma unroll
          for (int j = 0; j < 16; j += 4)
            *reinterpret_cast<uint4*>(part + cc * 16 + j) = make_uint4(v[b][j], v[b][j + 1], v[b][j + 2], v[b][j + 3]);
        }
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.tempty[acc]);
    if (lastp && wt == 0) stamp(g, t, R_WORK, 1);
    named_bar(kBarW, kWorkerThreads);
    if (whole) {
      if (wt == 0) signal_done(done, t);
      if (lastp && wt == 0) stamp(g, t, R_EPI, 3);
    } else {
      // Split tile: every contributor publishes its partial (arrival count).
      // The contributors whose LAST piece of this task is this tile (all but
      // possibly the one whose range continues past the tile) then fold one
      // row slice each, in parallel, once every partial has landed.
      const int l = f + nc - 1;
      const bool l_folds = ubeg(l + 1, U, T.gg) == te;
      const int nf = nc == 1 ? 1 : (l - f) + (l_folds ? 1 : 0);
      const bool folder = nc == 1 || c < l || l_folds;
      if (wt == 0) {
        // (the acq_rel add releases every worker's partial stores: they are
        // ordered before it by the bar.sync above — cumulativity)
        atom_add_acq_rel_gpu(T.ctr + tile, 1u);
        if (lastp) stamp(g, t, R_EPI, 1);
        if (folder && nc > 1) {  // wait for the other contributors' partials
          const unsigned target = (ep + 1u) * (unsigned)nc;
          const long long t0 = clock64();
          for (unsigned it2 = 0; ld_acq_gpu(T.ctr + tile) < target; ++it2) {
            __nanosleep(32);
            if ((it2 & 255u) == 255u && (aborted(S) || clock64() - t0 > kTimeout)) {
              if (!aborted(S)) report(S, err, 4u, 0x10000u + (unsigned)tile, 0u);
              break;
            }
          }
          fence_acq_rel_gpu();
        }
      }
      if (lastp && wt == 0) stamp(g, t, R_EPI, 2);
      named_bar(kBarW, kWorkerThreads);
      if (folder) {
        const float* pt = T.part + (size_t)tile * T.maxc * Mp * 128;
        const int n0 = tile * 128;
        const int fi = nc == 1 ? 0 : c - f;
        if (T.epi == 2) {
          // SiLU·mul: tile = gate block (rows 0-63) + up block (rows 64-127);
          // a[tok][64·tile + i] = silu(bf16 g)·bf16 u — silu_mul_kernel's math.
          // This folder's 4-column groups: [g0, g1) of 16
          const int F = N / 2;
          const int g0 = fi * 16 / nf, ng = (fi + 1) * 16 / nf - g0;
          const int nt4 = (M + 3) / 4;
          for (int e = wt; e < ng * nt4; e += kWorkerThreads) {
            const int gi = e / nt4, t4 = (e - gi * nt4) * 4, i4 = (g0 + gi) * 4;
            float4 ga[4], ua[4];
            for (int k = 0; k < nc; ++k) {
              float4 gv[4], uv[4];
#pragma unroll
              for (int r = 0; r < 4; ++r) {
                gv[r] = __ldcg(reinterpret_cast<const float4*>(pt + ((size_t)k * 128 + i4 + r) * Mp + t4));
                uv[r] = __ldcg(reinterpret_cast<const float4*>(pt + ((size_t)k * 128 + 64 + i4 + r) * Mp + t4));
              }
#pragma unroll
              for (int r = 0; r < 4; ++r) {
                if (k == 0) {
                  ga[r] = gv[r], ua[r] = uv[r];
                } else {
                  ga[r].x += gv[r].x, ga[r].y += gv[r].y, ga[r].z += gv[r].z, ga[r].w += gv[r].w;
                  ua[r].x += uv[r].x, ua[r].y += uv[r].y, ua[r].z += uv[r].z, ua[r].w += uv[r].w;
                }
              }
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int tok = t4 + j;
              if (tok >= M) break;
              float gq[4], uq[4];
#pragma unroll
              for (int r = 0; r < 4; ++r) {
                gq[r] = rbf(j == 0 ? ga[r].x : j == 1 ? ga[r].y : j == 2 ? ga[r].z : ga[r].w);
                uq[r] = rbf(j == 0 ? ua[r].x : j == 1 ? ua[r].y : j == 2 ? ua[r].z : ua[r].w);
              }
              uint2 o;
              o.x = pack_bf16(silu_fast(gq[0]) * uq[0], silu_fast(gq[1]) * uq[1]);
              o.y = pack_bf16(silu_fast(gq[2]) * uq[2], silu_fast(gq[3]) * uq[3]);
              *reinterpret_cast<uint2*>(Y + (size_t)tok * F + 64 * tile + i4) = o;
            }
          }
        } else {
          // this folder's 4-row groups [g0, g1) of 32; a thread folds a 4-row ×
          // 4-token block (4 float4 per contributor, rows are contiguous in
          // tokens), contributors in order (deterministic), then emits 4 tokens
          // × 4 consecutive outputs
          const int g0 = fi * 32 / nf, ng = (fi + 1) * 32 / nf - g0;
          const int nt4 = (M + 3) / 4;
          for (int e = wt; e < ng * nt4; e += kWorkerThreads) {
            const int gi = e / nt4, t4 = (e - gi * nt4) * 4, r4 = (g0 + gi) * 4;
            if (n0 + r4 >= N) continue;
            float4 acc[4];
            for (int k0 = 0; k0 < nc; k0 += 1) {
              float4 v[1][4];
#pragma unroll
              for (int k = 0; k < 1; ++k)
                if (k0 + k < nc)
#pragma unroll
                  for (int r = 0; r < 4; ++r)
                    v[k][r] = __ldcg(reinterpret_cast<const float4*>(pt + ((size_t)(k0 + k) * 128 + r4 + r) * Mp + t4));
#pragma unroll
              for (int k = 0; k < 1; ++k)
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                  if (k0 + k >= nc) continue;
                  if (k0 + k == 0) acc[r] = v[k][r];
                  else acc[r].x += v[k][r].x, acc[r].y += v[k][r].y, acc[r].z += v[k][r].z, acc[r].w += v[k][r].w;
                }
            }
            // acc[r] = rows r4 + r at tokens t4..t4+3 → per token the 4 rows
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int tok = t4 + j;
              if (tok >= M) break;
              const float4 o4 = j == 0 ? make_float4(acc[0].x, acc[1].x, acc[2].x, acc[3].x)
                              : j == 1 ? make_float4(acc[0].y, acc[1].y, acc[2].y, acc[3].y)
                              : j == 2 ? make_float4(acc[0].z, acc[1].z, acc[2].z, acc[3].z)
                                       : make_float4(acc[0].w, acc[1].w, acc[2].w, acc[3].w);
              if (T.epi == 1) {
                rope_quad_m(T, S, tok, n0 + r4, o4);
              } else {
                uint2 o;
                o.x = pack_bf16(o4.x, o4.y);
                o.y = pack_bf16(o4.z, o4.w);
                *reinterpret_cast<uint2*>(Y + (size_t)tok * N + n0 + r4) = o;
              }
            }
          }
        }
        named_bar(kBarW, kWorkerThreads);
        if (wt == 0) signal_done(done, t);
        if (lastp && wt == 0) stamp(g, t, R_EPI, 3);
      }
    }
    ++pc;
    u = pe;
  }
}

// a3 on one row with the worker threads: exactly add_rmsnorm_kernel's
// element mapping and reduction order (bitwise identical to it)
constexpr int kNormChunks = 4;
__device__ void norm_row(const Task& T, const Sm& S, int row) {
  const int tid = threadIdx.x - kW0 * 32;
  const int H = T.N, nch = H / 8;
  float* r = (float*)T.o1;
  const __nv_bfloat16* gamma = (const __nv_bfloat16*)T.a1;
  __nv_bfloat16* hout = (__nv_bfloat16*)T.o0;
  uint4 gm[kNormChunks];
#pragma unroll
  for (int c = 0; c < kNormChunks; ++c) {
    const int ch = tid + c * kWorkerThreads;
    if (ch < nch) gm[c] = reinterpret_cast<const uint4*>(gamma)[ch];
  }
  float v[kNormChunks][8];
  float ss = 0.f;
  float* rr = r + (size_t)row * H;
#pragma unroll
  for (int c = 0; c < kNormChunks; ++c) {
    const int ch = tid + c * kWorkerThreads;
    if (ch < nch) {
      const float4 a = __ldcg(reinterpret_cast<const float4*>(rr) + 2 * ch);
      const float4 b = __ldcg(reinterpret_cast<const float4*>(rr) + 2 * ch + 1);
      v[c][0] = a.x; v[c][1] = a.y; v[c][2] = a.z; v[c][3] = a.w;
      v[c][4] = b.x; v[c][5] = b.y; v[c][6] = b.z; v[c][7] = b.w;
      if (T.n_delta) {
        // (one delta — every decoder norm — stays in registers; more in index order)
        const uint4 d0 = __ldcg(reinterpret_cast<const uint4*>((const __nv_bfloat16*)T.dl[0] + (size_t)row * H) + ch);
        for (int i = 0; i < T.n_delta; ++i) {
          const uint4 d = i == 0 ? d0 : __ldcg(reinterpret_cast<const uint4*>((const __nv_bfloat16*)T.dl[i] + (size_t)row * H) + ch);
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
  ss = warp_sum(ss);
  if ((tid & 31) == 0) S.red[tid >> 5] = ss;
  named_bar(kBarW, kWorkerThreads);
  float tot = 0.f;
#pragma unroll
  for (int w = 0; w < kWorkers; ++w) tot += S.red[w];
  const float inv = rsqrtf(tot / (float)H + T.eps);
#pragma unroll
  for (int c = 0; c < kNormChunks; ++c) {
    const int ch = tid + c * kWorkerThreads;
    if (ch < nch) {
      const uint4 gg = gm[c];
      uint4 o;
      o.x = pack_bf16(v[c][0] * inv * bf16lo(gg.x), v[c][1] * inv * bf16hi(gg.x));
      o.y = pack_bf16(v[c][2] * inv * bf16lo(gg.y), v[c][3] * inv * bf16hi(gg.y));
      o.z = pack_bf16(v[c][4] * inv * bf16lo(gg.z), v[c][5] * inv * bf16hi(gg.z));
      o.w = pack_bf16(v[c][6] * inv * bf16lo(gg.w), v[c][7] * inv * bf16hi(gg.w));
      reinterpret_cast<uint4*>(hout)[(size_t)row * nch + ch] = o;
    }
  }
  named_bar(kBarW, kWorkerThreads);  // S.red reuse + every store before the release
}

// a5 on one (row, 8-head group) with 128 threads: rope_append_kernel's math
__device__ void rope_unit(const Task& T, int b, int y, int t128) {
  const int Hq = T.Hq, Hkv = T.Hkv, D = T.D, page = T.page, half = D / 2, G = Hq / Hkv;
  const int hh = y * 8 + (t128 >> 4), t16 = t128 & 15;
  const int n_rot = Hq + Hkv;
  const __nv_bfloat16* qkv = (const __nv_bfloat16*)T.a0;
  const int32_t* bt = (const int32_t*)T.a1;
  const int32_t* sl = (const int32_t*)T.a2;
  __nv_bfloat16* q_out = (__nv_bfloat16*)T.o0;
  __nv_bfloat16* kc = (__nv_bfloat16*)T.o1;
  __nv_bfloat16* vc = (__nv_bfloat16*)T.o2;
  if (hh < n_rot && t16 * 8 < half) {
    const int i0 = t16 * 8;
    const int pos = __ldg(sl + b) - 1;
    const __nv_bfloat16* src = qkv + (size_t)b * (Hq + 2 * Hkv) * D;
    const __nv_bfloat16* x;
    __nv_bfloat16* dst;
    if (hh < Hq) {
      const int g = hh / G, j = hh % G;
      x = src + (size_t)g * (G + 2) * D + (size_t)j * D;
      dst = q_out + (size_t)b * Hq * D + (size_t)hh * D;
    } else {
      const int g = hh - Hq, slot = pos - T.slot_offset;
      const int32_t pg = __ldg(bt + (size_t)b * T.pps + slot / page);
      x = src + (size_t)g * (G + 2) * D + (size_t)G * D;
      dst = kc + (((size_t)pg * Hkv + g) * page + slot % page) * D;
    }
    const uint4 xa = __ldcg(reinterpret_cast<const uint4*>(x + i0));
    const uint4 xb = __ldcg(reinterpret_cast<const uint4*>(x + half + i0));
    float cs[8], sn[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double ang = (double)pos * T.freq[i0 + k];
      const double kk = rint(ang * 0.15915494309189535);
      const double red = fma(-kk, 6.283185307179586, fma(-kk, 2.4492935982947064e-16, ang));
      sincosf((float)red, &sn[k], &cs[k]);
    }
    const uint32_t* pa = &xa.x;
    const uint32_t* pb = &xb.x;
    uint4 lo, hi;
    uint32_t* plo = &lo.x;
    uint32_t* phi = &hi.x;
#pragma unroll
    for (int qq = 0; qq < 4; ++qq) {
      const float x0 = bf16lo(pa[qq]), x1 = bf16hi(pa[qq]), y0 = bf16lo(pb[qq]), y1 = bf16hi(pb[qq]);
      const float c0 = cs[2 * qq], c1 = cs[2 * qq + 1], s0 = sn[2 * qq], s1 = sn[2 * qq + 1];
      plo[qq] = pack_bf16(x0 * c0 - y0 * s0, x1 * c1 - y1 * s1);
      phi[qq] = pack_bf16(y0 * c0 + x0 * s0, y1 * c1 + x1 * s1);
    }
    *reinterpret_cast<uint4*>(dst + i0) = lo;
    *reinterpret_cast<uint4*>(dst + half + i0) = hi;
  } else if (hh >= n_rot && hh < n_rot + Hkv) {
    const int g = hh - n_rot;
    const int slot = __ldg(sl + b) - 1 - T.slot_offset;
    const int32_t pg = __ldg(bt + (size_t)b * T.pps + slot / page);
    const __nv_bfloat16* x = qkv + (size_t)b * (Hq + 2 * Hkv) * D + (size_t)g * (G + 2) * D + (size_t)(G + 1) * D;
    __nv_bfloat16* dst = vc + (((size_t)pg * Hkv + g) * page + slot % page) * D;
    for (int c8 = t16 * 8; c8 < D; c8 += 128)
      *reinterpret_cast<uint4*>(dst + c8) = __ldcg(reinterpret_cast<const uint4*>(x + c8));
  }
}

// attention consumers (worker w): pages t ≡ w (mod 8) of every item, slot (base + t) mod A
template <int D>
__device__ void cons_attn(const Task& T, const Sm& S, const Geo& g, unsigned* err, unsigned& ak, unsigned& ci,
                          int& apos, uint32_t& apar) {
  constexpr int KS = D / 16;
  constexpr int SLAB_B = kPage * D * 2;
  const int lane = threadIdx.x & 31, w = (threadIdx.x >> 5) - kW0;
  const int gid = lane >> 2, c4 = lane & 3;
  const int mi = lane >> 3, r8 = lane & 7;
  const int k_tok = ((mi & 1) << 3) + r8, k_dc = mi >> 1;
  const int v_tok = ((mi >> 1) << 3) + r8, v_dc = mi & 1;
  const int Gq = T.G, A = g.A;
  const float scale = T.scale_log2;
  const int32_t* sl = (const int32_t*)T.a2;
  for (;;) {
    const int is = (int)(ak & 3u);
    mwait_sleep(&S.ifull[is], (ak >> 2) & 1u, err, S);
    const int it = S.s_item[is];
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.iempty[is]);
    ++ak;
    if (it < 0) break;
    const int split = it % T.splits, b = (it / T.splits) % T.rows;
    const int len = __ldg(sl + b) - T.slot_offset;
    const int p0 = split * T.pps_split;
    const int np = max(0, min((len + kPage - 1) / kPage, p0 + T.pps_split) - p0);
    int base = (apos + 7) / 8 * 8;
    if (base >= A) base -= A;
    uint32_t qb[KS][2];
    {
      const int qs = (int)(ci & 1u);
      mwait(&S.qfull[qs], (ci >> 1) & 1u, err, S);
      const uint32_t* qh = reinterpret_cast<const uint32_t*>(S.qsm + (size_t)qs * g.Gm * D + gid * D);
#pragma unroll
      for (int s = 0; s < KS; ++s) {
        qb[s][0] = gid < Gq ? qh[8 * s + c4] : 0u;
        qb[s][1] = gid < Gq ? qh[8 * s + 4 + c4] : 0u;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.qempty[qs]);
    }
    float o[KS][4];
#pragma unroll
    for (int j = 0; j < KS; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
    float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};
    int st = base + w;
    if (st >= A) st -= A;
    for (int j = w; j < np; j += kWorkers, st = st + kWorkers >= A ? st + kWorkers - A : st + kWorkers) {
      const uint32_t bit = 1u << (st >> 3);
      mwait(&S.afull[st], (apar & bit) ? 1u : 0u, err, S);
      apar ^= bit;
      if (g.dbg) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.aempty[st]);
        continue;
      }
      uint8_t* slot = S.arena + (size_t)st * kSlot;
      const uint32_t kt = smem_u32(slot), vt = kt + SLAB_B;
      const int tok0 = (p0 + j) * kPage;
      const int valid = min(kPage, len - tok0);
      if (valid < kPage) {  // zero the V rows past the end (0·garbage must not be NaN)
        uint4* vrow = reinterpret_cast<uint4*>(slot + SLAB_B + valid * D * 2);
        for (int e = lane; e < (kPage - valid) * D / 8; e += 32) vrow[e] = make_uint4(0, 0, 0, 0);
        __syncwarp();
      }
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
      float sv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) sv[i] = (sa[i] + sb[i]) * scale;
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
      const uint32_t pb0 = movm_t(pack_bf16(p0v, p1v));
      const uint32_t pb1 = movm_t(pack_bf16(p2v, p3v));
#pragma unroll
      for (int mb = 0; mb < KS; ++mb) {
        uint32_t a0, a1, a2, a3;
        ldsm_x4_t(vt + tile_off<D>(mb >> 2, v_tok, ((mb & 3) << 1) + v_dc), a0, a1, a2, a3);
        mma16816(o[mb], a0, a1, a2, a3, pb0, pb1);
      }
      // (the zeroing stores above were generic-proxy writes into a slot the
      // TMA overwrites next: order them before the release)
      if (valid < kPage) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.aempty[st]);
    }
    apos = (base + np) % A;  // (once per item)
#pragma unroll
    for (int x = 4; x < 32; x <<= 1) {
      l_run[0] += __shfl_xor_sync(0xffffffffu, l_run[0], x);
      l_run[1] += __shfl_xor_sync(0xffffffffu, l_run[1], x);
    }
    if (ci >= 1) mwait_sleep(&S.cempty[(ci - 1u) & 1u], ((ci - 1u) >> 1) & 1u, err, S);
    float* cw = S.comb + (size_t)w * g.Gm * D;
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int h = 2 * c4 + hh;
      if (h < Gq) {
#pragma unroll
        for (int mb = 0; mb < KS; ++mb) {
          cw[h * D + 16 * mb + gid] = o[mb][hh];
          cw[h * D + 16 * mb + gid + 8] = o[mb][2 + hh];
        }
        if (gid == 0) {
          S.comb_ml[(w * g.Gm + h) * 2 + 0] = m_run[hh];
          S.comb_ml[(w * g.Gm + h) * 2 + 1] = l_run[hh];
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.cfull[ci & 1u]);
    ++ci;
  }
}

// attention merge warp: 8 warp states (fixed order) → output or split partial;
// the last split of a (sequence, kv head) unit merges the splits (fixed order)
// two merge warps (the MMA warp is idle during attention): item ci is merged
// by warp ci mod 2, so one item's split handling (stores, fences, the arrival
// atomic, the last split's merge) overlaps the next item's merge
__device__ void merge_attn(const Task& T, int t, const Sm& S0, const Geo& g, unsigned* done, unsigned ep, unsigned* err,
                           unsigned& ak, unsigned& ci, int sub) {
  Sm S = S0;  // this merge warp's own scratch
  S.s_w += sub * (kWorkers * kMaxG + 2 * kMaxG + kFastSplitLse);
  S.s_M += sub * (kWorkers * kMaxG + 2 * kMaxG + kFastSplitLse);
  S.s_L += sub * (kWorkers * kMaxG + 2 * kMaxG + kFastSplitLse);
  S.s_lse += sub * (kWorkers * kMaxG + 2 * kMaxG + kFastSplitLse);
  const int lane = threadIdx.x & 31;
  const int Gq = T.G, D = T.D;
  __nv_bfloat16* out = (__nv_bfloat16*)T.o0;
  const bool single = T.splits == 1;
  for (;;) {
    const int is = (int)(ak & 3u);
    mwait_sleep(&S.ifull[is], (ak >> 2) & 1u, err, S);
    const int it = S.s_item[is];
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.iempty[is]);
    ++ak;
    if (it < 0) break;
    if ((int)(ci & 1u) != sub) {  // the other merge warp's item
      ++ci;
      continue;
    }
    const int split = it % T.splits, unit = it / T.splits;
    const int gh = unit / T.rows, b = unit % T.rows;
    mwait_sleep(&S.cfull[ci & 1u], (ci >> 1) & 1u, err, S);
    for (int x = lane; x < kWorkers * Gq; x += 32) {
      const int w = x / Gq, h = x % Gq;
      float M = -INFINITY;
      for (int x = 0; x < kWorkers; ++x) M = fmaxf(M, S.comb_ml[(x * g.Gm + h) * 2]);
      const float Mu = (M == -INFINITY) ? 0.f : M;
      float L = 0.f;
      for (int x = 0; x < kWorkers; ++x) L += exp2f(S.comb_ml[(x * g.Gm + h) * 2] - Mu) * S.comb_ml[(x * g.Gm + h) * 2 + 1];
      S.s_w[w * kMaxG + h] = exp2f(S.comb_ml[(w * g.Gm + h) * 2] - Mu);
      if (w == 0) S.s_M[h] = M, S.s_L[h] = L;
    }
    __syncwarp();
    for (int e4 = lane; e4 < Gq * D / 4; e4 += 32) {
      const int h = (e4 * 4) / D, d0 = (e4 * 4) % D;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int w = 0; w < kWorkers; ++w) {
        const float sc = S.s_w[w * kMaxG + h];
        const float4 v = *reinterpret_cast<const float4*>(S.comb + ((size_t)w * g.Gm + h) * D + d0);
        acc.x += sc * v.x, acc.y += sc * v.y, acc.z += sc * v.z, acc.w += sc * v.w;
      }
      const float L = S.s_L[h];
      const float inv = L > 0.f ? 1.f / L : 0.f;
      acc.x *= inv, acc.y *= inv, acc.z *= inv, acc.w *= inv;
      if (single) {
        uint2 pk;
        pk.x = pack_bf16(acc.x, acc.y);
        pk.y = pack_bf16(acc.z, acc.w);
        *reinterpret_cast<uint2*>(out + (size_t)b * T.Hq * D + (size_t)(gh * Gq + h) * D + d0) = pk;
      } else {
        const size_t pi = (((size_t)unit * T.splits + split) * Gq + h);
        *reinterpret_cast<float4*>(T.part + pi * D + d0) = acc;
        if (d0 == 0) T.part_lse[pi] = L > 0.f ? S.s_M[h] + log2f(L) : -INFINITY;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.cempty[ci & 1u]);
    ++ci;
    bool fin = single;
    if (!single) {
      fence_acq_rel_gpu();  // every lane: its partial stores before lane 0's release
      __syncwarp();
      unsigned prev = 0;
      if (lane == 0) prev = atom_add_acq_rel_gpu(T.ctr + unit, 1u);
      fin = __shfl_sync(0xffffffffu, prev, 0) + 1u == (ep + 1u) * (unsigned)T.splits;
      if (fin) {
        fence_acq_rel_gpu();
        const float* lse = T.part_lse + (size_t)unit * T.splits * Gq;
        const float* po = T.part + (size_t)unit * T.splits * Gq * D;
        const int nl = T.splits * Gq;
        if (nl <= kFastSplitLse) {
          for (int i = lane; i < nl; i += 32) S.s_lse[i] = __ldcg(lse + i);
          __syncwarp();
          if (lane < Gq) {
            float M = -INFINITY;
            for (int sp = 0; sp < T.splits; ++sp) M = fmaxf(M, S.s_lse[sp * Gq + lane]);
            const float Mu = (M == -INFINITY) ? 0.f : M;
            float L = 0.f;
            for (int sp = 0; sp < T.splits; ++sp) L += exp2f(S.s_lse[sp * Gq + lane] - Mu);
            S.s_M[lane] = Mu, S.s_L[lane] = L;
          }
          __syncwarp();
          for (int e4 = lane; e4 < Gq * D / 4; e4 += 32) {
            const int h = (e4 * 4) / D, d0 = (e4 * 4) % D;
            const float Mu = S.s_M[h];
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            int sp = 0;
            for (; sp + kFastSplits <= T.splits; sp += kFastSplits) {
              float4 v[kFastSplits];
#pragma unroll
              for (int u = 0; u < kFastSplits; ++u)
                v[u] = __ldcg(reinterpret_cast<const float4*>(po + ((size_t)(sp + u) * Gq + h) * D + d0));
#pragma unroll
              for (int u = 0; u < kFastSplits; ++u) {
                const float sc = exp2f(S.s_lse[(sp + u) * Gq + h] - Mu);
                acc.x += sc * v[u].x, acc.y += sc * v[u].y, acc.z += sc * v[u].z, acc.w += sc * v[u].w;
              }
            }
            for (; sp < T.splits; ++sp) {
              const float sc = exp2f(S.s_lse[sp * Gq + h] - Mu);
              const float4 v = __ldcg(reinterpret_cast<const float4*>(po + ((size_t)sp * Gq + h) * D + d0));
              acc.x += sc * v.x, acc.y += sc * v.y, acc.z += sc * v.z, acc.w += sc * v.w;
            }
            const float L = S.s_L[h];
            const float inv = L > 0.f ? 1.f / L : 0.f;
            acc.x *= inv, acc.y *= inv, acc.z *= inv, acc.w *= inv;
            uint2 pk;
            pk.x = pack_bf16(acc.x, acc.y);
            pk.y = pack_bf16(acc.z, acc.w);
            *reinterpret_cast<uint2*>(out + (size_t)b * T.Hq * D + (size_t)(gh * Gq + h) * D + d0) = pk;
          }
        } else {
          if (lane == 0) report(S, err, 6u, 0u, 0u);  // host guarantees splits·G ≤ kFastSplitLse
        }
      }
    }
    if (fin) {
      fence_acq_rel_gpu();
      __syncwarp();
      if (lane == 0) red_rel_gpu(done + t, 1u);
    }
  }
}

// ================================================================== the kernel
template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    mega_kernel(const Task* __restrict__ tasks, const __grid_constant__ Geo g, uint8_t* __restrict__ ctrl,
                unsigned* __restrict__ done, unsigned* __restrict__ err) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  Sm S;
  S.arena = smem;
  S.qsm = (__nv_bfloat16*)(smem + g.off_q);
  S.comb = (float*)(smem + g.off_comb);
  S.comb_ml = (float*)(smem + g.off_ml);
  uint64_t* bars = (uint64_t*)(smem + g.off_bar);
  S.gfull = bars;
  S.gempty = S.gfull + kMaxStages;
  S.afull = S.gempty + kMaxStages;
  S.aempty = S.afull + kMaxSlots;
  S.tfull = S.aempty + kMaxSlots;
  S.tempty = S.tfull + 2;
  S.qfull = S.tempty + 2;
  S.qempty = S.qfull + 2;
  S.ifull = S.qempty + 2;
  S.iempty = S.ifull + 4;
  S.cfull = S.iempty + 4;
  S.cempty = S.cfull + 2;
  S.xg = S.cempty + 2;
  S.xa = S.xg + 1;
  uint8_t* misc = smem + g.off_misc;
  S.s_item = (int*)misc;                      // 16 B
  S.bcast = (unsigned*)(misc + 16);           // 16 B
  S.red = (float*)(misc + 32);                // 32 B
  S.tmem_slot = (uint32_t*)(misc + 64);       // 16 B
  S.s_len = (int*)(misc + 80);                // 16 B (+16 spare)
  __shared__ int s_rpos[128], s_rpg[128];     // fused RoPE fold: per-token position and page
  S.rpos = s_rpos;
  S.rpg = s_rpg;
  S.s_w = (float*)(misc + 112);               // [8][8]
  S.s_M = S.s_w + kWorkers * kMaxG;           // [8]
  S.s_L = S.s_M + kMaxG;                      // [8]
  S.s_lse = S.s_L + kMaxG;                    // [128]
  __shared__ unsigned s_ep;
  __shared__ int s_cur[kWarps];
  S.cur = s_cur;
  S.abortp = (unsigned*)(ctrl + 8);
  S.rec = (unsigned*)(ctrl + 16);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kMaxStages; ++i) mbar_init(&S.gfull[i], 1), mbar_init(&S.gempty[i], 1);
    for (int i = 0; i < kMaxSlots; ++i) mbar_init(&S.afull[i], 1), mbar_init(&S.aempty[i], 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&S.tfull[i], 1);
      mbar_init(&S.tempty[i], kWorkers);
      mbar_init(&S.qfull[i], 1);
      mbar_init(&S.qempty[i], kWorkers);
    }
    for (int i = 0; i < 4; ++i) mbar_init(&S.ifull[i], 1), mbar_init(&S.iempty[i], kWorkers + 3);
    mbar_init(S.xg, 1);
    mbar_init(S.xa, 1);
    for (int i = 0; i < 2; ++i) mbar_init(&S.cfull[i], kWorkers), mbar_init(&S.cempty[i], 1);
    for (int w = 0; w < kWarps; ++w) s_cur[w] = -1;
    s_ep = *(volatile unsigned*)ctrl;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMma) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(S.tmem_slot)),
                 "r"(2 * kAccCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *S.tmem_slot;
  const unsigned ep = s_ep;
  const int Gr = (int)gridDim.x, c = blockIdx.x;
  if (g.n_tab) {
    // this step's RoPE (cos, sin) tables: entry e of the concatenated tables is
    // computed by CTA e mod grid — rope_append_kernel's arithmetic (fp64 angle,
    // reduced to [−π, π], fp32 sincos of the reduced angle)
    int base = 0;
    for (int i = 0; i < g.n_tab; ++i) {
      const int n = g.tab_rows[i] * g.tab_half[i];
      for (int e = base + c + Gr * (int)threadIdx.x; e < base + n; e += Gr * kThreads) {
        const int le = e - base, row = le / g.tab_half[i], p = le - row * g.tab_half[i];
        const int pos = __ldg(g.tab_sl[i] + row) - 1;
        const double ang = (double)pos * g.tab_freq[i][p];
        const double k = rint(ang * 0.15915494309189535);
        const double red = fma(-k, 6.283185307179586, fma(-k, 2.4492935982947064e-16, ang));
        float sn, cs;
        sincosf((float)red, &sn, &cs);
        g.tab[i][le] = make_float2(cs, sn);
      }
      base += n;
    }
    __syncthreads();
    if (threadIdx.x == 0) signal_done(g.tab_ready, 0);
  }

  // role state (each role keeps only its own; all advance identically)
  unsigned gs = 0, pc = 0, ak = 0, ci = 0;
  int apos = 0;
  uint32_t apar = 0;
  Ld ld;
  unsigned nattn = 0, xa_seen = 0;
  if (warp == kLoader) {
    for (int t = 0; t < g.n_tasks; ++t) {
      const Task& T = tasks[t];
      if (lane == 0) s_cur[warp] = t, stamp(g, t, R_LOAD, 0);
      if (lane == 0 && g.pf && (T.kind == MK_GEMM || T.kind == MK_ATTN)) {
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&T.tm0) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&T.tm1) : "memory");
      }
      if (T.kind == MK_GEMM) load_gemm(T, t, S, g, done, ep, err, ld, nattn, xa_seen);
      else if (T.kind == MK_ATTN) load_attn<true>(T, t, S, g, done, ep, err, ak, ci, ld, nattn, &xa_seen);
      __syncwarp();
      if (lane == 0) stamp(g, t, R_LOAD, 2);
    }
  } else if (warp == kMma) {
    for (int t = 0; t < g.n_tasks; ++t) {
      const Task& T = tasks[t];
      if (lane == 0) s_cur[warp] = t, stamp(g, t, R_MMA, 0);
      if (T.kind == MK_GEMM) mma_gemm(T, t, S, g, tmem, err, gs, pc);
      else if (T.kind == MK_ATTN) merge_attn(T, t, S, g, done, ep, err, ak, ci, 1);
      if (lane == 0) stamp(g, t, R_MMA, 2);
    }
  } else if (warp == kLoader2) {
    for (int t = 0; t < g.n_tasks; ++t) {
      const Task& T = tasks[t];
      if (lane == 0) s_cur[warp] = t;
      if (T.kind == MK_ATTN) load_attn<false>(T, t, S, g, done, ep, err, ak, ci, ld, nattn, nullptr);
    }
  } else if (warp == kMerge) {
    for (int t = 0; t < g.n_tasks; ++t) {
      const Task& T = tasks[t];
      if (lane == 0) s_cur[warp] = t, stamp(g, t, R_MERGE, 0);
      if (T.kind == MK_ATTN) merge_attn(T, t, S, g, done, ep, err, ak, ci, 0);
      if (lane == 0) stamp(g, t, R_MERGE, 2);
    }
  } else if (warp >= kW0) {
    const int wt = threadIdx.x - kW0 * 32;
    for (int t = 0; t < g.n_tasks; ++t) {
      const Task& T = tasks[t];
      if (lane == 0) s_cur[warp] = t;
      if (wt == 0) stamp(g, t, R_WORK, 0);
      switch (T.kind) {
        case MK_GEMM: epi_gemm(T, t, S, g, done, ep, tmem, err, pc, g.tab_ready); break;
        case MK_ATTN: cons_attn<D>(T, S, g, err, ak, ci, apos, apar); break;
        case MK_NORM:
        case MK_SILU:
        case MK_RESID: {
          bool waited = false;
          unsigned nu = 0;
          const int first = ((c - T.rot) % Gr + Gr) % Gr;
          for (int u = first; u < T.n_units; u += Gr, ++nu) {
            if (!waited) {
              if (wt == 0) deps_wait(T, done, ep, err, S), stamp(g, t, R_WORK, 1);
              named_bar(kBarW, kWorkerThreads);
              waited = true;
            }
            if (T.kind == MK_NORM) {
              norm_row(T, S, u);
            } else if (T.kind == MK_SILU) {
              const size_t n = (size_t)T.M * (T.N / 8);
              const size_t e8 = (size_t)u * kWorkerThreads + wt;
              if (e8 < n) {
                const int F = T.N;
                const size_t row = e8 / (F / 8), i8 = e8 % (F / 8);
                const int j = (int)(i8 / 8), i = (int)(i8 % 8) * 8;
                const __nv_bfloat16* gp = (const __nv_bfloat16*)T.a0 + row * 2 * F + 128 * j + i;
                const uint4 gv = __ldcg(reinterpret_cast<const uint4*>(gp));
                const uint4 uv = __ldcg(reinterpret_cast<const uint4*>(gp + 64));
                const uint32_t* gq = &gv.x;
                const uint32_t* uq = &uv.x;
                uint4 o;
                uint32_t* op = &o.x;
#pragma unroll
                for (int qq = 0; qq < 4; ++qq) {
                  const float g0 = bf16lo(gq[qq]), g1 = bf16hi(gq[qq]);
                  op[qq] = pack_bf16(silu_fast(g0) * bf16lo(uq[qq]), silu_fast(g1) * bf16hi(uq[qq]));
                }
                reinterpret_cast<uint4*>(T.o0)[e8] = o;
              }
              named_bar(kBarW, kWorkerThreads);
            } else {  // residual add
              const size_t i = (size_t)u * kWorkerThreads + wt;
              if (i < (size_t)T.K) {
                float* r = (float*)T.o0;
                float4 a = __ldcg(reinterpret_cast<const float4*>(r) + 2 * i);
                float4 b = __ldcg(reinterpret_cast<const float4*>(r) + 2 * i + 1);
                for (int k = 0; k < T.n_delta; ++k) {
                  const uint4 x = __ldcg(reinterpret_cast<const uint4*>(T.dl[k]) + i);
                  a.x += bf16lo(x.x); a.y += bf16hi(x.x); a.z += bf16lo(x.y); a.w += bf16hi(x.y);
                  b.x += bf16lo(x.z); b.y += bf16hi(x.z); b.z += bf16lo(x.w); b.w += bf16hi(x.w);
                }
                reinterpret_cast<float4*>(r)[2 * i] = a;
                reinterpret_cast<float4*>(r)[2 * i + 1] = b;
              }
              named_bar(kBarW, kWorkerThreads);
            }
          }
          // one release for all of this CTA's units (every unit ended in a worker barrier)
          if (nu && wt == 0) signal_done(done, t, nu);
          break;
        }
        case MK_ROPE: {
          // two 128-thread halves, units alternate between them
          const int hf = wt >> 7, t128 = wt & 127;
          const int ny = (T.Hq + 2 * T.Hkv + 7) / 8;
          bool waited = false;
          unsigned nu = 0;
          const int first = ((c - T.rot) % Gr + Gr) % Gr;
          int k = 0;
          for (int u = first; u < T.n_units; u += Gr, ++k) {
            if ((k & 1) != hf) continue;
            ++nu;
            if (!waited) {
              if (t128 == 0) deps_wait(T, done, ep, err, S), stamp(g, t, R_WORK, 1);
              named_bar(kBarHalf0 + hf, 128);
              waited = true;
            }
            rope_unit(T, u / ny, u % ny, t128);
            named_bar(kBarHalf0 + hf, 128);
          }
          if (nu && t128 == 0) signal_done(done, t, nu);
          break;
        }
        default: break;
      }
      if (wt == 0) stamp(g, t, R_WORK, 2);
    }
  }
  // ---- end of step: every role is done; the last CTA out advances the epoch
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == kMma) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * kAccCols));
  }
  if (threadIdx.x == 0) {
    fence_acq_rel_gpu();
    unsigned* ex = (unsigned*)(ctrl + 4);
    const unsigned prev = atom_add_acq_rel_gpu(ex, 1u);
    if (prev + 1u == (ep + 1u) * (unsigned)Gr) {
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"((unsigned*)ctrl), "r"(ep + 1u) : "memory");
    }
  }
}

}  // namespace mega

// ================================================================== host side
struct MegaPlan {
  std::vector<mega::Task> tasks;
  mega::Geo geo{};
  int D = 0;
  size_t smem = 0;
  int grid = 0;
  // workspace layout (bytes)
  uint64_t off_ctrl = 0, off_done = 0, off_tick = 0, off_ctr = 0, off_freq = 0, off_tasks = 0, off_gpart = 0,
           off_apart = 0, total = 0;
  uint64_t gpart_bytes = 0, apart_bytes = 0;
  std::vector<uint64_t> ctr_off;  // per task: offset of its counters within the counter region
  std::vector<int> gpar, apar;    // scratch parity per task (-1 none)
  std::vector<double> freq;       // concatenated RoPE tables
  std::vector<int> freq_off;      // per task (doubles)
  struct Tab {
    const void* sl;
    int rows, half;
    double theta;
    int freq_off;      // its θ^(−2i/D) in freq
    uint64_t off;      // byte offset of its (cos, sin) table in the workspace
  };
  std::vector<Tab> tabs;
  std::vector<int> tab_of;        // per task (-1 none)
  uint64_t off_tab = 0;
  std::vector<MegaOpDesc> ops;
  uint8_t* ws = nullptr;
  unsigned* err = nullptr;
  bool bound = false;
  unsigned long long* trace = nullptr;
};

namespace {

struct Range {
  uintptr_t a, b;
};
bool overlap(const std::vector<Range>& x, const std::vector<Range>& y) {
  for (const auto& p : x)
    for (const auto& q : y)
      if (p.a < q.b && q.a < p.b) return true;
  return false;
}

template <typename T>
T get_attr(const MegaOpDesc& o) {
  T a;
  std::memcpy(&a, o.attrs.data(), sizeof(T));
  return a;
}

}  // namespace

kd_status mega_create(const std::vector<MegaOpDesc>& ops, MegaPlan** out, uint64_t* ws_bytes) {
  using namespace mega;
  int dev = 0;
  KD_CUDA_CHECK(cudaGetDevice(&dev), "cudaGetDevice");
  int sms = 0;
  KD_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "SM count");
  auto* P = new MegaPlan();
  P->ops = ops;
  P->grid = sms;
  const int n = (int)ops.size();
  if (n == 0) {
    delete P;
    return fail(KD_ERR_INVALID_ARG, "megakernel: empty schedule");
  }
  P->tasks.resize(n);
  P->ctr_off.assign(n, 0);
  P->gpar.assign(n, -1);
  P->apar.assign(n, -1);
  P->freq_off.assign(n, -1);
  P->tab_of.assign(n, -1);
  int D = 0, Gm = 1, maxM = 0;
  uint64_t ctr_words = 0;
  int last_g[2] = {-1, -1}, last_a[2] = {-1, -1}, ng = 0, na = 0;
  std::vector<std::vector<int>> extra(n);  // scratch-reuse guards
  auto bad = [&](const std::string& m) {
    delete P;
    return fail(KD_ERR_UNSUPPORTED, "megakernel: " + m);
  };
  int rot = 0;
  for (int t = 0; t < n; ++t) {
    const MegaOpDesc& o = ops[t];
    Task& T = P->tasks[t];
    std::memset(&T, 0, sizeof(T));
    T.rot = rot % sms;
    switch (o.op) {
      case KD_OP_ADD_RMSNORM: {
        auto a = get_attr<kd_attr_add_rmsnorm>(o);
        if (a.dtype != KD_BF16 || a.hidden % 8 || a.hidden > 8 * kWorkerThreads * kNormChunks) return bad("add_rmsnorm shape/dtype");
        T.kind = MK_NORM;
        T.M = a.rows, T.N = a.hidden, T.eps = a.eps;
        T.n_delta = a.n_delta;
        for (uint32_t i = 0; i < a.n_delta; ++i) T.dl[i] = o.rd[1 + i];
        T.a1 = o.rd[1 + a.n_delta];
        T.o0 = o.wr[0];
        T.o1 = o.wr[1];
        T.n_units = a.rows;
        T.done_units = a.rows;
        break;
      }
      case KD_OP_RESIDUAL_ADD: {
        auto a = get_attr<kd_attr_residual_add>(o);
        if (a.dtype != KD_BF16 || a.hidden % 8) return bad("residual_add shape/dtype");
        T.kind = MK_RESID;
        T.K = (int)((uint64_t)a.rows * a.hidden / 8);
        T.n_delta = a.n_delta;
        for (uint32_t i = 0; i < a.n_delta; ++i) T.dl[i] = o.rd[1 + i];
        T.o0 = o.wr[0];
        T.n_units = (T.K + kWorkerThreads - 1) / kWorkerThreads;
        T.done_units = T.n_units;
        break;
      }
      case KD_OP_SILU_MUL: {
        auto a = get_attr<kd_attr_silu_mul>(o);
        if (a.dtype != KD_BF16 || a.ffn % 64) return bad("silu_mul shape/dtype");
        T.kind = MK_SILU;
        T.M = a.rows, T.N = a.ffn;
        T.a0 = o.rd[0];
        T.o0 = o.wr[0];
        const uint64_t n8 = (uint64_t)a.rows * a.ffn / 8;
        T.n_units = (int)((n8 + kWorkerThreads - 1) / kWorkerThreads);
        T.done_units = T.n_units;
        break;
      }
      case KD_OP_ROPE_APPEND: {
        auto a = get_attr<kd_attr_rope_append>(o);
        if (a.dtype != KD_BF16 || a.head_dim % 16 || a.head_dim > 256 || a.n_heads % a.n_kv_heads)
          return bad("rope_append shape/dtype");
        T.kind = MK_ROPE;
        T.Hq = a.n_heads, T.Hkv = a.n_kv_heads, T.D = a.head_dim, T.page = a.page, T.pps = a.pages_per_seq;
        T.slot_offset = a.slot_offset;
        T.a0 = o.rd[0], T.a1 = o.rd[1], T.a2 = o.rd[2];
        T.o0 = o.wr[0], T.o1 = o.wr[1], T.o2 = o.wr[2];
        const int ny = (int)((a.n_heads + 2 * a.n_kv_heads + 7) / 8);
        T.n_units = a.rows * ny;
        T.done_units = T.n_units;
        P->freq_off[t] = (int)P->freq.size();
        const double l2t = std::log2(a.theta);
        for (uint32_t i = 0; i < a.head_dim / 2; ++i) P->freq.push_back(std::exp2(-2.0 * (double)i / (double)a.head_dim * l2t));
        break;
      }
      case KD_OP_GEMM:
      case KD_OP_GEMM_SILU:
      case KD_OP_QKV_ROPE: {
        kd_attr_gemm a{};
        if (o.op == KD_OP_QKV_ROPE) {
          auto r = get_attr<kd_attr_qkv_rope>(o);
          if (r.head_dim % 4 || 128 % r.head_dim || r.n_heads % r.n_kv_heads) return bad("QKV+RoPE head shape");
          a.M = r.rows, a.N = (r.n_heads + 2 * r.n_kv_heads) * r.head_dim, a.K = r.hidden, a.dtype = r.dtype;
          T.epi = 1;
          T.Hq = r.n_heads, T.Hkv = r.n_kv_heads, T.D = r.head_dim, T.page = r.page, T.pps = r.pages_per_seq;
          {  // one (cos, sin) table per distinct (seq_len buffer, rows, D/2, θ)
            int ti = -1;
            for (int i = 0; i < (int)P->tabs.size(); ++i)
              if (P->tabs[i].sl == o.rd[3] && P->tabs[i].rows == (int)r.rows && P->tabs[i].half == (int)r.head_dim / 2 &&
                  P->tabs[i].theta == r.theta)
                ti = i;
            if (ti < 0) {
              if (P->tabs.size() == 4) return bad("more than 4 distinct RoPE position sets");
              P->tabs.push_back({o.rd[3], (int)r.rows, (int)r.head_dim / 2, r.theta, (int)P->freq.size(), 0});
              ti = (int)P->tabs.size() - 1;
            }
            P->tab_of[t] = ti;
          }
          P->freq_off[t] = (int)P->freq.size();
          const double l2t = std::log2(r.theta);
          for (uint32_t i = 0; i < r.head_dim / 2; ++i)
            P->freq.push_back(std::exp2(-2.0 * (double)i / (double)r.head_dim * l2t));
        } else {
          a = get_attr<kd_attr_gemm>(o);
          T.epi = o.op == KD_OP_GEMM_SILU ? 2 : 0;
        }
        if (a.dtype != KD_BF16) return bad("fp32 GEMM");
        if (a.M == 0 || a.M > 128 || a.K % 128 || a.N % 8) return bad("GEMM shape (M <= 128, K % 128 == 0, N % 8 == 0)");
        T.kind = MK_GEMM;
        T.M = a.M, T.N = a.N, T.K = a.K;
        T.mma_n = (a.M + 15) / 16 * 16;
        T.kbs = 2;
        T.KB = a.K / 128;
        T.tiles = (a.N + 127) / 128;
        const long long U = (long long)T.tiles * T.KB;
        T.gg = (int)std::min<long long>(sms, U);
        int maxc = 0;
        for (int tl = 0; tl < T.tiles; ++tl)
          maxc = std::max(maxc, (int)(uowner((long long)(tl + 1) * T.KB - 1, U, T.gg) - uowner((long long)tl * T.KB, U, T.gg) + 1));
        T.maxc = maxc;
        T.n_units = (int)U;
        {  // completion units: one per tile slice (a whole tile or a folder's share of a split tile)
          unsigned units = 0;
          for (int tl = 0; tl < T.tiles; ++tl) {
            const long long tb = (long long)tl * T.KB, te = tb + T.KB;
            const int f = (int)uowner(tb, U, T.gg), l = (int)uowner(te - 1, U, T.gg);
            const int nc = l - f + 1;
            units += nc == 1 ? 1u : (unsigned)((l - f) + (ubeg(l + 1, U, T.gg) == te ? 1 : 0));
          }
          T.done_units = units;
        }
        T.a0 = o.rd[0];  // X
        T.a1 = o.rd[1];  // W
        T.o0 = o.wr[0];
        if (T.epi == 1) {
          T.ctr2 = o.rd[2];  // block table
          T.a2 = o.rd[3];    // seq_len
          T.o1 = o.wr[1];
          T.o2 = o.wr[2];
        }
        maxM = std::max(maxM, T.mma_n);
        P->ctr_off[t] = ctr_words;
        ctr_words += T.tiles;
        const int p = ng++ & 1;
        P->gpar[t] = p;
        if (last_g[p] >= 0) extra[t].push_back(last_g[p]);
        last_g[p] = t;
        P->gpart_bytes = std::max<uint64_t>(P->gpart_bytes, (uint64_t)T.tiles * maxc * T.mma_n * 128 * 4);
        break;
      }
      case KD_OP_ATTENTION: {
        auto a = get_attr<kd_attr_attention>(o);
        if (a.dtype != KD_BF16 || (a.head_dim != 64 && a.head_dim != 128) || a.page != kPage || a.flags ||
            a.n_heads % a.n_kv_heads || a.n_heads / a.n_kv_heads > kMaxG)
          return bad("attention shape/dtype/flags");
        if (D && D != (int)a.head_dim) return bad("one head_dim per megakernel");
        D = a.head_dim;
        T.kind = MK_ATTN;
        T.Hq = a.n_heads, T.Hkv = a.n_kv_heads, T.D = a.head_dim, T.G = a.n_heads / a.n_kv_heads, T.pps = a.pages_per_seq;
        T.rows = a.rows;
        T.page = kPage;
        Gm = std::max(Gm, T.G);
        const long units = (long)a.rows * a.n_kv_heads;
        int splits = (int)std::max<long>(1, (8L * sms + units - 1) / units);
        if (const char* e = getenv("KD_MEGA_SPLITS")) splits = std::max(1, atoi(e));
        splits = std::min(splits, std::max(1, (int)a.pages_per_seq / 16));
        splits = std::min(splits, kFastSplitLse / T.G);
        int ppsp = ((int)a.pages_per_seq + splits - 1) / splits;
        splits = ((int)a.pages_per_seq + ppsp - 1) / ppsp;
        T.splits = splits;
        T.pps_split = ppsp;
        T.n_units = (int)(units * splits);
        T.n_dyn = std::max(0, T.n_units - sms);
        T.done_units = (unsigned)units;
        T.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)a.head_dim));
        T.a0 = o.rd[0];  // q
        T.a1 = o.rd[3];  // block table
        T.a2 = o.rd[4];  // seq_len
        T.o0 = o.wr[0];
        P->ctr_off[t] = ctr_words;
        ctr_words += units + 1;  // unit arrivals + ticket
        const int p = na++ & 1;
        P->apar[t] = p;
        if (last_a[p] >= 0) extra[t].push_back(last_a[p]);
        last_a[p] = t;
        if (splits > 1) P->apart_bytes = std::max<uint64_t>(P->apart_bytes, (uint64_t)units * splits * T.G * (a.head_dim + 1) * 4);
        break;
      }
      default:
        return bad("op " + std::to_string(o.op) + " has no megakernel task (dense decoder ops only)");
    }
    rot += (T.kind == MK_GEMM || T.kind == MK_ATTN) ? 0 : T.n_units;
  }
  if (!D) D = 128;
  // ---- dependencies: conflicting declared spans (RAW / WAR / WAW), + scratch guards
  std::vector<std::vector<Range>> R(n), W(n);
  for (int t = 0; t < n; ++t) {
    for (size_t i = 0; i < ops[t].rd.size(); ++i)
      R[t].push_back({(uintptr_t)ops[t].rd[i], (uintptr_t)ops[t].rd[i] + ops[t].rd_len[i]});
    for (size_t i = 0; i < ops[t].wr.size(); ++i)
      W[t].push_back({(uintptr_t)ops[t].wr[i], (uintptr_t)ops[t].wr[i] + ops[t].wr_len[i]});
  }
  const int nw = (n + 63) / 64;
  std::vector<std::vector<uint64_t>> anc(n, std::vector<uint64_t>(nw, 0));
  for (int t = 0; t < n; ++t) {
    std::vector<int> cand = extra[t];
    for (int s = 0; s < t; ++s)
      if (overlap(W[s], R[t]) || overlap(W[s], W[t]) || overlap(R[s], W[t])) cand.push_back(s);
    std::sort(cand.begin(), cand.end());
    cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
    std::vector<int> kept;
    for (int i = (int)cand.size() - 1; i >= 0; --i) {
      const int s = cand[i];
      if (anc[t][s / 64] >> (s % 64) & 1) continue;  // implied by a later kept dependency
      kept.push_back(s);
      for (int x = 0; x < nw; ++x) anc[t][x] |= anc[s][x];
      anc[t][s / 64] |= 1ull << (s % 64);
    }
    if ((int)kept.size() > kMaxDep) return bad("a task with more than 8 direct dependencies");
    Task& T = P->tasks[t];
    T.n_dep = (int)kept.size();
    for (int i = 0; i < T.n_dep; ++i) {
      T.dep[i] = kept[i];
      T.dep_units[i] = P->tasks[kept[i]].done_units;
    }
  }
  // ---- geometry (shared memory)
  int SPS = 0;
  if (maxM) SPS = (2 * 16384 + 2 * maxM * 128 + kSlot - 1) / kSlot;
  const size_t fixed = (size_t)2 * Gm * D * 2 + (size_t)kWorkers * Gm * D * 4 + (size_t)kWorkers * Gm * 2 * 4 +
                       (2 * kMaxStages + 2 * kMaxSlots + 24) * 8 + 112 + 2 * (kWorkers * kMaxG + 2 * kMaxG + kFastSplitLse) * 4 +
                       2048 /* static */ + 1024 /* alignment */;
  int smem_max = 0;
  KD_CUDA_CHECK(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev), "smem opt-in");
  int NS = std::min<int>(kMaxSlots, (int)(((size_t)smem_max - fixed) / kSlot));
  Geo& g = P->geo;
  g.NS = NS;
  g.SPS = SPS ? SPS : 1;
  g.NG = SPS ? std::min(kMaxStages, NS / SPS) : 1;
  g.A = NS / 8 * 8;
  if (const char* e = getenv("KD_MEGA_A")) g.A = std::max(8, std::min(g.A, atoi(e) / 8 * 8));  // A/B knob
  if ((SPS && g.NG < 2) || g.A < 8) return bad("not enough shared memory for the arena");
  g.n_tasks = n;
  g.Gm = Gm;
  g.pf = getenv("KD_MEGA_PF") ? atoi(getenv("KD_MEGA_PF")) : 1;
  g.dbg = getenv("KD_MEGA_DBG") ? atoi(getenv("KD_MEGA_DBG")) : 0;
  g.l2pf = getenv("KD_MEGA_L2PF") ? atoi(getenv("KD_MEGA_L2PF")) : 0;  // (8/16: no gain, measured)
  size_t off = (size_t)NS * kSlot;
  g.off_q = (uint32_t)off;
  off += (size_t)2 * Gm * D * 2;
  off = (off + 15) / 16 * 16;
  g.off_comb = (uint32_t)off;
  off += (size_t)kWorkers * Gm * D * 4;
  g.off_ml = (uint32_t)off;
  off += (size_t)kWorkers * Gm * 2 * 4;
  off = (off + 7) / 8 * 8;
  g.off_bar = (uint32_t)off;
  off += (2 * kMaxStages + 2 * kMaxSlots + 24) * 8;
  g.off_misc = (uint32_t)off;
  off += 112 + 2 * (kWorkers * kMaxG + 2 * kMaxG + kFastSplitLse) * 4;
  P->smem = off + 1024;  // + alignment slack
  if (P->smem > (size_t)smem_max) return bad("shared memory layout exceeds the opt-in limit");
  P->D = D;
  // ---- workspace layout
  uint64_t w = 0;
  auto take = [&](uint64_t bytes) {
    const uint64_t o2 = w;
    w = (w + bytes + 255) / 256 * 256;
    return o2;
  };
  P->off_ctrl = take(256);
  P->off_done = take((uint64_t)n * 4);
  P->off_ctr = take(ctr_words * 4 + 4);
  P->off_freq = take(P->freq.size() * 8 + 8);
  P->off_tasks = take((uint64_t)n * sizeof(Task));
  {
    uint64_t tb = 0;
    for (auto& tbl : P->tabs) tbl.off = tb, tb += (uint64_t)tbl.rows * tbl.half * 8;
    P->off_tab = take(tb + 8);
  }
  P->off_gpart = take(2 * P->gpart_bytes);
  P->off_apart = take(2 * P->apart_bytes);
  P->total = w;
  auto fn = D == 64 ? mega_kernel<64> : mega_kernel<128>;
  KD_CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P->smem), "mega smem attr");
  int occ = 0;
  KD_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kThreads, P->smem), "mega occupancy");
  if (occ < 1) return bad("the megakernel does not fit one SM");
  *out = P;
  *ws_bytes = P->total;
  return KD_OK;
}

kd_status mega_bind(MegaPlan* P, void* ws, uint64_t bytes, unsigned* err) {
  using namespace mega;
  if (!P || !ws) return fail(KD_ERR_INVALID_ARG, "megakernel: NULL workspace");
  if (bytes < P->total) return fail(KD_ERR_OOM, "megakernel: workspace too small");
  if ((uintptr_t)ws & 255) return fail(KD_ERR_INVALID_ARG, "megakernel: workspace needs 256-byte alignment");
  uint8_t* b = (uint8_t*)ws;
  P->ws = b;
  P->err = err;
  const int n = (int)P->tasks.size();
  for (int t = 0; t < n; ++t) {
    Task& T = P->tasks[t];
    const MegaOpDesc& o = P->ops[t];
    if (T.kind == MK_GEMM) {
      T.ctr = (unsigned*)(b + P->off_ctr) + P->ctr_off[t];
      T.part = (float*)(b + P->off_gpart + (uint64_t)P->gpar[t] * P->gpart_bytes);
      kd_status s = encode_bf16_2d_sw128(&T.tm0, o.rd[1], T.K, T.N, 64, 128);
      if (s) return s;
      s = encode_bf16_2d_sw128(&T.tm1, o.rd[0], T.K, T.M, 64, T.mma_n);
      if (s) return s;
    } else if (T.kind == MK_ATTN) {
      T.ctr = (unsigned*)(b + P->off_ctr) + P->ctr_off[t];
      T.ticket = T.ctr + (uint64_t)T.rows * T.Hkv;
      T.part = (float*)(b + P->off_apart + (uint64_t)P->apar[t] * P->apart_bytes);
      T.part_lse = T.part + (uint64_t)T.rows * T.Hkv * T.splits * T.G * T.D;
      const uint64_t dims[3] = {64, (uint64_t)T.D / 64u, 1ull << 30};
      const uint64_t strides[2] = {128, (uint64_t)T.D * 2u};
      const uint32_t box[3] = {64, (uint32_t)T.D / 64u, (uint32_t)kPage};
      kd_status s = encode_bf16_sw128(&T.tm0, o.rd[1], 3, dims, strides, box);
      if (s) return s;
      s = encode_bf16_sw128(&T.tm1, o.rd[2], 3, dims, strides, box);
      if (s) return s;
    } else if (T.kind == MK_ROPE) {
      T.freq = (const double*)(b + P->off_freq) + P->freq_off[t];
    }
    if (T.kind == MK_GEMM && T.epi == 1) {
      T.freq = (const double*)(b + P->off_freq) + P->freq_off[t];
      T.rtab = (const float2*)(b + P->off_tab + P->tabs[P->tab_of[t]].off);
    }
  }
  Geo& g = P->geo;
  g.n_tab = (int)P->tabs.size();
  for (int i = 0; i < g.n_tab; ++i) {
    g.tab_sl[i] = (const int32_t*)P->tabs[i].sl;
    g.tab_freq[i] = (const double*)(b + P->off_freq) + P->tabs[i].freq_off;
    g.tab[i] = (float2*)(b + P->off_tab + P->tabs[i].off);
    g.tab_rows[i] = P->tabs[i].rows;
    g.tab_half[i] = P->tabs[i].half;
  }
  g.tab_ready = (unsigned*)(b + P->off_ctrl + 64);
  KD_CUDA_CHECK(cudaMemset(b, 0, P->off_tasks), "megakernel: zero counters");
  if (!P->freq.empty())
    KD_CUDA_CHECK(cudaMemcpy(b + P->off_freq, P->freq.data(), P->freq.size() * 8, cudaMemcpyHostToDevice), "freq upload");
  KD_CUDA_CHECK(cudaMemcpy(b + P->off_tasks, P->tasks.data(), (size_t)n * sizeof(Task), cudaMemcpyHostToDevice),
                "task upload");
  P->bound = true;
  return KD_OK;
}

kd_status mega_launch(MegaPlan* P, cudaStream_t s) {
  using namespace mega;
  if (!P || !P->bound) return fail(KD_ERR_STATE, "megakernel: workspace not set");
  auto fn = P->D == 64 ? mega_kernel<64> : mega_kernel<128>;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P->grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = P->smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // every CTA resident (in-kernel waits)
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const Task* tasks = (const Task*)(P->ws + P->off_tasks);
  P->geo.trace = P->trace;
  KD_CUDA_CHECK(cudaLaunchKernelEx(&cfg, fn, tasks, P->geo, P->ws + P->off_ctrl, (unsigned*)(P->ws + P->off_done), P->err),
                "megakernel launch");
  return KD_OK;
}

void mega_destroy(MegaPlan* P) { delete P; }

void mega_set_trace(MegaPlan* P, void* buf) {
  if (P) P->trace = (unsigned long long*)buf;
}

kd_status mega_diag(const MegaPlan* P, std::string* what) {
  if (!P || !P->bound) return KD_OK;
  unsigned rec[8] = {};
  KD_CUDA_CHECK(cudaMemcpy(rec, P->ws + P->off_ctrl + 16, sizeof rec, cudaMemcpyDeviceToHost), "read megakernel record");
  if (!rec[7]) return KD_OK;
  static const char* kinds[] = {"?", "norm", "gemm", "rope", "attention", "silu", "residual"};
  const int t = (int)rec[4];
  const char* kind = (t >= 0 && t < (int)P->tasks.size() && P->tasks[t].kind <= 6) ? kinds[P->tasks[t].kind] : "?";
  char buf[256];
  snprintf(buf, sizeof buf, "megakernel %s timed out: CTA %u warp %u lane %u, task %d (%s), words %u %u",
           rec[0] == 4 ? "dependency wait" : rec[0] == 5 ? "pipeline (mbarrier) wait" : "split merge", rec[1], rec[2],
           rec[3], t, kind, rec[5], rec[6]);
  *what = buf;
  return KD_OK;
}

kd_status mega_info(const MegaPlan* P, uint32_t* n_tasks, uint32_t* smem, uint32_t* grid) {
  if (!P) return fail(KD_ERR_INVALID_ARG, "megakernel: NULL plan");
  if (n_tasks) *n_tasks = (uint32_t)P->tasks.size();
  if (smem) *smem = (uint32_t)P->smem;
  if (grid) *grid = (uint32_t)P->grid;
  return KD_OK;
}

}  // namespace kd
