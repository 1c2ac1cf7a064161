// common.cuh — shared device helpers for the sm_100a kernels of libkd.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "kd.h"

namespace kd {

constexpr int kNumSMs = 148;
#ifdef KD_SMALL_PARAMS  // A/B: kernel-parameter size
constexpr int kMaxPeers = 4;
#else
constexpr int kMaxPeers = 8;  // consumer devices per producer (a 7:1 layout scatters to 7)
#endif
// Kernel scratch layout shared by every kernel of a device (they run in
// stream order): [0, kScratchCounterBytes) holds self-resetting u32 counters
// (always zero between launches), partial results start after it.
constexpr uint64_t kScratchCounterBytes = 64 * 1024;
constexpr uint32_t kMaxCounters = kScratchCounterBytes / 4;

// ------------------------------------------------------------------ chunked P2P handoff
// Producer side ("send after k", fused into the producer): every value a
// kernel stores to its primary output at element index e is also stored to
// dst[p] + e (another device's landing slot, mapped through NVLink P2P / CUDA
// IPC, or a local slot in loopback), then released with a system-scope
// red.release on u64 flags in the consumer's workspace. Two release modes:
//  * COUNT (nch > 0): the output is a [rows][row_bytes] matrix whose row is
//    cut into nch column chunks (byte bounds cb[0..nch], the plan's chunk table,
//    R10). A CTA (or warp) that finished storing bytes [lo, hi) of some rows
//    adds rows·|[lo,hi) ∩ chunk c| to flag[c]: chunk c is complete at
//    epoch·rows·(cb[c+1] − cb[c]) bytes, whichever CTAs wrote it, so the
//    consumer can start on chunk c while later chunks are still produced.
//  * CTA (nch == 0): flag[0] += 1 per signalling CTA; complete at
//    epoch·signals (kernels whose stores are not a dense [rows][cols] block).
// Flags are monotonic across steps (epochs), never reset.
constexpr int kMaxChunks = 8;
struct Epi {
  int n = 0;                                 // peers (consumer devices)
  int nch = 0;                               // 0: CTA mode; else COUNT mode with nch chunks
  uint32_t row_bytes = 0;                    // COUNT: bytes per output row
  uint32_t cb[kMaxChunks + 1] = {};          // COUNT: chunk byte bounds within a row
  void* dst[kMaxPeers] = {};
  unsigned long long* flag[kMaxPeers] = {};     // [max(nch,1)] in the peer
  unsigned long long* started[kMaxPeers] = {};  // loopback residency (nullable)
  unsigned long long* logt[kMaxPeers] = {};     // LOG: per-chunk records (nullable)
  // delta replication (KD_BUF_REPLICATED): the peer's replica base of this
  // kernel's j-th replicated output; a write at byte offset o of the local
  // replica is mirrored to mir[p][j] + o (nullable)
  void* mir[kMaxPeers][2] = {};
  // row filter (scatter of a GEMM output to memory shards, R24): peer p
  // receives rows [r0, r0 + rn) only; rn == 0: every row
  uint32_t r0[kMaxPeers] = {}, rn[kMaxPeers] = {};
};
__device__ __forceinline__ bool epi_row_in(const Epi& e, int p, uint32_t row) {
  return e.rn[p] == 0 || row - e.r0[p] < e.rn[p];
}
// rows of [row_begin, row_end) that peer p receives
__device__ __forceinline__ uint32_t epi_rows_for(const Epi& e, int p, uint32_t row_begin, uint32_t row_end) {
  if (e.rn[p] == 0) return row_end - row_begin;
  const uint32_t a = max(row_begin, e.r0[p]), b = min(row_end, e.r0[p] + e.rn[p]);
  return b > a ? b - a : 0u;
}

// ------------------------------------------------------------------ memory model
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_sys64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_sys_add(unsigned* p, unsigned v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_release_sys_add64(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
// gpu-scope acq_rel fetch-add (split-K / split-KV arrival counters): the
// releasing side publishes its partials, the last arriver acquires them all
__device__ __forceinline__ unsigned atom_add_acq_rel_gpu(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ unsigned long long gtimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// LOG-mode record per (incoming transfer, chunk) in the consumer's workspace,
// 4 u64: [0] epoch of the first acquire, [1] that acquirer's wait start, [2]
// its acquire time, [3] the producer's latest release (%globaltimer, ns;
// monotonic across steps, so atomicMax needs no per-step reset)
constexpr int kLogWords = 4;

// COUNT mode: add rows·|[lo, hi) ∩ chunk c| bytes to every chunk the byte range
// [lo, hi) of a row touches (a caller that stored those bytes of rows
// [row_begin, row_end) — each peer counts the rows it receives — after the
// stores are ordered before this thread: fence / bar.sync)
__device__ __forceinline__ void epi_release_range(const Epi& e, uint32_t lo, uint32_t hi, uint32_t row_begin,
                                                  uint32_t row_end) {
  for (int c = 0; c < e.nch; ++c) {
    const uint32_t a = max(lo, e.cb[c]), b = min(hi, e.cb[c + 1]);
    if (a >= b) continue;
    for (int p = 0; p < e.n; ++p) {
      const uint32_t rows = epi_rows_for(e, p, row_begin, row_end);
      if (!rows) continue;
      red_release_sys_add64(e.flag[p] + c, (unsigned long long)(b - a) * rows);
      if (e.logt[p]) atomicMax(e.logt[p] + c * kLogWords + 3, gtimer_ns());
    }
  }
}
// CTA mode: one release per peer (thread-level; caller orders the CTA's stores first)
__device__ __forceinline__ void epi_release_cta(const Epi& e) {
  for (int p = 0; p < e.n; ++p) {
    red_release_sys_add64(e.flag[p], 1ull);
    if (e.logt[p]) atomicMax(e.logt[p] + 3, gtimer_ns());
  }
}
// loopback residency: every CTA of a COUNT-mode producer announces itself at
// entry (the consumer's gate waits for the whole grid before the consumer
// launches and spins on chunks in-kernel; see runtime.cu)
__device__ __forceinline__ void epi_started(const Epi& e) {
  if (threadIdx.x == 0)
    for (int p = 0; p < e.n; ++p)
      if (e.started[p]) atomicAdd(e.started[p], 1ull);
}

// publish this CTA's peer stores: call by ALL threads of the CTA after their
// stores. CTA mode: one increment; COUNT mode: the CTA declares the byte range
// [lo, hi) of `rows` rows it wrote (nch == 0 ignores them).
__device__ __forceinline__ void epi_signal(const Epi& epi, uint32_t lo = 0, uint32_t hi = 0, uint32_t row_begin = 0,
                                           uint32_t row_end = 0) {
  if (epi.n == 0) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_acq_rel_sys();
    if (epi.nch)
      epi_release_range(epi, lo, hi, row_begin, row_end);
    else
      epi_release_cta(epi);
  }
}

// COUNT-mode release of per-CTA byte tallies (kernels whose stores are not one
// rectangle per CTA): s_cnt[c] = bytes this CTA stored into chunk c (of every
// row together). Call by ALL threads after the stores.
// per_peer: s_cnt is [kMaxPeers][kMaxChunks] (row-filtered producers tally per peer)
__device__ __forceinline__ void epi_signal_counts(const Epi& epi, const unsigned* s_cnt, bool per_peer = false) {
  if (epi.n == 0) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_acq_rel_sys();
    if (epi.nch == 0) {
      epi_release_cta(epi);
      return;
    }
    for (int c = 0; c < epi.nch; ++c)
      for (int p = 0; p < epi.n; ++p) {
        const unsigned v = s_cnt[(per_peer ? p * kMaxChunks : 0) + c];
        if (!v) continue;
        red_release_sys_add64(epi.flag[p] + c, (unsigned long long)v);
        if (epi.logt[p]) atomicMax(epi.logt[p] + c * kLogWords + 3, gtimer_ns());
      }
  }
}
__device__ __forceinline__ int epi_chunk_of(const Epi& epi, uint32_t byte_in_row) {
  int c = 0;
  while (c + 1 < epi.nch && byte_in_row >= epi.cb[c + 1]) ++c;
  return c;
}

// ------------------------------------------------------------------ consumer side ("recv before k")
// A chunk-aware consumer acquires chunk c of a remote input right before it
// reads it: spin until flag[c] >= (epoch − base)·mult[c] (ld.acquire.sys),
// watchdog → *err = 1. One thread acquires; the caller then orders the other
// threads behind it (bar.sync / __syncwarp) — or, for TMA reads, a proxy fence.
#ifdef KD_SMALL_PARAMS
constexpr int kMaxAcqIn = 1;
#else
constexpr int kMaxAcqIn = 4;
#endif
struct AcqIn {
  const unsigned long long* flag = nullptr;  // [nch]
  unsigned long long* log = nullptr;         // LOG: per-chunk records (nullable)
  int slot = 0;                              // operand index (GEMM: 0 = X; add_rmsnorm / residual: delta index)
  int nch = 0;
  uint32_t row_bytes = 0;
  uint32_t cb[kMaxChunks + 1] = {};
  unsigned long long mult[kMaxChunks] = {};
};
struct Acq {
  int n = 0;                      // remote inputs acquired in-kernel (0: none)
  unsigned base = 0;              // steps run without transfers (their epochs carry no releases)
  const unsigned* epoch = nullptr;
  unsigned* err = nullptr;
  AcqIn in[kMaxAcqIn];
};

__device__ __forceinline__ int acq_find(const Acq& a, int slot) {
  for (int i = 0; i < a.n; ++i)
    if (a.in[i].slot == slot) return i;
  return -1;
}
__device__ __forceinline__ void acq_chunk(const Acq& a, int i, int c) {
  const AcqIn& in = a.in[i];
  const unsigned e = *(volatile const unsigned*)a.epoch;
  const unsigned long long target = (unsigned long long)(e - a.base) * in.mult[c];
  if (ld_acquire_sys64(in.flag + c) >= target) {
    if (in.log && atomicMax(in.log + c * kLogWords, (unsigned long long)e) < e) {
      const unsigned long long t = gtimer_ns();
      in.log[c * kLogWords + 1] = t;
      in.log[c * kLogWords + 2] = t;
    }
    return;
  }
  const unsigned long long t0 = in.log ? gtimer_ns() : 0ull;
  long long spins = 0;
  while (ld_acquire_sys64(in.flag + c) < target) {
    if (++spins > (1ll << 24)) {  // watchdog (~10 s): record (KD_ERR_TIMEOUT at kd_runtime_check) and give up
      if (a.err) atomicExch(a.err, 1u);
      break;
    }
    __nanosleep(40);
  }
  if (in.log && atomicMax(in.log + c * kLogWords, (unsigned long long)e) < e) {
    in.log[c * kLogWords + 1] = t0;
    in.log[c * kLogWords + 2] = gtimer_ns();
  }
}
// acquire every chunk of remote input i that the byte range [lo, hi) of a row
// touches, in ascending order; `done` caches the chunks this thread already holds
__device__ __forceinline__ void acq_range(const Acq& a, int i, uint32_t lo, uint32_t hi, uint32_t* done) {
  const AcqIn& in = a.in[i];
  for (int c = 0; c < in.nch; ++c)
    if (lo < in.cb[c + 1] && in.cb[c] < hi && !(*done & (1u << c))) {
      acq_chunk(a, i, c);
      *done |= 1u << c;
    }
}

// ------------------------------------------------------------------ programmatic dependent launch
// Every kernel lets its dependent grid launch early and waits for its
// prerequisite grid before touching memory the prerequisite may write (or
// read). Every CTA executes the wait, so no grid can complete before its
// predecessor (keeps the dependency chain transitive). No-ops without PDL.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ------------------------------------------------------------------ bf16 helpers
__device__ __forceinline__ float bf16lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16hi(uint32_t v) { return __uint_as_float(v & 0xFFFF0000u); }
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float to_f(const __nv_bfloat16 x) { return __bfloat162float(x); }
__device__ __forceinline__ float to_f(const float x) { return x; }
template <typename T>
__device__ __forceinline__ T from_f(float x);
template <>
__device__ __forceinline__ float from_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

// silu(x) = x·sigmoid(x) with the fast divide (≈2 ulp; outputs are bf16): the
// one definition shared by the SiLU kernel and the fused gate_up+SiLU epilogue,
// so the two produce identical bits
__device__ __forceinline__ float silu_fast(float x) { return __fdividef(x, 1.f + __expf(-x)); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

}  // namespace kd
