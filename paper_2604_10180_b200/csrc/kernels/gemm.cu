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
#include <mutex>

#include "launch.hpp"

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
  long long units;
  Epi epi;
  unsigned long long* trace;  // debug: 32 %globaltimer stamps per CTA (nullable)
  // grouped (MoE expert) mode: groups > 0; tile t → group t / tpg, n-tile t % tpg;
  // meta = int32 count[groups], offset[groups] (rows of X/Y), read on device
  int groups, tpg;
  const int* meta;
  int dbg;                    // debug A/B knob (KD_GEMM_DBG): 1 skip owner Y stores, 2 skip owner fold
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define KD_TRACE(slot) \
  do {                 \
    if (A.trace) A.trace[blockIdx.x * 32 + (slot)] = gtimer(); \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n\t}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// K-major operand tile in smem, 128-byte swizzle: 8-row atoms of 1024 B (SBO),
// descriptor version 1 (sm_100), layout type 2 = SWIZZLE_128B.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15]))
      : "memory");
}
__device__ __forceinline__ float4 lds128(uint32_t saddr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(saddr));
  return v;
}
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n)); }

// unit range of CTA c: [c·U/G, (c+1)·U/G); owner of unit u: ⌈(u+1)·G/U⌉ − 1
__host__ __device__ __forceinline__ long long unit_begin(long long c, long long U, long long G) { return c * U / G; }
__host__ __device__ __forceinline__ long long unit_owner(long long u, long long U, long long G) {
  return ((u + 1) * G + U - 1) / U - 1;
}

__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmap_w, const __grid_constant__ CUtensorMap tmap_x, Args A) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int S = A.stages;
  const int stage_b = A.mma_n * kBK * 2;
  uint8_t* sa = smem;                          // S × 16 KB
  uint8_t* sb = smem + (size_t)S * kStageA;    // S × mma_n·128 B
  uint64_t* full = (uint64_t*)(sb + (size_t)S * stage_b);
  uint64_t* empty = full + kMaxStages;
  uint64_t* tfull = empty + kMaxStages;        // [2]
  uint64_t* tempty = tfull + 2;                // [2]
  uint64_t* fixbar = tempty + 2;               // owner's partial bulk loads
  uint32_t* tmem_slot = (uint32_t*)(fixbar + 1);
  __nv_bfloat16* ystage = (__nv_bfloat16*)(fixbar + 2);  // 2 x [16][128] bf16 epilogue transpose

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) KD_TRACE(0);
  pdl_launch_dependents();
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

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (lane == 0) {
      const uint64_t pw = policy_evict_first(), px = policy_evict_last();
      const unsigned tx = kStageA + stage_b;
      // weights never depend on the previous kernel: fill the first ring of W
      // tiles before the grid-dependency wait (overlaps the previous kernel's
      // tail), then the activations of those stages, then steady state
      const long long n_pre = std::min<long long>(S, u1 - u0);
      auto w_row = [&](int t) { return A.groups ? (t / A.tpg) * A.N + (t % A.tpg) * kBM : t * kBM; };
      for (long long i = 0; i < n_pre; ++i) {
        const long long u = u0 + i;
        const int t = (int)(u / KB), kb = (int)(u % KB);
        mbar_expect_tx(&full[i], tx);
        tma_load_2d(sa + (size_t)i * kStageA, &tmap_w, kb * kBK, w_row(t), &full[i], pw);
        if (i == 0) KD_TRACE(2);
      }
      pdl_wait();
      auto x_row = [&](int t) { return A.groups ? __ldg(A.meta + A.groups + t / A.tpg) : 0; };
      for (long long i = 0; i < n_pre; ++i) {
        const long long u = u0 + i;
        tma_load_2d(sb + (size_t)i * stage_b, &tmap_x, (int)(u % KB) * kBK, x_row((int)(u / KB)), &full[i], px);
      }
      long long i = n_pre;
      for (long long u = u0 + n_pre; u < u1; ++u, ++i) {
        const int s = (int)(i % S);
        const long long r = i / S;
        if (r > 0) mbar_wait(&empty[s], (unsigned)((r - 1) & 1));
        const int t = (int)(u / KB), kb = (int)(u % KB);
        mbar_expect_tx(&full[s], tx);
        tma_load_2d(sa + (size_t)s * kStageA, &tmap_w, kb * kBK, w_row(t), &full[s], pw);
        tma_load_2d(sb + (size_t)s * stage_b, &tmap_x, kb * kBK, x_row(t), &full[s], px);
      }
      KD_TRACE(3);
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    if (lane == 0) {
      pdl_wait();
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(A.mma_n >> 3) << 17) |
                             ((uint32_t)(kBM >> 4) << 24);
      long long i = 0;
      int seg = 0;
      long long u = u0;
      while (u < u1) {
        const int t = (int)(u / KB);
        const long long seg_end = std::min<long long>(u1, (long long)(t + 1) * KB);
        const int a = seg & 1, use = seg >> 1;
        if (use > 0) mbar_wait(&tempty[a], (unsigned)((use - 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t tmem_d = tmem_base + (uint32_t)(a * A.mma_n);
        bool first = true;
        for (; u < seg_end; ++u, ++i) {
          const int s = (int)(i % S);
          mbar_wait(&full[s], (unsigned)((i / S) & 1));
          if (i == 0) KD_TRACE(4);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t a_addr = smem_u32(sa + (size_t)s * kStageA);
          const uint32_t b_addr = smem_u32(sb + (size_t)s * stage_b);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            // advance 16 bf16 = 32 B inside the 128 B swizzle row
            mma_bf16(tmem_d, sw128_desc(a_addr + 32 * k), sw128_desc(b_addr + 32 * k), idesc,
                     (first && k == 0) ? 0u : 1u);
          }
          first = false;
          mma_commit(&empty[s]);  // smem stage free once these MMAs retire
        }
        mma_commit(&tfull[a]);    // accumulator ready for the epilogue
        ++seg;
      }
      KD_TRACE(5);
    }
  } else if (warp >= 4) {
    // ------------------------------------------------ epilogue (TMEM → HBM / peers)
    // Split tiles (stream-K): every contributor c of tile t publishes its fp32
    // partial [M][128] to slot (c - first contributor), release-increments
    // arrive[t], waits until all n_contrib partials are published, then folds
    // ITS 1/n slice of the tile (fixed contributor order → bitwise
    // deterministic) and stores it. depart[t] lets the last leaver reset both
    // counters for the next launch. Contributors only wait for partials that
    // are published before anyone waits, so this cannot deadlock.
    const int q = warp - 4;                 // TMEM lane quarter
    const int row_in_tile = q * 32 + lane;  // output feature within the tile
    const int ep_tid = threadIdx.x - 128;
    const size_t part_elems = (size_t)A.M * kBM;
    pdl_wait();  // scratch and Y may still be in use by the previous kernel
    int seg = 0;
    long long u = u0;
    while (u < u1) {
      const int t = (int)(u / KB);
      const long long t_begin = (long long)t * KB, t_end = t_begin + KB;
      const long long seg_end = std::min<long long>(u1, t_end);
      const bool whole = (u == t_begin && seg_end == t_end);
      const int a = seg & 1;
      mbar_wait(&tfull[a], (unsigned)((seg >> 1) & 1));
      if (ep_tid == 0 && seg < 3) KD_TRACE(6 + 2 * seg);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(a * A.mma_n);
      // output coordinates of tile t: column base nb0, row base y0, valid rows mv
      const int grp = A.groups ? t / A.tpg : 0;
      const int nb0 = (A.groups ? t % A.tpg : t) * kBM;
      const int y0 = A.groups ? __ldg(A.meta + A.groups + grp) : 0;
      const int mv = A.groups ? min(__ldg(A.meta + grp), A.M) : A.M;
      if (!whole) {
        const long long first = unit_owner(t_begin, U, G);
        const long long lastc = unit_owner(t_end - 1, U, G);
        const int n_contrib = (int)(lastc - first + 1);
        const int my_idx = (int)(c - first);
        // participants fold: contributors for which this tile is their LAST
        // segment. Only the last contributor can have more work after this
        // tile (a "tail" part at the start of its range); it publishes only.
        const bool tail_exists = unit_begin(lastc + 1, U, G) > t_end;
        const int n_part = n_contrib - (tail_exists ? 1 : 0);
        const bool participant = (seg_end == u1);
        const float* parts = A.part + (size_t)t * A.max_contrib * part_elems;
        float* my_part = A.part + ((size_t)t * A.max_contrib + my_idx) * part_elems;
        for (int j0 = 0; j0 < A.M; j0 += kChunk) {
          float v[kChunk];
          tmem_ld16(tbase + j0, v);
#pragma unroll
          for (int j = 0; j < kChunk; ++j)
            if (j0 + j < A.M) my_part[(size_t)(j0 + j) * kBM + row_in_tile] = v[j];
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[a]);
        named_bar(1, 128);
        unsigned* arrive = A.counter + 2 * t;
        unsigned* depart = arrive + 1;
        if (ep_tid == 0) {
          KD_TRACE(18);
          fence_acq_rel_gpu();
          atom_add_acq_rel_gpu(arrive, 1u);
          if (participant) {
            long long spins = 0;
            while (ld_acquire_gpu(arrive) < (unsigned)n_contrib)
              if (++spins > 64) __nanosleep(32);
            KD_TRACE(16);
            if (atom_add_acq_rel_gpu(depart, 1u) == (unsigned)n_part - 1) {
              *arrive = 0u;  // every participant has left the wait: reset for the next launch
              *depart = 0u;
            }
          }
        }
        named_bar(1, 128);
        // fold my slice: float4 elements [e0, e1) of the [M][128] tile
        const int n4 = participant ? (int)(part_elems / 4) : 0;
        const int e0 = (int)((long long)n4 * my_idx / n_part), e1 = (int)((long long)n4 * (my_idx + 1) / n_part);
        // 4 elements per thread per round: all (element, contributor) loads of a
        // round are in flight together (memory-level parallelism for the L2 reads)
        constexpr int EB = 4;
        for (int eb = e0 + ep_tid; eb < e1; eb += 128 * EB) {
          float4 acc[EB];
          for (int c0 = 0; c0 < n_contrib; c0 += 8) {
            const int cn = min(8, n_contrib - c0);
            float4 xs[EB][8];
#pragma unroll
            for (int k = 0; k < EB; ++k)
#pragma unroll
              for (int ci = 0; ci < 8; ++ci) {
                const int e = eb + k * 128;
                if (ci < cn && e < e1)
                  xs[k][ci] = __ldcg(reinterpret_cast<const float4*>(parts + (size_t)(c0 + ci) * part_elems) + e);
              }
#pragma unroll
            for (int k = 0; k < EB; ++k)
#pragma unroll
              for (int ci = 0; ci < 8; ++ci)
                if (ci < cn) {
                  if (c0 + ci == 0) {
                    acc[k] = xs[k][ci];
                  } else {
                    acc[k].x += xs[k][ci].x;
                    acc[k].y += xs[k][ci].y;
                    acc[k].z += xs[k][ci].z;
                    acc[k].w += xs[k][ci].w;
                  }
                }
          }
#pragma unroll
          for (int k = 0; k < EB; ++k) {
            const int e = eb + k * 128;
            if (e >= e1) break;
            const int j = (e * 4) / kBM, r = (e * 4) % kBM;
            const int nn = nb0 + r;
            if (nn < A.N && j < mv) {
              uint2 o;
              o.x = pack_bf16(acc[k].x, acc[k].y);
              o.y = pack_bf16(acc[k].z, acc[k].w);
              const size_t yo = (size_t)(y0 + j) * A.N + nn;
              if (nn + 4 <= A.N && (A.N & 3) == 0) {
                *reinterpret_cast<uint2*>(A.Y + yo) = o;
                for (int p = 0; p < A.epi.n; ++p) *reinterpret_cast<uint2*>((__nv_bfloat16*)A.epi.dst[p] + yo) = o;
              } else {
                const float vv[4] = {acc[k].x, acc[k].y, acc[k].z, acc[k].w};
                for (int x = 0; x < 4 && nn + x < A.N; ++x) {
                  A.Y[yo + x] = __float2bfloat16_rn(vv[x]);
                  for (int p = 0; p < A.epi.n; ++p) ((__nv_bfloat16*)A.epi.dst[p])[yo + x] = __float2bfloat16_rn(vv[x]);
                }
              }
            }
          }
        }
        if (ep_tid == 0) KD_TRACE(13);
      } else {
        // ---- whole tile: TMEM → bf16 → smem transpose → 16-byte stores
        for (int j0 = 0; j0 < A.M; j0 += kChunk) {
          float v[kChunk];
          tmem_ld16(tbase + j0, v);
          __nv_bfloat16* st = ystage + (size_t)((j0 / kChunk) & 1) * kChunk * kBM;
#pragma unroll
          for (int j = 0; j < kChunk; ++j) st[j * kBM + row_in_tile] = __float2bfloat16_rn(v[j]);
          named_bar(2, 128);
          const int jn = min(kChunk, mv - j0);
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            const int e = ep_tid + r * 128;  // 256 vectors of 8 bf16 per chunk
            const int j = e >> 4, col = (e & 15) * 8;
            const int nn = nb0 + col;
            if (j < jn && nn < A.N) {
              const uint4 val = *reinterpret_cast<const uint4*>(st + j * kBM + col);
              const size_t yo = (size_t)(y0 + j0 + j) * A.N + nn;
              if (nn + 8 <= A.N && (A.N & 7) == 0) {
                *reinterpret_cast<uint4*>(A.Y + yo) = val;
                for (int p = 0; p < A.epi.n; ++p) *reinterpret_cast<uint4*>((__nv_bfloat16*)A.epi.dst[p] + yo) = val;
              } else {
                const __nv_bfloat16* sv = reinterpret_cast<const __nv_bfloat16*>(&val);
                for (int x = 0; x < 8 && nn + x < A.N; ++x) {
                  A.Y[yo + x] = sv[x];
                  for (int p = 0; p < A.epi.n; ++p) ((__nv_bfloat16*)A.epi.dst[p])[yo + x] = sv[x];
                }
              }
            }
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[a]);
      }
      // publish this segment's share of the output to consumer devices
      // (whole tiles and fold participants; a tail contributor stored nothing)
      const bool stored = whole || seg_end == u1;
      if (A.epi.n && stored) {
        named_bar(1, 128);
        if (ep_tid == 0) {
          fence_acq_rel_sys();
          for (int p = 0; p < A.epi.n; ++p) red_release_sys_add(A.epi.flag[p], 1u);
        }
      }
      if (ep_tid == 0 && seg < 3) KD_TRACE(7 + 2 * seg);
      u = seg_end;
      ++seg;
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
  int mma_n, stages, kblocks, tiles, grid, max_contrib;
  long long units;
};

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      n = kNumSMs;
  }
  return n;
}

static kd_status geometry(const GemmShape& a, Geometry* g, int sms) {
  if (a.dtype != KD_BF16) return fail(KD_ERR_UNSUPPORTED, "gemm: only bf16 (fp32 path not built)");
  if (a.M == 0 || a.N == 0 || a.K == 0 || a.rows_total == 0) return fail(KD_ERR_INVALID_ARG, "gemm: empty shape");
  if (a.M > 256) return fail(KD_ERR_UNSUPPORTED, "gemm: decode GEMM supports M <= 256 rows (per group)");
  if (a.K % 8) return fail(KD_ERR_UNSUPPORTED, "gemm: K must be a multiple of 8 (16-byte TMA rows)");
  if (a.groups && a.N % kBM) return fail(KD_ERR_UNSUPPORTED, "grouped gemm: N must be a multiple of 128");
  g->mma_n = (int)((a.M + 15) / 16 * 16);
  const int stage_bytes = kStageA + g->mma_n * kBK * 2;
  g->stages = std::min(kMaxStages, (kSmemBudget - 2 * kChunk * kBM * 2) / stage_bytes);
  g->kblocks = (int)((a.K + kBK - 1) / kBK);
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
  return 1024 + (size_t)g.stages * (kStageA + g.mma_n * kBK * 2) + (2 * kMaxStages + 6) * 8 + 2 * kChunk * kBM * 2 + 16;
}

}  // namespace gemm

GemmShape gemm_shape(const kd_attr_gemm& a) {
  GemmShape s;
  s.M = a.M;
  s.rows_total = a.M;
  s.N = a.N;
  s.K = a.K;
  s.groups = 0;
  s.dtype = a.dtype;
  return s;
}

GemmShape gemm_shape(const kd_attr_grouped_gemm& a) {
  GemmShape s;
  s.M = a.rows_cap;
  s.rows_total = a.rows_total;
  s.N = a.N;
  s.K = a.K;
  s.groups = a.experts;
  s.dtype = a.dtype;
  return s;
}

kd_status gemm_scratch_bytes(const GemmShape& a, uint64_t* bytes) {
  gemm::Geometry g;
  kd_status s = gemm::geometry(a, &g, kNumSMs);
  if (s) return s;
  if (2ull * g.tiles > kMaxCounters) return fail(KD_ERR_UNSUPPORTED, "gemm: too many output tiles");
  uint64_t n = kScratchCounterBytes + (uint64_t)g.tiles * g.max_contrib * a.M * gemm::kBM * 4;
  *bytes = (n + 255) / 256 * 256;
  return KD_OK;
}

kd_status gemm_prepare(const GemmShape& a, const void* X, const void* W, const void* meta, GemmPlan* gp) {
  gemm::Geometry g;
  kd_status s = gemm::geometry(a, &g, kNumSMs);
  if (s) return s;
  if (!X || !W || (a.groups && !meta)) return fail(KD_ERR_INVALID_ARG, "gemm: NULL operand");
  if (((uintptr_t)X | (uintptr_t)W) & 15) return fail(KD_ERR_INVALID_ARG, "gemm: operands must be 16-byte aligned");
  s = gemm::encode(&gp->tmap_w, W, a.K, (uint64_t)a.N * std::max<uint32_t>(1, a.groups), gemm::kBM);
  if (s) return s;
  s = gemm::encode(&gp->tmap_x, X, a.K, a.rows_total, (uint32_t)g.mma_n);
  if (s) return s;
  gp->sh = a;
  gp->meta = (const int*)meta;
  return KD_OK;
}

static unsigned long long* g_gemm_trace = nullptr;

kd_status launch_gemm(const GemmPlan& gp, void* Y, const LaunchCtx& c, uint32_t* signals) {
  gemm::Geometry g;
  kd_status s = gemm::geometry(gp.sh, &g, kNumSMs);
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
  A.mma_n = g.mma_n;
  A.stages = g.stages;
  A.kblocks = g.kblocks;
  A.tiles = g.tiles;
  A.max_contrib = g.max_contrib;
  A.units = g.units;
  A.epi = c.epi;
  A.trace = g_gemm_trace;
  {
    static int dbg = -1;
    if (dbg < 0) dbg = getenv("KD_GEMM_DBG") ? atoi(getenv("KD_GEMM_DBG")) : 0;
    A.dbg = dbg;
  }
  size_t sm = gemm::smem_bytes(g);
  kd_status ks = kernels_init();
  if (ks) return ks;
  KD_CUDA_CHECK(kd_launch(gemm::gemm_kernel, dim3(g.grid), dim3(gemm::kThreads), sm, c.stream, gp.tmap_w, gp.tmap_x, A),
                "gemm launch");
  if (signals) return gemm_signals(gp.sh, signals);
  return KD_OK;
}

}  // namespace kd

extern "C" kd_status kd_debug_gemm_trace(void* dev_buf) {  // 32 u64 stamps per CTA
  kd::g_gemm_trace = (unsigned long long*)dev_buf;
  return KD_OK;
}

namespace kd {

kd_status gemm_signals(const GemmShape& a, uint32_t* s) {
  gemm::Geometry g;
  kd_status st = gemm::geometry(a, &g, kNumSMs);
  if (st) return st;
  // one flag increment per (tile, contributing CTA) segment: whole tiles count
  // once, a split tile once per contributor (each stores its slice)
  uint64_t n = 0;
  for (int t = 0; t < g.tiles; ++t) {
    const long long tb = (long long)t * g.kblocks, te = tb + g.kblocks;
    long long f = gemm::unit_owner(tb, g.units, g.grid);
    long long l = gemm::unit_owner(te - 1, g.units, g.grid);
    const bool tail = gemm::unit_begin(l + 1, g.units, g.grid) > te;
    n += (uint64_t)(l - f + 1) - (l > f && tail ? 1 : 0);
  }
  *s = (uint32_t)n;
  return KD_OK;
}

kd_status gemm_init_attrs() {
  KD_CUDA_CHECK(cudaFuncSetAttribute(gemm::gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024),
                "gemm smem attr");
  KD_CUDA_CHECK(cudaFuncSetAttribute(gemm::gemm_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100),
                "gemm carveout");
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
