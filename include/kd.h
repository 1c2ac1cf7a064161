/*
 * kd.h — C ABI of the B200-native kernel-disaggregation hot path
 * (arXiv 2604.10180, "kernel disaggregation"; P:n = PAPER.md line n,
 *  S:n = SPEC.md line n, R# = readings in DESIGN.md / SURVEY §8(c)).
 *
 * The path: build a kernel DAG from declared per-kernel buffer read/write
 * sets (P:241-242 library kernels, P:276 DDG) → assign kernels to devices
 * (E1-E7) → plan a per-device schedule → run a
 * decode step with N micro-batches on B200s, where cut edges are streamed
 * into the consumer GPU's HBM by the producer kernel itself (fused peer-store
 * epilogue + flag release) instead of the paper's NCCL/IBGDA send/recv
 * kernels.
 *
 * Conventions (apply to every call unless stated):
 *  - No exception crosses the ABI. Every call returns kd_status; on failure a
 *    thread-local message is available from kd_last_error(). Out-parameters
 *    are written only when KD_OK is returned.
 *  - Host pointers are plain C arrays owned by the caller and only read during
 *    the call. Device pointers ("dev ptr") are owned by the caller (PyTorch
 *    allocations); the library borrows them for the lifetime of the object it
 *    was given to and owns no device memory itself.
 *  - cudaStream_t is passed as void*.
 *  - Objects are not thread-safe; distinct objects may be used concurrently.
 *  - Integer time is picoseconds, sizes are bytes (R7).
 */
#ifndef KD_H_
#define KD_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ status */
typedef int32_t kd_status;
enum {
  KD_OK = 0,
  KD_ERR_INVALID_ARG = 1,   /* null pointer, zero-length span, bad enum, bad shape */
  KD_ERR_RANGE = 2,         /* span outside its buffer; output capacity too small */
  KD_ERR_STATE = 3,         /* wrong call order (e.g. add after finalize) */
  KD_ERR_PIN_CONFLICT = 4,  /* two pins disagree inside one template class */
  KD_ERR_INFEASIBLE = 5,    /* no candidate placement / schedule deadlock */
  KD_ERR_UNSUPPORTED = 6,   /* op, shape or cut pattern the runtime cannot execute */
  KD_ERR_CUDA = 7,          /* a CUDA runtime/driver call failed (message has the CUDA error) */
  KD_ERR_NCCL = 8,          /* reserved for the TP all-reduce path */
  KD_ERR_TIMEOUT = 9,       /* a device-side flag wait exceeded its watchdog */
  KD_ERR_OOM = 10           /* workspace smaller than kd_plan_workspace_bytes */
};
const char* kd_status_str(kd_status s);
const char* kd_last_error(void);
/* library version: (major << 16) | minor */
uint32_t kd_version(void);

/* ------------------------------------------------------------------ graph
 * Buffers and kernels are declared in PROGRAM ORDER (= execution order,
 * P:276 "By iterating over kernels in execution order"). A kernel's read and
 * write sets are declared spans (the paper's library-kernel case, P:241-242:
 * "cublasSgemm(.,A,B,.,C,.) reads bufferA and bufferB and writes bufferC").
 * The graph describes ONE micro-batch of the step; kd_plan_create instantiates
 * it N times (buffers flagged KD_BUF_PER_MICROBATCH get one instance per
 * micro-batch, others are shared).
 */
typedef struct kd_graph kd_graph;

enum {
  KD_BUF_WEIGHT = 1u << 0,         /* read-only, initialised by the caller: never a DAG source (R5) */
  KD_BUF_INPUT = 1u << 1,          /* initialised by the caller before each step */
  KD_BUF_OUTPUT = 1u << 2,         /* read by the caller after the step */
  KD_BUF_PERSISTENT = 1u << 3,     /* cross-iteration state (KV cache, SSM state); all
                                      kernels touching it must be co-located (R6) */
  KD_BUF_PER_MICROBATCH = 1u << 4, /* one instance per micro-batch */
  /* with PERSISTENT: cross-iteration state REPLICATED on every device whose
   * kernels touch it, writes propagated as deltas ("maintains a
   * replica on each GPU and propagates the delta memory to other replicas").
   * The caller binds one identically initialised replica per device; a kernel
   * writing it mirrors exactly the bytes it writes into every peer replica
   * (fused stores, released with its transfer to that device), so readers on
   * other devices see them; the cost model charges the delta (e.g. RoPE/append:
   * the appended K or V slot, rows·Hkv·D·elem), not the declared span. */
  KD_BUF_REPLICATED = 1u << 5
};

typedef struct {
  uint32_t buf;     /* buffer id from kd_graph_add_buffer */
  uint32_t pad_;
  uint64_t offset;  /* bytes from the buffer start */
  uint64_t len;     /* bytes, > 0; offset + len <= buffer size */
} kd_span;

/* op codes: the kernels of the decoder-layer graph */
enum {
  KD_OP_NONE = 0,          /* bookkeeping node: costs a launch, executes nothing */
  KD_OP_ADD_RMSNORM = 1,   /* a3  reads [r, delta_0..delta_{n-1}, gamma] writes [h, r] */
  KD_OP_GEMM = 2,          /* a4/a7/a9/a10 reads [X, W] writes [Y]: Y = X·Wᵀ       */
  KD_OP_ROPE_APPEND = 3,   /* a5  reads [qkv, block_table, seq_len] writes [q, Kc, Vc] */
  KD_OP_ATTENTION = 4,     /* a6  reads [q, Kc, Vc, block_table, seq_len] writes [out] */
  KD_OP_SILU_MUL = 5,      /* a8  reads [gu] writes [a]                          */
  KD_OP_RESIDUAL_ADD = 6,  /* C1.11 reads [r, delta_0..delta_{n-1}] writes [r]   */
  KD_OP_MOE_ROUTE = 7,     /* a11 reads [h, W_router] writes [route]            */
  KD_OP_MOE_DISPATCH = 8,  /* a11 reads [h, route] writes [xg, meta]            */
  KD_OP_GROUPED_GEMM = 9,  /* a11 reads [xg, W_experts, meta] writes [yg]       */
  KD_OP_MOE_COMBINE = 10,  /* a11 reads [yg, route, meta] writes [out]          */
  KD_OP_SSM_CONV = 11,     /* a12 reads [zxbcdt, conv_w, conv_b, conv_state] writes [xbc, conv_state] */
  KD_OP_SSM_UPDATE = 12,   /* a12 reads [xbc, zxbcdt, dt_bias, A_log, D, ssm_state] writes [y, ssm_state] */
  KD_OP_GATED_NORM = 13,   /* a12 reads [y, zxbcdt, norm_w] writes [yn]          */
  KD_OP_GEMM_SILU = 14,    /* a9+a8 fused (co-located gate_up and SiLU·mul): reads [X, W_gu] writes [a]:
                            * a = silu_mul_blocked(bf16(X·W_guᵀ)) with kd_attr_gemm, N = 2F weight rows
                            * (64-row gate/up blocks, R12), a [M, F]; bits identical to a9 then a8 */
  KD_OP_QKV_ROPE = 15,     /* a4+a5 fused (co-located QKV GEMM and RoPE + KV append): reads [X, W_qkv',
                            * block_table, seq_len] writes [q, Kc, Vc] with kd_attr_qkv_rope. W_qkv' = the
                            * kv-group-interleaved QKV weight with rows pair-interleaved inside every head
                            * (row 2p ← dim p, row 2p+1 ← dim p + D/2); bits identical to a4 then a5 */
  KD_OP_ATTN_MERGE = 16,   /* f2 reads [part_0 .. part_{n-1}] ([out|lse] of KD_ATTN_LSE attentions) writes [out] */
  KD_OP_ROPE_PREFILL = 18,  /* f4 reads [qkv, block_table] writes [q, Kc, Vc]: RoPE at every prompt position
                            * (token row r = b·S + t rotated by t·θ^(−2i/D)) and the paged-cache fill of slots
                            * 0..S−1 (oracle/prefill.py rope_prefill) */
  KD_OP_PREFILL_ATTENTION = 19,  /* f4 reads [q, Kc, Vc, block_table] writes [out]: causal GQA self-attention
                            * over each sequence's S prompt tokens (row r = b·S + t attends keys 0..t) */
  KD_OP_GEMM_RMSNORM = 17  /* a7+a3 / a10+a3 fused (co-located O or down GEMM and the next residual add +
                            * RMSNorm): reads [X, W, r, gamma] writes [h, r] with kd_attr_gemm_rmsnorm:
                            * r' = r + bf16(X·Wᵀ) (bits identical to a GEMM then a3's add), h =
                            * r'/sqrt(mean r'² + eps)·gamma (Σr'² in another order than a3: not bitwise).
                            * flags KD_NORM_DEFER: writes [xs, r, ssq] instead — xs = bf16(r'·gamma) and the
                            * per-token partial sums of r'² (layout KD_DNORM_*, one per CTA), no grid-wide
                            * wait; the 1/rms factor is applied by the co-located consumer GEMM
                            * (KD_OP_GEMM_SILU / KD_OP_QKV_ROPE with ssq as an extra last read), which
                            * scales its fp32 sums row by row: (xs·Wᵀ)·rsqrt(Σ ssq / N + eps) — RMSNorm's
                            * per-token factor moved past the linear map (same math, other rounding point) */
};

/* element types of activations / KV */
enum { KD_BF16 = 0, KD_F32 = 1 };

/* Op attributes (the op's "API signature"). The FIRST write span of
 * every op is its primary output: the only output the runtime may stream to
 * another device (other outputs must stay co-located with their readers). */
/* n_delta (0..8) residual deltas are added to r in index order in fp32:
 * r' = ((r + δ_0) + δ_1) + … — with n_delta > 1 this is the reduction half of
 * a tensor-parallel all-reduce whose partials were streamed in by the
 * row-parallel GEMMs' fused peer stores. */
typedef struct { uint32_t rows, hidden, n_delta, dtype; float eps; uint32_t pad_; } kd_attr_add_rmsnorm;
typedef struct { uint32_t M, N, K, dtype; } kd_attr_gemm;            /* X [M,K], W [N,K] row-major, Y [M,N] */
/* X [M,K], W [N,K] (N = hidden), r fp32 [M,N], gamma [N], h [M,N]; bf16 only */
typedef struct { uint32_t M, N, K, dtype; float eps; uint32_t flags; } kd_attr_gemm_rmsnorm;
/* KD_OP_GEMM_RMSNORM flags; deferred-norm partial sums (fp32 buffer of
 * KD_DNORM_BYTES(M) bytes): [0] eps, [1] N (as float), then from float
 * KD_DNORM_HDR on, row j (token) holds KD_DNORM_PARTS partials (unused ones
 * zero) summed in index order by the consumer */
enum { KD_NORM_DEFER = 1 };
enum { KD_DNORM_HDR = 16, KD_DNORM_PARTS = 160 };
#define KD_DNORM_BYTES(M) (4ull * (KD_DNORM_HDR + (uint64_t)(M) * KD_DNORM_PARTS))
/* slot_offset: tokens of each sequence held by earlier KV shards (f2, long
 * context split over devices): the rotation angle uses the absolute position
 * seq_len − 1, the appended slot is (seq_len − 1 − slot_offset) in this
 * shard's block table. 0 for an unsharded cache. */
typedef struct {
  uint32_t rows, n_heads, n_kv_heads, head_dim, page, pages_per_seq, dtype, slot_offset;
  double theta;   /* RoPE base (R12) */
} kd_attr_rope_append;
/* flags: KD_ATTN_LSE → the output buffer is [out bf16 rows×Hq×D | lse fp32
 * rows×Hq], lse = log2 Σ_t 2^(s_t·log2e) (the base-2 log-sum-exp of the
 * scaled scores; −inf for an empty context): one KV shard's partial for
 * KD_OP_ATTN_MERGE (f2). */
enum { KD_ATTN_LSE = 1 };
typedef struct {
  uint32_t rows, n_heads, n_kv_heads, head_dim, page, pages_per_seq, dtype, flags;
} kd_attr_attention;
/* f2: merge of n_parts attention partials of the
 * same queries over disjoint KV shards: out = Σ_s 2^(lse_s − M)·out_s /
 * Σ_s 2^(lse_s − M), M = max_s lse_s, shards in index order (deterministic). */
typedef struct { uint32_t rows, n_heads, head_dim, n_parts; } kd_attr_attn_merge;
typedef struct {
  uint32_t rows, hidden, n_heads, n_kv_heads, head_dim, page, pages_per_seq, dtype;
  double theta;   /* RoPE base (R12) */
} kd_attr_qkv_rope;  /* X [rows, hidden]; q [rows, n_heads·D]; caches as for rope_append */
typedef struct { uint32_t rows, ffn, dtype, pad_; } kd_attr_silu_mul;  /* gu [rows, 2F] 64-col gate/up blocks */
/* f4 prefill: `seqs` sequences of `seq_len` prompt tokens each;
 * activations have seqs·seq_len rows (row b·seq_len + t). Caches as for
 * rope_append (HND pages of `page` tokens, block_table [seqs, pages_per_seq],
 * pages_per_seq·page ≥ seq_len). The prefill GEMMs are KD_OP_GEMM with
 * M = seqs·seq_len > 256 rows (the tensor-bound tcgen05 kernel). */
typedef struct {
  uint32_t seqs, seq_len, n_heads, n_kv_heads, head_dim, page, pages_per_seq, dtype;
  double theta;
} kd_attr_rope_prefill;
typedef struct {
  uint32_t seqs, seq_len, n_heads, n_kv_heads, head_dim, page, pages_per_seq, dtype;
} kd_attr_prefill_attention;  /* seq_len % 16 == 0, head_dim 64 or 128, page 16 */
typedef struct { uint32_t rows, hidden, n_delta, dtype; } kd_attr_residual_add; /* r fp32 [rows,H] += Σ deltas (dtype: bf16 or fp32) */
/* MoE. route buffer: int32 idx[rows][top_k] then fp32
 * w[rows][top_k]; meta buffer: int32 count[E], offset[E], slot_of[rows][top_k]
 * (grouped row of each (row, choice)), row_of[rows*top_k]; grouped rows are
 * expert-major, ascending row index inside an expert. */
typedef struct { uint32_t rows, hidden, experts, top_k; } kd_attr_moe_route;    /* h bf16 [rows,H], W_r fp32 [E,H] */
typedef struct { uint32_t rows, hidden, experts, top_k; } kd_attr_moe_dispatch; /* xg bf16 [rows*top_k, H] */
typedef struct {
  uint32_t rows_total;  /* rows of xg / yg (= rows * top_k) */
  uint32_t N, K;        /* per-expert W [N, K]; W_experts [experts, N, K] row-major */
  uint32_t experts;     /* groups this GEMM runs: experts expert0 .. expert0 + experts − 1 */
  uint32_t rows_cap;    /* static bound on rows per expert (<= 256) */
  uint32_t dtype;
  /* expert parallelism (SURVEY §8(e) "MoE: EP with P2P dispatch and combine"):
   * the meta block describes meta_experts experts (0 = experts); this GEMM's
   * group j is expert expert0 + j (count at meta[expert0 + j], offset at
   * meta[meta_experts + expert0 + j]); W_experts holds only its experts. */
  uint32_t expert0, meta_experts;
} kd_attr_grouped_gemm;                                                          /* yg bf16 [rows_total, N] */
/* n_parts (0 or 1: one yg): expert-parallel combine reads [yg_0 .. yg_{n_parts−1},
 * route, meta]; expert e's rows are in part e / (experts / n_parts) (each
 * expert device writes its experts' rows of its own yg buffer). */
typedef struct { uint32_t rows, hidden, experts, top_k, n_parts, pad_; } kd_attr_moe_combine;  /* out bf16 [rows, H] */
/* Mamba-2 decode. zxbcdt = in_proj output bf16 [rows, P_in]
 * with columns [z (d_inner) | xBC (d_inner + 2·G·N) | dt (nheads)], P_in =
 * 2·d_inner + 2·G·N + nheads, d_inner = nheads·head_dim. conv_state bf16
 * [rows, d_inner + 2GN, d_conv-1] (oldest first), conv_w bf16 [ch, d_conv],
 * conv_b bf16 [ch]; ssm_state fp32 [rows, nheads, head_dim, N]; dt_bias,
 * A_log, D fp32 [nheads]; norm_w bf16 [d_inner]; xbc bf16 [rows, ch]; y, yn
 * bf16 [rows, d_inner]. The gated norm normalises groups of d_inner/G. */
typedef struct {
  uint32_t rows, nheads, head_dim, d_state, ngroups, d_conv, dtype;
  float eps;
} kd_attr_ssm;

typedef struct {
  uint32_t op;              /* KD_OP_* */
  uint32_t n_reads, n_writes;
  int32_t pin_device;       /* -1: free; else the kernel is fixed there (A4 indirect-access fallback) */
  int32_t template_id;      /* -1: none; kernels with equal ids get one device (A15 repeated layers) */
  uint32_t pad_;
  uint64_t flops;           /* declared algorithmic flops (cost model) */
  const kd_span* reads;
  const kd_span* writes;
  const void* attrs;        /* one of kd_attr_*; copied */
  uint32_t attrs_size;
  uint32_t pad2_;
} kd_kernel_desc;

typedef struct {
  uint32_t src, dst, buf, pad_;
  uint64_t offset, len;     /* one maximal span whose last writer is src (R1-R3) */
} kd_edge;

kd_status kd_graph_create(kd_graph** out);
void kd_graph_destroy(kd_graph* g);
/* Declares a buffer of `bytes` bytes. ids are dense from 0. */
kd_status kd_graph_add_buffer(kd_graph* g, uint64_t bytes, uint32_t flags, uint32_t* id);
/* Declares the next kernel in program order; ids dense from 0. Spans are
 * validated (KD_ERR_RANGE if outside the buffer, KD_ERR_INVALID_ARG if empty);
 * reads and writes may overlap (in-place kernels). */
kd_status kd_graph_add_kernel(kd_graph* g, const kd_kernel_desc* desc, uint32_t* id);
/* Builds the RAW DDG: a global registry of the last writer of every
 * byte; for each kernel in order, every read byte whose last writer w is not
 * the kernel itself yields an edge (w → k); then the kernel's writes update
 * the registry (R2). No WAR/WAW edges (R4). Weights/inputs never written have
 * no writer (R5). After finalize, add_* returns KD_ERR_STATE. */
kd_status kd_graph_finalize(kd_graph* g);
kd_status kd_graph_num_kernels(const kd_graph* g, uint32_t* n);
kd_status kd_graph_num_buffers(const kd_graph* g, uint32_t* n);
/* Edge records sorted by (dst, src, buf, offset). If cap < required, returns
 * KD_ERR_RANGE and writes the required count to *n. */
kd_status kd_graph_edges(const kd_graph* g, kd_edge* out, uint32_t cap, uint32_t* n);

/* ------------------------------------------------------------------ cost / placement
 * Machine description in integers (R7). link matrices are n×n row-major
 * [u*n + g], diagonal ignored. */
typedef struct {
  uint32_t n_dev, pad_;
  const uint64_t* hbm_Bps;      /* [n] HBM bytes/s */
  const uint64_t* tc_flops;     /* [n] tensor flop/s */
  const uint64_t* link_Bps;     /* [n*n] bw_{u,g} (Table 2) */
  const uint64_t* link_lat_ps;  /* [n*n] ℓ_{u,g} (Table 2) */
  uint64_t launch_ps;           /* per-kernel launch floor */
} kd_machine;

/* t_{k,g} (Table 2, replaced by a roofline, A10):
 * t = max(⌈bytes·10¹²/hbm_g⌉, ⌈flops·10¹²/tc_g⌉) + launch_ps, where bytes =
 * union-of-read-spans + union-of-write-spans of kernel k. t_ps is K×n_dev. */
kd_status kd_cost(const kd_graph* g, const kd_machine* m, int64_t* t_ps);

enum { KD_OBJ_AUTO = 0, KD_OBJ_THROUGHPUT = 1, KD_OBJ_LATENCY = 2 };
typedef struct {
  uint32_t n_micro;      /* N ≥ 1 */
  uint32_t objective;    /* AUTO: LATENCY (E7) when N == 1, THROUGHPUT (E6) otherwise (R8) */
  uint64_t max_nodes;    /* search budget (0 = unlimited); exceeding it → KD_ERR_INFEASIBLE */
} kd_place_opts;

/* Objective of a given assignment: E2 T_g = N·Σ t, E3/E4 M_g = N·Σ over cut
 * edges into g of (ℓ + ⌈d_ij·10¹²/bw⌉), E5/E6 max_g max(T_g, M_g) or E7
 * Σ T + Σ M. T and M (nullable) receive n_dev values each. */
kd_status kd_objective(const kd_graph* g, const kd_machine* m, const int32_t* assign,
                       uint32_t n_micro, uint32_t objective, int64_t* obj_ps, int64_t* T_ps, int64_t* M_ps);
/* Exact search over template classes (A15) with pins (A4): branch and bound
 * in lexicographic device order; the optimum returned is the
 * lexicographically smallest assign among optima (R7). */
kd_status kd_place(const kd_graph* g, const kd_machine* m, const kd_place_opts* opts,
                   int32_t* assign, int64_t* objective_ps, uint64_t* nodes_visited);

/* Device-role search (SURVEY §8(a) a1 "search over device roles"; the E6
 * throughput objective, evaluated over role layouts). `g` is ONE
 * memory shard's step graph with rows_per_micro rows per micro-batch. A layout
 * puts every template class (A15) in the memory role or the GEMM role (pins:
 * pin_device 0 = memory, 1 = GEMM) and runs it on `a` memory-role GPUs (each
 * its own rows: sequences are sharded) and `gr` GEMM-role GPUs (weights split
 * over them, all a·rows rows per micro-batch), with N micro-batches:
 *   memory kernel   t = max(⌈(W + A)·10¹²/HBM⌉, ⌈F·10¹²/TC⌉) + launch
 *   GEMM-role kernel t = max(⌈(⌈W/gr⌉ + a·A)·10¹²/HBM⌉, ⌈⌈a·F/gr⌉·10¹²/TC⌉) + launch
 * (W = bytes of its WEIGHT spans, A = its other bytes, F = flops);
 * T_mem = N·Σ t_mem, T_gemm = N·Σ t_gemm; per cut edge of d bytes,
 * memory → GEMM: M_gemm += N·a·(ℓ + ⌈d·10¹²/bw⌉), GEMM → memory:
 * M_mem += N·gr·(ℓ + ⌈⌈d/gr⌉·10¹²/bw⌉); step period = max of the four (N ≥ 2)
 * or their sum (N = 1: nothing overlaps inside one step, R8). gpus = 1 is the
 * monolithic layout (a = 1, gr = 0, no transfers). For every gpus ∈ {1,2,4,8},
 * gpus ≤ max_gpus, the layout with the most tokens per second per GPU
 * (a·N·rows / (gpus·period)) is returned, ties → smallest (a, N, role mask)
 * (mask bit c = class c in the GEMM role, classes in first-use order). The
 * machine's device 0 HBM/TC and link 0→1 are used (homogeneous NVSwitch box).
 * roles receives K values per returned layout (0 memory, 1 GEMM). At most 20
 * free classes (KD_ERR_UNSUPPORTED otherwise). */
typedef struct {
  uint32_t gpus, a, gr, n_micro;
  int64_t period_ps;
  int64_t T_mem_ps, T_gemm_ps, M_mem_ps, M_gemm_ps;
  uint64_t tokens_per_step;   /* a · N · rows_per_micro */
  uint64_t role_mask;
} kd_role_layout;
kd_status kd_place_roles(const kd_graph* g, const kd_machine* m, uint32_t rows_per_micro, uint32_t max_gpus,
                         uint32_t micro_mask, kd_role_layout* best, int32_t* roles, uint32_t cap, uint32_t* n_out);

/* ------------------------------------------------------------------ online monitor
 * Queueing-aware policy switching (§3.4): requests are
 * attributed to the fixed window ⌊t_end/W⌋ in which they finish; at each window
 * boundary the ratio L̄_req / L̄_exec of mean request latency to mean pure
 * execution latency (compute + communication, queueing excluded)
 * selects KD_OBJ_THROUGHPUT when > β, else KD_OBJ_LATENCY; an empty window
 * keeps the policy. Paper defaults W = 300 ms, β = 1.5. Times are
 * integer ns, β = beta_num/beta_den: decisions are exact. Switching itself
 * (re-planning, synchronising the workers at an iteration boundary) is
 * the caller's: it keeps one plan per policy. Errors: KD_ERR_INVALID_ARG;
 * KD_ERR_STATE when a request finishes in a window already evaluated. */
typedef struct kd_monitor kd_monitor;
kd_status kd_monitor_create(uint64_t window_ns, uint32_t beta_num, uint32_t beta_den, uint32_t initial_policy,
                            kd_monitor** out);
kd_status kd_monitor_destroy(kd_monitor* m);
kd_status kd_monitor_record(kd_monitor* m, uint64_t t_end_ns, uint64_t req_latency_ns, uint64_t exec_latency_ns);
/* evaluates every window that ended before now_ns, in order; *policy = current
 * policy, *switches (nullable) = switches so far */
kd_status kd_monitor_poll(kd_monitor* m, uint64_t now_ns, uint32_t* policy, uint32_t* switches);

/* Chunk partition (R10): q = ⌈⌈len/unit⌉/n⌉·unit; chunk c = [c·q, min((c+1)·q, len)),
 * empty chunks dropped. begin_end receives 2·(*n_out) values; cap in chunks. */
kd_status kd_chunks(uint64_t len, uint64_t unit, uint32_t n, uint64_t* begin_end, uint32_t cap, uint32_t* n_out);

/* ------------------------------------------------------------------ plan
 * Deterministic list schedule of (micro-batch i, kernel k) under the cost
 * model (P:380 recv-before/send-after; P:401-402 earlier micro-batch first):
 * one kernel at a time per device, ready-set priority (i, k), one transfer at
 * a time per ordered channel. The global order (start, dev, i, k) is
 * topological; each device executes its subsequence in that order (which
 * makes the spin-waits deadlock free). */
typedef struct kd_plan kd_plan;
typedef struct {
  uint32_t dev, micro, kernel, pad_;
  int64_t start_ps, end_ps;
} kd_sched_entry;
typedef struct {
  uint32_t micro, producer, dst_dev, pad_;
  uint64_t bytes;               /* union of spans the dst device's consumers read */
  int64_t issue_ps, arrival_ps; /* simulated */
} kd_transfer;

/* n_chunks (1..8): chunks per transfer along the consumer's streamable axis
 * (reading R10; the paper streams whole buffers). */
kd_status kd_plan_create(const kd_graph* g, const kd_machine* m, const int32_t* assign,
                         uint32_t n_micro, uint32_t n_chunks, kd_plan** out);
void kd_plan_destroy(kd_plan* p);
kd_status kd_plan_schedule(const kd_plan* p, kd_sched_entry* out, uint32_t cap, uint32_t* n);
kd_status kd_plan_transfers(const kd_plan* p, kd_transfer* out, uint32_t cap, uint32_t* n);
kd_status kd_plan_makespan(const kd_plan* p, int64_t* ps);
/* Chunk table (R10; the a13 handoff). Every transfer's data — the producer's
 * primary output — is viewed as [rows][row_bytes] and each row is cut into
 * column chunks: q = ⌈⌈row_bytes/unit⌉/n_chunks⌉·unit, chunk c = [c·q,
 * min((c+1)·q, row_bytes)), empty chunks dropped. unit = the lcm of the chunk
 * units of the producer's remote chunk-aware consumers (a GEMM's 64·kbs-column
 * k-block, SiLU·mul's 128-column gate/up block, RoPE/append's kv group of
 * (G+2)·D columns, add+RMSNorm's 8 columns), or the whole row without one.
 * count_mode = 1: the producer releases chunk c's flag by the bytes it stored
 * there (complete at rows·(end − begin) per step) and a chunk-aware consumer
 * acquires chunk c right before reading it, inside its kernel, while later
 * chunks are still produced. count_mode = 0 (outputs that are not a dense
 * [rows][cols] block written once: MoE dispatch/grouped GEMM, SSM, fp32, LSE
 * partials, QKV+RoPE): one chunk, released once per signalling CTA. Entries
 * are ordered by (transfer, chunk); if cap is too small → KD_ERR_RANGE with
 * *n = required. */
typedef struct {
  uint32_t transfer;    /* index into kd_plan_transfers */
  uint32_t chunk;       /* ascending within the transfer */
  uint32_t count_mode;  /* 1: byte-count release per chunk; 0: per-CTA release, one chunk */
  uint32_t pad_;
  uint64_t row0, rows;  /* rows [row0, row0 + rows) of the output travel (a GEMM output scattered
                           to memory shards carries only the rows that device reads, R24) */
  uint64_t row_bytes, unit;
  uint64_t begin, end;  /* byte range within every row */
} kd_chunk;
kd_status kd_plan_chunks(const kd_plan* p, kd_chunk* out, uint32_t cap, uint32_t* n);
/* Device workspace the runtime carves into activations, landing slots,
 * flags and kernel scratch. Must be ZERO-initialised once by the caller. */
kd_status kd_plan_workspace_bytes(const kd_plan* p, uint32_t dev, uint64_t* bytes);
/* The carve-up of that workspace (byte offsets from its base; debug / race
 * hardening): control words, per-chunk flags, LOG records, kernel
 * scratch (self-resetting counters), then [act_off, total) = this device's
 * instances of the graph's internal buffers, which include every landing slot
 * (a transfer lands in the destination's own instance of the producer's
 * buffer). Every byte of [act_off, total) is rewritten by its producer (or
 * transfer) before any kernel of the same step reads it, so a caller may
 * overwrite that range between steps (tests poison it with NaN bytes); the
 * ranges before act_off must be left alone. */
typedef struct kd_ws_layout {
  uint64_t ctrl_off, ctrl_bytes, flags_off, flags_bytes, log_off, log_bytes;
  uint64_t scratch_off, scratch_bytes, act_off, total;
} kd_ws_layout;
kd_status kd_plan_workspace_layout(const kd_plan* p, uint32_t dev, kd_ws_layout* out);
/* Whether the caller must bind (buf, dev): 1 for external buffers
 * (WEIGHT/INPUT/OUTPUT/PERSISTENT) touched by a kernel placed on dev. */
kd_status kd_plan_needs_binding(const kd_plan* p, uint32_t buf, uint32_t dev, int32_t* needed);

/* ------------------------------------------------------------------ runtime
 * One runtime drives the logical devices listed at creation. Logical device d
 * runs on CUDA device cuda_ordinal[d]; several logical devices may share one
 * physical GPU ("loopback": same flag protocol, landing slots in the same HBM).
 * Multi-process use: create with n_local = 1 (this rank's logical device) and
 * give every peer's workspace pointer, as mapped in this process (CUDA IPC),
 * with kd_runtime_set_peer_workspace. */
typedef struct kd_runtime kd_runtime;
enum {
  KD_MODE_DISAGG = 0,       /* default: execute the plan                                    */
  KD_MODE_NO_TRANSFER = 1,  /* ablation: peer stores and waits removed (exposed-transfer = DISAGG − this) */
  KD_MODE_LOG = 2           /* DISAGG + per-chunk %globaltimer records (kd_runtime_log, kd_step_stats.wait) */
};
kd_status kd_runtime_create(const kd_plan* p, const uint32_t* local_devs, const int32_t* cuda_ordinal,
                            uint32_t n_local, kd_runtime** out);
void kd_runtime_destroy(kd_runtime* rt);
/* External buffer instance: micro is ignored (use 0) unless the buffer is
 * KD_BUF_PER_MICROBATCH. dev_ptr must stay valid for the runtime lifetime. */
kd_status kd_runtime_bind(kd_runtime* rt, uint32_t buf, uint32_t micro, uint32_t dev, void* dev_ptr);
kd_status kd_runtime_set_workspace(kd_runtime* rt, uint32_t dev, void* dev_ptr, uint64_t bytes);
kd_status kd_runtime_set_peer_workspace(kd_runtime* rt, uint32_t dev, void* mapped_ptr);
/* Multi-process delta replication: the replica of REPLICATED buffer `buf`
 * (micro-batch instance `micro`) on remote device `dev`, as mapped in this
 * process (CUDA IPC). In loopback the runtime uses the local bindings. */
kd_status kd_runtime_set_peer_buffer(kd_runtime* rt, uint32_t buf, uint32_t micro, uint32_t dev, void* mapped_ptr);
kd_status kd_runtime_set_mode(kd_runtime* rt, uint32_t mode);
/* 1 = capture each device's step into a CUDA graph on first kd_step and
 * replay it afterwards (default 1). */
kd_status kd_runtime_set_graph(kd_runtime* rt, int32_t enable);
/* Resolves every pointer, encodes TMA descriptors, enables peer access. */
kd_status kd_runtime_prepare(kd_runtime* rt);
/* Execution strategy (launch overhead P:281):
 *  KD_EXEC_GRAPH (default): one kernel per schedule entry, replayed from a
 *    per-device CUDA graph with programmatic dependent launch;
 *  KD_EXEC_MEGAKERNEL: ONE persistent cooperative launch per device per step
 *    executes the device's whole static schedule (every op a task, in-kernel
 *    dependency waits on per-task completion counters, weights / KV pages
 *    streamed across task boundaries). Supported: single-device schedules
 *    (no cross-device transfers) of bf16 ADD_RMSNORM, GEMM (M <= 128,
 *    K % 128 == 0, N % 8 == 0), ROPE_APPEND, ATTENTION (head_dim 64/128, no
 *    LSE flag), SILU_MUL and RESIDUAL_ADD; anything else → KD_ERR_UNSUPPORTED
 *    at kd_runtime_prepare. Its outputs match the per-kernel path's within
 *    rounding (add+RMSNorm, RoPE, SiLU and residual add are bitwise identical;
 *    the GEMM split-K and attention merge orders differ) and are bitwise
 *    reproducible step to step.
 * The megakernel needs its own zeroed device workspace per local device:
 * after kd_runtime_prepare, kd_runtime_exec_workspace_bytes gives the size;
 * kd_runtime_set_exec_workspace binds it (caller-owned, 256-byte aligned,
 * zero-initialised; borrowed for the runtime's lifetime). kd_step before that
 * → KD_ERR_STATE. Device-side watchdogs (a dependency or pipeline wait that
 * does not complete in ~20 s) record the runtime error word and abort the
 * launch (kd_runtime_check reports KD_ERR_TIMEOUT). */
enum { KD_EXEC_GRAPH = 0, KD_EXEC_MEGAKERNEL = 1 };
kd_status kd_runtime_set_exec(kd_runtime* rt, uint32_t exec);
kd_status kd_runtime_exec_workspace_bytes(kd_runtime* rt, uint32_t dev, uint64_t* bytes);
kd_status kd_runtime_set_exec_workspace(kd_runtime* rt, uint32_t dev, void* dev_ptr, uint64_t bytes);
/* KD_EXEC_MEGAKERNEL: tasks, dynamic shared memory bytes per CTA and grid
 * (one CTA per SM) of local device j's megakernel (after prepare). */
kd_status kd_runtime_exec_info(kd_runtime* rt, uint32_t j, uint32_t* n_tasks, uint32_t* smem_bytes, uint32_t* grid);
/* Per-step statistics (filled by kd_step when `stats` is non-NULL; that call
 * synchronises every local device). Times are ns; index j = local device j.
 *  step_ns[j]: device time of the step on device j (CUDA events on its stream);
 *  wait_ns[j]: KD_MODE_LOG only (else 0): Σ over device j's incoming (transfer,
 *    chunk) of the first acquirer's stall (acquire − wait start) — the exposed
 *    transfer time the consumer observed; chunk_waits[j] counts them;
 *  link_bytes[u·n_dev + v]: bytes streamed u → v per step (the plan's transfers,
 *    all logical devices; diagonal 0). */
#define KD_STATS_MAX_DEV 8
typedef struct {
  uint64_t step_id;
  uint32_t n_local, n_dev;
  uint64_t step_ns[KD_STATS_MAX_DEV];
  uint64_t wait_ns[KD_STATS_MAX_DEV];
  uint32_t chunk_waits[KD_STATS_MAX_DEV];
  uint64_t link_bytes[KD_STATS_MAX_DEV * KD_STATS_MAX_DEV];
} kd_step_stats;
/* Enqueue decode step `step_id` on streams[j] for local device j (async unless
 * stats is non-NULL). step_id counts kd_step calls on this runtime from 0; the
 * device epoch of the step (the value its flags are released to) is step_id + 1.
 * A step_id other than the next one → KD_ERR_INVALID_ARG (steps are issued in
 * order; UINT64_MAX = "the next one"). Device errors (flag / barrier
 * watchdogs) surface at kd_runtime_check or the next kd_step. */
kd_status kd_step(kd_runtime* rt, void* const* streams, uint64_t step_id, kd_step_stats* stats);
kd_status kd_runtime_check(kd_runtime* rt);
/* KD_MODE_LOG records of the last step (call after a sync), one per (incoming
 * transfer, chunk) of every local device, ordered by (dev, transfer, chunk):
 * epoch = the step's device epoch seen by the first consumer acquire (0 if not
 * yet acquired), t_wait (that acquirer's wait start), t_acquire, t_release (the
 * producer's last release into the chunk, %globaltimer ns — chunk complete).
 * R10's "ascending consumption": every consumer acquires a transfer's chunks in
 * ascending order. Errors: KD_ERR_STATE if the mode is not LOG, KD_ERR_RANGE
 * with *n = required if cap is too small. */
typedef struct {
  uint32_t dev, transfer, chunk, pad_;
  uint64_t epoch, t_wait, t_acquire, t_release;
} kd_log_record;
kd_status kd_runtime_log(kd_runtime* rt, kd_log_record* out, uint32_t cap, uint32_t* n);
/* Number of kernel launches one kd_step enqueues on local device j. */
kd_status kd_runtime_launch_count(const kd_runtime* rt, uint32_t j, uint32_t* n);
/* Profiling: record CUDA events around every launch of `op` (0 = off) on the
 * stream it is launched on; kd_runtime_op_time returns the summed event time
 * (ms) and launch count since the last reset (events are read after a sync). */
kd_status kd_runtime_profile_op(kd_runtime* rt, uint32_t op);
kd_status kd_runtime_op_time(kd_runtime* rt, double* ms, uint64_t* launches);

/* CUDA IPC helpers for the multi-process runtime (one process per GPU under
 * torchrun): export the allocation that contains dev_ptr (handle: 64 opaque
 * bytes written to handle64, offset: dev_ptr minus the allocation base), and
 * map a peer's handle into this process (returns base + offset). The mapping
 * is released with kd_ipc_close(mapped_ptr). Errors: KD_ERR_CUDA. */
kd_status kd_ipc_get_handle(const void* dev_ptr, void* handle64, uint64_t* offset);
kd_status kd_ipc_open(const void* handle64, uint64_t offset, void** mapped_ptr);
kd_status kd_ipc_close(void* mapped_ptr);

/* Programmatic dependent launch for every kernel of the path (default on):
 * each kernel lets its successor launch early and waits for its predecessor
 * with griddepcontrol.wait before touching dependent memory; the GEMM streams
 * its first ring of weight tiles before that wait. Takes effect for launches
 * (and graph captures) made after the call. */
kd_status kd_set_pdl(int32_t enable);

/* Debug: when dev_buf is non-NULL, every subsequent GEMM launch writes 16
 * %globaltimer stamps per CTA (entry, setup, first/last TMA, first full wait,
 * last commit, per-segment epilogue start/end, fixup start/end, exit) to
 * dev_buf[cta*32 + slot] (u64, >= 148*32 entries). NULL disables (default). */
kd_status kd_debug_gemm_trace(void* dev_buf);
/* Debug: step timeline. When dev_buf is non-NULL (device, zeroed, `bytes`
 * long), launch i made after this call (e.g. the launches captured into a
 * step graph) writes %globaltimer stamps per CTA to dev_buf[i*16384 + cta*32 +
 * slot] (u64): GEMMs the kd_debug_gemm_trace slots, attention [0] entry, [1]
 * producer past its dependency wait, [2] producer done, [3] epilogue done, [4]
 * consumers done (max over CTAs' warps), [5]/[6] and [7]/[8] the epilogue
 * warp's combine-slot acquire / done of its last two items, [9] its last split
 * counter atomic. Launches beyond bytes/131072 are not
 * traced. kd_debug_timeline_kinds returns each traced launch's kind: 100 +
 * rope + 2·norm (cluster split-K GEMM), 200 + silu (stream-K GEMM), 300
 * (decode attention). Off by default; NULL turns it off and clears the list. */
kd_status kd_debug_timeline(void* dev_buf, uint64_t bytes);
kd_status kd_debug_timeline_kinds(int32_t* out, uint32_t cap, uint32_t* n);
/* Debug: KD_EXEC_MEGAKERNEL timeline. dev_buf (device, >= n_tasks·grid·5·4
 * u64, see kd_runtime_exec_info; NULL = off) receives, for every (task, CTA,
 * role ∈ {loader, MMA, merge, workers}), the %globaltimer ns at the role's task
 * start, after its dependency wait (0 if it waited none) and at its end; role 4
 * = the GEMM epilogue of the CTA's last piece (TMEM ready, partial published,
 * all partials present, fold done). */
kd_status kd_debug_mega_trace(kd_runtime* rt, uint32_t j, void* dev_buf);

/* Tiling the library picks for a plain decode GEMM Y[M,N] = X[M,K]·W[N,K]ᵀ on
 * the current device (a4/a7/a9/a10): out[0] = kernel (1 = dense tokens-as-rows
 * cluster split-K, 0 = stream-K), out[1] = split (cluster size), out[2] = n_t
 * (output columns per tile), out[3] = tiles, out[4] = pipeline stages,
 * out[5] = dynamic smem bytes. Needs a CUDA device (queries co-resident
 * clusters). Environment overrides for tuning: KD_GEMM_TILE="split,n_t",
 * KD_GEMM_STREAMK=1. Errors: KD_ERR_INVALID_ARG (NULL), KD_ERR_UNSUPPORTED. */
kd_status kd_gemm_tiling(uint32_t M, uint32_t N, uint32_t K, int32_t* out6);

/* ------------------------------------------------------------------ single ops
 * Direct entry points to the device kernels the runtime launches (for parity
 * tests and micro-benchmarks). Pointers are device pointers; layouts as in
 * the kd_attr_* comments. `scratch` is a ZERO-initialised device buffer of at
 * least kd_op_scratch_bytes(op, attrs) bytes (left zeroed on return). */
kd_status kd_op_scratch_bytes(uint32_t op, const void* attrs, uint64_t* bytes);
/* a3: r' = r + Σ_i deltas[i] (fp32, in place, index order; deltas is a host array of
 * n_delta device pointers, may be NULL when n_delta == 0), h = r'/sqrt(mean r'^2 + eps)·gamma */
kd_status kd_op_add_rmsnorm(const kd_attr_add_rmsnorm* a, float* r, const void* const* deltas,
                            const void* gamma, void* h, void* stream);
/* a4/a7/a9/a10: Y[M,N] = X[M,K]·W[N,K]ᵀ, bf16 in, fp32 accumulate (tcgen05, TMEM), bf16 out. */
/* a4+a5 fused: the QKV GEMM whose epilogue rotates q/k (NeoX RoPE) and appends
 * k/v to the paged cache; W_qkv rows pair-interleaved per head (see
 * KD_OP_QKV_ROPE). bf16 only. Errors: KD_ERR_UNSUPPORTED when no cluster
 * tiling exists for the shape. */
kd_status kd_op_qkv_rope(const kd_attr_qkv_rope* a, const void* X, const void* W, const int32_t* block_table,
                         const int32_t* seq_len, void* q_out, void* k_cache, void* v_cache, void* scratch,
                         void* stream);
/* a9+a8 fused: a [M, N/2] = silu(g)·u of the bf16-rounded gate/up GEMM output
 * (same bits as kd_op_gemm then kd_op_silu_mul). bf16 only; scratch as for the
 * plain GEMM of the same attrs. */
kd_status kd_op_gemm_silu(const kd_attr_gemm* a, const void* X, const void* W, void* out, void* scratch,
                          void* stream);
kd_status kd_op_gemm(const kd_attr_gemm* a, const void* X, const void* W, void* Y,
                     void* scratch, void* stream);
/* a7/a10 + a3 fused (KD_OP_GEMM_RMSNORM): r (fp32 [M,N], in place) += bf16(X·Wᵀ),
 * h [M,N] = RMSNorm(r)·gamma. One cluster split-K launch; the per-token Σr² is
 * completed across its CTAs after an in-kernel grid barrier (all CTAs are
 * co-resident by construction). bf16 only, N % 8 == 0; r and gamma 16-byte
 * aligned; scratch as kd_op_scratch_bytes(KD_OP_GEMM_RMSNORM). Errors:
 * KD_ERR_UNSUPPORTED when no co-resident cluster tiling exists for the shape.
 * The in-kernel grid barrier needs every CTA of the launch resident at once:
 * do not run it concurrently with kernels that wait on its completion. */
kd_status kd_op_gemm_rmsnorm(const kd_attr_gemm_rmsnorm* a, const void* X, const void* W, float* r,
                             const void* gamma, void* h, void* scratch, void* stream);
/* a5: NeoX RoPE of q and k at pos = seq_len[b]-1, append (k_rot, v) to the
 * HND paged cache [pages][Hkv][page][D]; q_out [rows, Hq·D]. */
kd_status kd_op_rope_append(const kd_attr_rope_append* a, const void* qkv, const int32_t* block_table,
                            const int32_t* seq_len, void* q_out, void* k_cache, void* v_cache, void* stream);
/* a6: split-KV paged GQA decode attention, deterministic fixed-order combine. */
kd_status kd_op_attention(const kd_attr_attention* a, const void* q, const void* k_cache, const void* v_cache,
                          const int32_t* block_table, const int32_t* seq_len, void* out,
                          void* scratch, void* stream);
/* f2: merge n_parts KD_ATTN_LSE partials (parts: n_parts device pointers to
 * [out|lse] buffers) into out bf16 [rows, n_heads·head_dim]. */
kd_status kd_op_attn_merge(const kd_attr_attn_merge* a, const void* const* parts, void* out, void* stream);
/* a8: a[:, 64j+i] = silu(gu[:, 128j+i]) · gu[:, 128j+64+i] */
kd_status kd_op_silu_mul(const kd_attr_silu_mul* a, const void* gu, void* out, void* stream);
/* f4: KD_OP_ROPE_PREFILL and KD_OP_PREFILL_ATTENTION as single launches (bf16). */
kd_status kd_op_rope_prefill(const kd_attr_rope_prefill* a, const void* qkv, const int32_t* block_table, void* q_out,
                             void* k_cache, void* v_cache, void* stream);
kd_status kd_op_prefill_attention(const kd_attr_prefill_attention* a, const void* q, const void* k_cache,
                                  const void* v_cache, const int32_t* block_table, void* out, void* stream);
/* C1.11: r += Σ_i deltas[i] (index order) */
kd_status kd_op_residual_add(const kd_attr_residual_add* a, float* r, const void* const* deltas, void* stream);
/* a12: conv step: window = [state, x]; xbc = silu(window·w + b); state ← window[1:] (in place) */
kd_status kd_op_ssm_conv(const kd_attr_ssm* a, const void* zxbcdt, const void* conv_w, const void* conv_b,
                         void* conv_state, void* xbc, void* stream);
/* a12: S ← S·exp(softplus(dt+b)·(−e^{A_log})) + softplus(dt+b)·x⊗B; y = S·C + D·x (in place on S) */
kd_status kd_op_ssm_update(const kd_attr_ssm* a, const void* xbc, const void* zxbcdt, const float* dt_bias,
                           const float* A_log, const float* D, float* ssm_state, void* y, void* stream);
/* a12: yn = groupwise RMSNorm(y · silu(z)) · norm_w */
kd_status kd_op_gated_norm(const kd_attr_ssm* a, const void* y, const void* zxbcdt, const void* norm_w, void* yn,
                           void* stream);
/* a11 router: logits = h·W_rᵀ in fp32 (fixed-order warp reduction), top_k by
 * logit (ties → lower expert index), weights = softmax over the selected. */
kd_status kd_op_moe_route(const kd_attr_moe_route* a, const void* h, const float* w_router, void* route, void* stream);
/* a11 dispatch: slot map (meta) + gather of h rows into expert-major xg. */
kd_status kd_op_moe_dispatch(const kd_attr_moe_dispatch* a, const void* h, const void* route, void* xg, void* meta,
                             void* stream);
/* Bytes of the dispatch meta block (256-byte aligned). In a kernel graph the
 * dispatch op writes ONE buffer [meta | xg] (its primary output, so both cross
 * devices together); xg starts at this offset. */
kd_status kd_moe_meta_bytes(uint32_t rows, uint32_t experts, uint32_t top_k, uint64_t* bytes);
/* a11 grouped GEMM: for every expert e, yg[off_e + j] = xg[off_e + j]·W_eᵀ for
 * j < count_e (off/count from meta, read on device). tcgen05 stream-K over all
 * experts' tiles in one launch. */
kd_status kd_op_grouped_gemm(const kd_attr_grouped_gemm* a, const void* xg, const void* w_experts, const void* meta,
                             void* yg, void* scratch, void* stream);
/* a11 combine: out[b] = Σ_j w[b][j]·yg[slot_of[b][j]], ascending expert order. */
kd_status kd_op_moe_combine(const kd_attr_moe_combine* a, const void* yg, const void* route, const void* meta,
                            void* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* KD_H_ */
