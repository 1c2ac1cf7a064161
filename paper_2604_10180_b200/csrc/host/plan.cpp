// plan.cpp — deterministic list schedule of (micro-batch, kernel) entries and
// the per-device workspace layout (§3.3: recv before k / send after k
// on communication streams; pipelined requests with earlier-first
// priority; readings R3, R4, R7, R10, R11 in DESIGN.md).
#include <algorithm>
#include <set>

#include "internal.hpp"

using namespace kd;

namespace kd {
kd_status op_scratch_bytes(uint32_t op, const std::vector<uint8_t>& attrs, u64* bytes);  // ops.cu

static u64 align_up(u64 x, u64 a) { return (x + a - 1) / a * a; }

template <typename T>
static bool attrs_as(const Kernel& k, T* a) {
  if (k.attrs.size() != sizeof(T)) return false;
  std::memcpy(a, k.attrs.data(), sizeof(T));
  return true;
}

// Producers whose primary output is a dense bf16 [rows][cols] block written
// exactly once per step release per chunk in bytes (COUNT); the device code
// of each (elementwise.cu, attention.cu, gemm.cu) tallies its stores the
// same way. Everything else releases once per signalling CTA.
bool op_count_geometry(const Kernel& k, u64* rows, u64* row_bytes) {
  switch (k.op) {
    case KD_OP_ADD_RMSNORM: {
      kd_attr_add_rmsnorm a;
      if (!attrs_as(k, &a) || a.dtype != KD_BF16) return false;
      *rows = a.rows, *row_bytes = 2ull * a.hidden;
      return true;
    }
    case KD_OP_GEMM:
    case KD_OP_GEMM_SILU: {
      kd_attr_gemm a;
      // (M > 256: the f4 prefill kernel releases once per CTA — CTA mode)
      if (!attrs_as(k, &a) || a.dtype != KD_BF16 || a.M > 256) return false;
      *rows = a.M, *row_bytes = 2ull * (k.op == KD_OP_GEMM_SILU ? a.N / 2 : a.N);
      return true;
    }
    case KD_OP_GEMM_RMSNORM: {
      kd_attr_gemm_rmsnorm a;
      if (!attrs_as(k, &a) || a.dtype != KD_BF16) return false;
      *rows = a.M, *row_bytes = 2ull * a.N;
      return true;
    }
    case KD_OP_ROPE_APPEND: {
      kd_attr_rope_append a;
      if (!attrs_as(k, &a) || a.dtype != KD_BF16) return false;
      *rows = a.rows, *row_bytes = 2ull * a.n_heads * a.head_dim;
      return true;
    }
    case KD_OP_ATTENTION: {
      kd_attr_attention a;
      if (!attrs_as(k, &a) || a.dtype != KD_BF16 || (a.flags & KD_ATTN_LSE)) return false;
      *rows = a.rows, *row_bytes = 2ull * a.n_heads * a.head_dim;
      return true;
    }
    case KD_OP_ATTN_MERGE: {
      kd_attr_attn_merge a;
      if (!attrs_as(k, &a)) return false;
      *rows = a.rows, *row_bytes = 2ull * a.n_heads * a.head_dim;
      return true;
    }
    case KD_OP_SILU_MUL: {
      kd_attr_silu_mul a;
      if (!attrs_as(k, &a) || a.dtype != KD_BF16) return false;
      *rows = a.rows, *row_bytes = 2ull * a.ffn;
      return true;
    }
  }
  return false;
}

// Consumer chunk units (SURVEY §8(a) a2 "chunk axis = consumer's streamable
// axis"): a GEMM reads X by k-blocks of 64·kbs columns (kbs = 2 while the MMA
// N ≤ 128); SiLU·mul reads 128-column gate/up blocks; RoPE/append reads a kv
// group's (G+2)·D columns; add+RMSNorm and the residual add read 8-column
// groups. The input row must be the producer's row (row_bytes).
u64 op_consumer_unit(const Kernel& k, uint32_t ri, u64 row_bytes) {
  switch (k.op) {
    case KD_OP_GEMM:
    case KD_OP_GEMM_SILU: {
      kd_attr_gemm a;
      if (ri != 0 || !attrs_as(k, &a) || a.dtype != KD_BF16 || 2ull * a.K != row_bytes || a.M > 256) return 0;
      return ((a.M + 15) / 16 * 16 <= 128 ? 2ull : 1ull) * 64 * 2;
    }
    case KD_OP_GEMM_RMSNORM: {
      kd_attr_gemm_rmsnorm a;
      if (ri != 0 || !attrs_as(k, &a) || a.dtype != KD_BF16 || 2ull * a.K != row_bytes) return 0;
      return ((a.M + 15) / 16 * 16 <= 128 ? 2ull : 1ull) * 64 * 2;
    }
    case KD_OP_QKV_ROPE: {
      kd_attr_qkv_rope a;
      if (ri != 0 || !attrs_as(k, &a) || a.dtype != KD_BF16 || 2ull * a.hidden != row_bytes) return 0;
      return ((a.rows + 15) / 16 * 16 <= 128 ? 2ull : 1ull) * 64 * 2;
    }
    case KD_OP_ADD_RMSNORM: {
      kd_attr_add_rmsnorm a;
      if (!attrs_as(k, &a) || a.dtype != KD_BF16 || ri < 1 || ri > a.n_delta || 2ull * a.hidden != row_bytes) return 0;
      return 16;
    }
    case KD_OP_RESIDUAL_ADD: {
      kd_attr_residual_add a;
      if (!attrs_as(k, &a) || a.dtype != KD_BF16 || ri < 1 || ri > a.n_delta || 2ull * a.hidden != row_bytes) return 0;
      return 16;
    }
    case KD_OP_SILU_MUL: {
      kd_attr_silu_mul a;
      if (ri != 0 || !attrs_as(k, &a) || a.dtype != KD_BF16 || 4ull * a.ffn != row_bytes) return 0;
      return 256;
    }
    case KD_OP_ROPE_APPEND: {
      kd_attr_rope_append a;
      if (ri != 0 || !attrs_as(k, &a) || a.dtype != KD_BF16 || a.n_kv_heads == 0) return 0;
      if (2ull * (a.n_heads + 2ull * a.n_kv_heads) * a.head_dim != row_bytes) return 0;
      return 2ull * (a.n_heads / a.n_kv_heads + 2) * a.head_dim;
    }
  }
  return 0;
}

u64 op_delta_bytes(const Kernel& k, uint32_t wi) {
  if (wi >= k.writes.size()) return 0;
  if ((k.op == KD_OP_ROPE_APPEND || k.op == KD_OP_QKV_ROPE) && (wi == 1 || wi == 2)) {
    uint32_t rows = 0, hkv = 0, hd = 0, dt = 0;
    if (k.op == KD_OP_ROPE_APPEND) {
      kd_attr_rope_append a;
      if (!attrs_as(k, &a)) return k.writes[wi].len;
      rows = a.rows, hkv = a.n_kv_heads, hd = a.head_dim, dt = a.dtype;
    } else {
      kd_attr_qkv_rope a;
      if (!attrs_as(k, &a)) return k.writes[wi].len;
      rows = a.rows, hkv = a.n_kv_heads, hd = a.head_dim, dt = a.dtype;
    }
    return std::min<u64>(k.writes[wi].len, (u64)rows * hkv * hd * (dt == KD_F32 ? 4 : 2));
  }
  return k.writes[wi].len;
}

bool op_row_filter(const Kernel& k) {
  return k.op == KD_OP_GEMM || k.op == KD_OP_GEMM_SILU || k.op == KD_OP_GEMM_RMSNORM;
}

bool buf_replicated(const kd_graph& g, uint32_t buf) {
  return (g.buffers[buf].flags & (KD_BUF_REPLICATED | KD_BUF_PERSISTENT)) == (KD_BUF_REPLICATED | KD_BUF_PERSISTENT);
}

u64 delta_of(const kd_graph& g, uint32_t src, uint32_t buf) {
  const Kernel& K = g.kernels[src];
  u64 d = 0;
  for (uint32_t wi = 0; wi < K.writes.size(); ++wi)
    if (K.writes[wi].buf == buf) d += op_delta_bytes(K, wi);
  return d;
}

static u64 gcd_u64(u64 a, u64 b) {
  while (b) {
    u64 t = a % b;
    a = b;
    b = t;
  }
  return a;
}
}  // namespace kd

extern "C" {

kd_status kd_plan_create(const kd_graph* g, const kd_machine* m, const int32_t* assign, uint32_t n_micro,
                         uint32_t n_chunks, kd_plan** out) {
  if (!g || !assign || !out) return fail(KD_ERR_INVALID_ARG, "kd_plan_create: NULL argument");
  if (!g->finalized) return fail(KD_ERR_STATE, "kd_plan_create: graph not finalized");
  if (!machine_valid(m) || n_micro == 0) return fail(KD_ERR_INVALID_ARG, "kd_plan_create: bad machine/n_micro");
  if (n_chunks == 0 || n_chunks > kMaxPlanChunks)
    return fail(KD_ERR_INVALID_ARG, "kd_plan_create: n_chunks must be 1.." + std::to_string(kMaxPlanChunks));
  const uint32_t K = (uint32_t)g->kernels.size(), n = m->n_dev, N = n_micro;
  for (uint32_t k = 0; k < K; ++k)
    if (assign[k] < 0 || (uint32_t)assign[k] >= n) return fail(KD_ERR_INVALID_ARG, "kd_plan_create: bad assign");
  // R6: every kernel touching a PERSISTENT buffer sits on one device, unless
  // the buffer is REPLICATED (one replica per device, deltas propagated)
  {
    std::map<uint32_t, int32_t> dev_of_buf;
    for (uint32_t k = 0; k < K; ++k) {
      const Kernel& Kk = g->kernels[k];
      for (const auto* v : {&Kk.reads, &Kk.writes})
        for (const auto& s : *v)
          if ((g->buffers[s.buf].flags & KD_BUF_PERSISTENT) && !buf_replicated(*g, s.buf)) {
            auto it = dev_of_buf.find(s.buf);
            if (it == dev_of_buf.end())
              dev_of_buf[s.buf] = assign[k];
            else if (it->second != assign[k])
              return fail(KD_ERR_UNSUPPORTED, "kd_plan_create: PERSISTENT buffer touched from two devices (R6)");
          }
    }
  }

  auto* p = new kd_plan();
  p->g = g;
  p->n_dev = n;
  p->n_micro = N;
  p->n_chunks = n_chunks;
  p->assign.assign(assign, assign + K);

  // predecessors and transfers (producer k, remote device d) = union of spans
  // (R3) + the deltas of replicated buffers read there (once per buffer)
  std::vector<std::vector<uint32_t>> preds(K);
  std::map<std::pair<uint32_t, uint32_t>, std::vector<Span>> xspans;
  std::map<std::pair<uint32_t, uint32_t>, std::set<uint32_t>> xrepl;  // (k, dev) -> replicated bufs
  for (const auto& e : g->edges) {
    auto& pv = preds[e.dst];
    if (std::find(pv.begin(), pv.end(), e.src) == pv.end()) pv.push_back(e.src);
    uint32_t gd = assign[e.dst];
    if (gd == (uint32_t)assign[e.src]) continue;
    if (buf_replicated(*g, e.buf)) {
      xrepl[{e.src, gd}].insert(e.buf);
      xspans[{e.src, gd}];  // the transfer exists even without a primary-output span
    } else {
      xspans[{e.src, gd}].push_back({e.buf, e.offset, e.len});
    }
  }
  std::vector<std::vector<std::pair<uint32_t, u64>>> out_x(K);  // k -> [(dev, bytes)] ascending dev
  for (auto& kv : xspans) {
    u64 b = union_bytes(kv.second);
    for (uint32_t rb : xrepl[kv.first]) b += delta_of(*g, kv.first.first, rb);
    out_x[kv.first.first].push_back({kv.first.second, b});
  }

  std::vector<i64> t(K);
  for (uint32_t k = 0; k < K; ++k) t[k] = kernel_time(*g, *m, k, assign[k]);

  // ---- discrete-event list schedule (same semantics as oracle/schedule.py)
  const i64 UNSET = -1;
  std::vector<i64> end((size_t)N * K, UNSET);
  std::map<std::tuple<uint32_t, uint32_t, uint32_t>, i64> arrival;  // (i, producer, dev)
  std::map<std::tuple<uint32_t, uint32_t, uint32_t>, i64> issue;
  std::vector<i64> chan_free((size_t)n * n, 0);
  struct Run {
    bool on = false;
    i64 e = 0;
    uint32_t i = 0, k = 0;
  };
  std::vector<Run> running(n);
  std::set<std::pair<uint32_t, uint32_t>> todo;
  for (uint32_t i = 0; i < N; ++i)
    for (uint32_t k = 0; k < K; ++k) todo.insert({i, k});
  i64 tau = 0;
  auto available = [&](uint32_t i, uint32_t k, i64 now) {
    uint32_t gd = assign[k];
    for (uint32_t q : preds[k]) {
      i64 e = end[(size_t)i * K + q];
      if (e == UNSET || e > now) return false;
      if ((uint32_t)assign[q] != gd && arrival.at({i, q, gd}) > now) return false;
    }
    return true;
  };
  size_t n_running = 0;
  while (!todo.empty() || n_running) {
    // 1) completions in (end, i, k, dev) order issue their transfers
    std::vector<std::tuple<i64, uint32_t, uint32_t, uint32_t>> fin;
    for (uint32_t d = 0; d < n; ++d)
      if (running[d].on && running[d].e <= tau) fin.emplace_back(running[d].e, running[d].i, running[d].k, d);
    std::sort(fin.begin(), fin.end());
    for (const auto& f : fin) {
      i64 e = std::get<0>(f);
      uint32_t i = std::get<1>(f), k = std::get<2>(f), d = std::get<3>(f);
      running[d].on = false;
      --n_running;
      for (const auto& x : out_x[k]) {
        uint32_t u = assign[k], v = x.first;
        i64 st = std::max(e, chan_free[(size_t)u * n + v]);
        i64 arr = st + edge_cost(*m, x.second, u, v);
        chan_free[(size_t)u * n + v] = arr;
        arrival[{i, k, v}] = arr;
        issue[{i, k, v}] = e;
      }
    }
    // 2) idle devices start their smallest available (i, k)  (R11)
    for (uint32_t d = 0; d < n; ++d) {
      if (running[d].on) continue;
      for (auto it = todo.begin(); it != todo.end(); ++it) {
        uint32_t i = it->first, k = it->second;
        if ((uint32_t)assign[k] != d || !available(i, k, tau)) continue;
        i64 e = tau + t[k];
        end[(size_t)i * K + k] = e;
        running[d] = {true, e, i, k};
        ++n_running;
        p->sched.push_back({d, i, k, 0, tau, e});
        todo.erase(it);
        break;
      }
    }
    // 3) next event
    i64 nxt = -1;
    for (uint32_t d = 0; d < n; ++d)
      if (running[d].on && running[d].e > tau && (nxt < 0 || running[d].e < nxt)) nxt = running[d].e;
    for (const auto& a : arrival)
      if (a.second > tau && (nxt < 0 || a.second < nxt)) nxt = a.second;
    if (nxt < 0) {
      if (!todo.empty()) {
        delete p;
        return fail(KD_ERR_INFEASIBLE, "kd_plan_create: schedule deadlock");
      }
      break;
    }
    tau = nxt;
  }
  std::sort(p->sched.begin(), p->sched.end(), [](const kd_sched_entry& a, const kd_sched_entry& b) {
    if (a.start_ps != b.start_ps) return a.start_ps < b.start_ps;
    if (a.dev != b.dev) return a.dev < b.dev;
    if (a.micro != b.micro) return a.micro < b.micro;
    return a.kernel < b.kernel;
  });
  for (const auto& s : p->sched) p->makespan = std::max(p->makespan, s.end_ps);
  for (uint32_t i = 0; i < N; ++i)
    for (uint32_t k = 0; k < K; ++k)
      for (const auto& x : out_x[k]) {
        kd_transfer tr{i, k, x.first, 0, x.second, issue[{i, k, x.first}], arrival[{i, k, x.first}]};
        p->transfers.push_back(tr);
      }

  // ---- chunk tables (R10): per producer, the unit is the lcm of its remote
  // chunk-aware consumers' units (reads of its whole primary output whose
  // bytes all come from it); every transfer of a producer shares the table
  {
    std::map<uint32_t, u64> unit_of;  // producer -> lcm unit (bytes)
    std::map<std::pair<uint32_t, uint32_t>, std::set<uint32_t>> srcs;  // (consumer, buf) -> producers
    for (const auto& e : g->edges) srcs[{e.dst, e.buf}].insert(e.src);
    for (uint32_t k = 0; k < K; ++k) {
      const Kernel& C = g->kernels[k];
      for (uint32_t ri = 0; ri < C.reads.size(); ++ri) {
        const Span& sp = C.reads[ri];
        auto it = srcs.find({k, sp.buf});
        if (it == srcs.end() || it->second.size() != 1) continue;
        const uint32_t src = *it->second.begin();
        if (assign[src] == assign[k]) continue;
        const Kernel& P = g->kernels[src];
        u64 rows = 0, rb = 0;
        if (P.writes.empty() || !op_count_geometry(P, &rows, &rb)) continue;
        const Span& w0 = P.writes[0];
        // the consumer reads whole rows of the producer's output (all of them,
        // or its row span of a scattered GEMM output)
        if (sp.buf != w0.buf || sp.off < w0.off || sp.off + sp.len > w0.off + w0.len || rows * rb != w0.len ||
            (sp.off - w0.off) % rb || sp.len % rb)
          continue;
        const u64 u = op_consumer_unit(C, ri, rb);
        if (!u) continue;
        u64& cur = unit_of[src];
        cur = cur ? cur / gcd_u64(cur, u) * u : u;
      }
    }
    p->xchunks.resize(p->transfers.size());
    for (uint32_t t = 0; t < p->transfers.size(); ++t) {
      const kd_transfer& tr = p->transfers[t];
      const Kernel& P = g->kernels[tr.producer];
      auto& X = p->xchunks[t];
      const u64 len = P.writes.empty() ? 0 : P.writes[0].len;
      u64 rows = 0, rb = 0;
      bool mirrors = false;  // a producer mirroring replicated-buffer deltas releases per CTA
      for (const auto& w : P.writes)
        if (buf_replicated(*g, w.buf)) mirrors = true;
      if (!mirrors && op_count_geometry(P, &rows, &rb) && rows * rb == len && rb > 0) {
        X.count = true;
        X.row0 = 0;
        X.rows = rows;
        X.row_bytes = rb;
        if (op_row_filter(P)) {  // only the rows the destination's consumers read (one contiguous range)
          const Span& w0 = P.writes[0];
          u64 lo = ~0ull, hi = 0, covered = 0;
          std::vector<Span> sp;
          for (const auto& e : g->edges)
            if (e.src == tr.producer && (uint32_t)assign[e.dst] == tr.dst_dev && e.buf == w0.buf)
              sp.push_back({e.buf, e.offset, e.len});
          for (const auto& kv : span_union(sp))
            for (const auto& iv : kv.second) {
              lo = std::min(lo, iv.s);
              hi = std::max(hi, iv.e);
              covered += iv.e - iv.s;
            }
          if (hi > lo && covered == hi - lo) {  // contiguous: widen to whole rows
            const u64 r0 = (lo - w0.off) / rb, r1 = ceil_div(hi - w0.off, rb);
            X.row0 = r0;
            X.rows = r1 - r0;
          }
        }
        auto it = unit_of.find(tr.producer);
        X.unit = (it == unit_of.end() || it->second > rb) ? rb : it->second;
        const u64 U = ceil_div(rb, X.unit), q = ceil_div(U, n_chunks) * X.unit;
        for (u64 c = 0; c < n_chunks; ++c) {
          const u64 a = c * q, b = std::min((c + 1) * q, rb);
          if (a < b) X.ch.push_back({a, b});
        }
      } else {
        X.count = false;
        X.rows = 1;
        X.row_bytes = X.unit = std::max<u64>(len, 1);
        X.ch.push_back({0, X.row_bytes});
      }
    }
  }

  // ---- workspace layout per device
  const u64 AL = 256;
  p->layout.resize(n);
  p->needs_bind.assign(g->buffers.size(), std::vector<uint8_t>(n, 0));
  const uint32_t EXT = KD_BUF_WEIGHT | KD_BUF_INPUT | KD_BUF_OUTPUT | KD_BUF_PERSISTENT;
  for (uint32_t d = 0; d < n; ++d) {
    auto& L = p->layout[d];
    u64 off = 0;
    L.ctrl_off = 0;
    L.ctrl_bytes = align_up(64 + 4ull * n, AL);
    off = L.ctrl_bytes;
    // flags: per incoming transfer one u64 per chunk + the residency counter;
    // log: kLogWords (4) u64 per chunk
    L.flags_off = off;
    u64 nflags = 0, nlog = 0;
    for (uint32_t ti = 0; ti < p->transfers.size(); ++ti)
      if (p->transfers[ti].dst_dev == d) {
        const u64 nch = p->xchunks[ti].ch.size();
        L.landing[ti] = {0, L.flags_off + 8 * nflags};
        nflags += nch + 1;
        L.xlog[ti] = 32 * nlog;  // relative to log_off (fixed below)
        nlog += nch;
      }
    L.flags_bytes = align_up(std::max<u64>(8 * nflags, 8), AL);
    off += L.flags_bytes;
    L.log_off = off;
    L.log_bytes = align_up(std::max<u64>(32 * nlog, 32), AL);
    for (auto& kv : L.xlog) kv.second += L.log_off;
    off += L.log_bytes;
    // scratch = max over kernels placed here
    u64 scr = 0;
    for (uint32_t k = 0; k < K; ++k)
      if ((uint32_t)assign[k] == d) {
        u64 b = 0;
        kd_status s = op_scratch_bytes(g->kernels[k].op, g->kernels[k].attrs, &b);
        if (s) {
          delete p;
          return s;
        }
        scr = std::max(scr, b);
      }
    L.scratch_off = off;
    L.scratch_bytes = align_up(std::max<u64>(scr, 4), AL);
    off += L.scratch_bytes;
    // local instances of internal buffers touched here; binding needs of external ones
    std::set<uint32_t> touched;
    for (uint32_t k = 0; k < K; ++k)
      if ((uint32_t)assign[k] == d) {
        for (const auto& s : g->kernels[k].reads) touched.insert(s.buf);
        for (const auto& s : g->kernels[k].writes) touched.insert(s.buf);
      }
    for (uint32_t b : touched) {
      const auto& B = g->buffers[b];
      if (B.flags & EXT) {
        p->needs_bind[b][d] = 1;
        continue;
      }
      uint32_t inst = (B.flags & KD_BUF_PER_MICROBATCH) ? N : 1;
      for (uint32_t i = 0; i < inst; ++i) {
        L.act[{b, i}] = off;
        off = align_up(off + B.bytes, AL);
      }
    }
    // landing: a transfer lands in the destination's own instance of the
    // producer's output buffer, at the producer's offset — so several
    // producers (on several devices) can fill disjoint row spans of one
    // buffer that a consumer reads as a whole (the bipartite gather of a:g
    // layouts); external buffers get a private landing slot
    for (auto& kv : L.landing) {
      const kd_transfer& tr = p->transfers[kv.first];
      const Kernel& P = g->kernels[tr.producer];
      u64 len = P.writes.empty() ? 0 : P.writes[0].len;
      if (!P.writes.empty() && !(g->buffers[P.writes[0].buf].flags & EXT)) {
        const uint32_t b = P.writes[0].buf;
        const uint32_t inst = (g->buffers[b].flags & KD_BUF_PER_MICROBATCH) ? tr.micro : 0;
        auto it = L.act.find({b, inst});
        if (it != L.act.end()) {
          kv.second.first = it->second + P.writes[0].off;
          continue;
        }
      }
      kv.second.first = off;
      off = align_up(off + std::max<u64>(len, 1), AL);
    }
    L.total = align_up(off, AL);
  }
  *out = p;
  return KD_OK;
}

void kd_plan_destroy(kd_plan* p) { delete p; }

kd_status kd_plan_schedule(const kd_plan* p, kd_sched_entry* out, uint32_t cap, uint32_t* n) {
  if (!p || !n) return fail(KD_ERR_INVALID_ARG, "kd_plan_schedule: NULL argument");
  uint32_t need = (uint32_t)p->sched.size();
  if (cap < need || (need && !out)) {
    *n = need;
    return fail(KD_ERR_RANGE, "kd_plan_schedule: capacity too small");
  }
  std::copy(p->sched.begin(), p->sched.end(), out);
  *n = need;
  return KD_OK;
}

kd_status kd_plan_transfers(const kd_plan* p, kd_transfer* out, uint32_t cap, uint32_t* n) {
  if (!p || !n) return fail(KD_ERR_INVALID_ARG, "kd_plan_transfers: NULL argument");
  uint32_t need = (uint32_t)p->transfers.size();
  if (cap < need || (need && !out)) {
    *n = need;
    return fail(KD_ERR_RANGE, "kd_plan_transfers: capacity too small");
  }
  std::copy(p->transfers.begin(), p->transfers.end(), out);
  *n = need;
  return KD_OK;
}

kd_status kd_plan_chunks(const kd_plan* p, kd_chunk* out, uint32_t cap, uint32_t* n) {
  if (!p || !n) return fail(KD_ERR_INVALID_ARG, "kd_plan_chunks: NULL argument");
  uint32_t need = 0;
  for (const auto& X : p->xchunks) need += (uint32_t)X.ch.size();
  if (cap < need || (need && !out)) {
    *n = need;
    return fail(KD_ERR_RANGE, "kd_plan_chunks: capacity too small");
  }
  uint32_t i = 0;
  for (uint32_t t = 0; t < p->xchunks.size(); ++t) {
    const auto& X = p->xchunks[t];
    for (uint32_t c = 0; c < X.ch.size(); ++c) {
      kd_chunk& o = out[i++];
      o.transfer = t;
      o.chunk = c;
      o.count_mode = X.count ? 1u : 0u;
      o.pad_ = 0;
      o.row0 = X.row0;
      o.rows = X.rows;
      o.row_bytes = X.row_bytes;
      o.unit = X.unit;
      o.begin = X.ch[c].first;
      o.end = X.ch[c].second;
    }
  }
  *n = need;
  return KD_OK;
}

kd_status kd_plan_makespan(const kd_plan* p, int64_t* ps) {
  if (!p || !ps) return fail(KD_ERR_INVALID_ARG, "kd_plan_makespan: NULL argument");
  *ps = p->makespan;
  return KD_OK;
}

kd_status kd_plan_workspace_bytes(const kd_plan* p, uint32_t dev, uint64_t* bytes) {
  if (!p || !bytes || dev >= p->n_dev) return fail(KD_ERR_INVALID_ARG, "kd_plan_workspace_bytes: bad argument");
  *bytes = p->layout[dev].total;
  return KD_OK;
}

kd_status kd_plan_workspace_layout(const kd_plan* p, uint32_t dev, kd_ws_layout* out) {
  if (!p || !out || dev >= p->n_dev) return fail(KD_ERR_INVALID_ARG, "kd_plan_workspace_layout: bad argument");
  const auto& L = p->layout[dev];
  out->ctrl_off = L.ctrl_off;
  out->ctrl_bytes = L.ctrl_bytes;
  out->flags_off = L.flags_off;
  out->flags_bytes = L.flags_bytes;
  out->log_off = L.log_off;
  out->log_bytes = L.log_bytes;
  out->scratch_off = L.scratch_off;
  out->scratch_bytes = L.scratch_bytes;
  out->act_off = L.scratch_off + L.scratch_bytes;
  out->total = L.total;
  return KD_OK;
}

kd_status kd_plan_needs_binding(const kd_plan* p, uint32_t buf, uint32_t dev, int32_t* needed) {
  if (!p || !needed || dev >= p->n_dev || buf >= p->needs_bind.size())
    return fail(KD_ERR_INVALID_ARG, "kd_plan_needs_binding: bad argument");
  *needed = p->needs_bind[buf][dev];
  return KD_OK;
}

}  // extern "C"
