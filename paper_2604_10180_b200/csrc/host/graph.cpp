// graph.cpp — kernel DAG from declared read/write sets (§3.1,
// "Data dependency analysis"; declared sets = library-kernel case
// P:241-242). Readings R1-R5.
#include <algorithm>
#include <cstdio>

#include "internal.hpp"

namespace kd {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
kd_status fail(kd_status s, const std::string& msg) {
  set_error(msg);
  return s;
}

std::map<uint32_t, std::vector<Interval>> span_union(const std::vector<Span>& spans) {
  std::map<uint32_t, std::vector<Interval>> per;
  for (const auto& s : spans) per[s.buf].push_back({s.off, s.off + s.len});
  for (auto& kv : per) {
    auto& v = kv.second;
    std::sort(v.begin(), v.end(), [](const Interval& a, const Interval& b) {
      return a.s < b.s || (a.s == b.s && a.e < b.e);
    });
    std::vector<Interval> m;
    for (const auto& iv : v) {
      if (!m.empty() && iv.s <= m.back().e)
        m.back().e = std::max(m.back().e, iv.e);
      else
        m.push_back(iv);
    }
    v.swap(m);
  }
  return per;
}

u64 union_bytes(const std::vector<Span>& spans) {
  u64 b = 0;
  for (const auto& kv : span_union(spans))
    for (const auto& iv : kv.second) b += iv.e - iv.s;
  return b;
}

// Last-writer registry at byte-span granularity: per buffer a map
// start -> (end, writer) of disjoint intervals (R1).
class Registry {
 public:
  struct Piece {
    u64 e;
    uint32_t w;
  };
  // pieces of [s,e) that have a writer, in address order
  void lookup(uint32_t buf, u64 s, u64 e, std::vector<std::tuple<u64, u64, uint32_t>>& out) const {
    auto it = reg_.find(buf);
    if (it == reg_.end()) return;
    const auto& m = it->second;
    auto p = m.upper_bound(s);
    if (p != m.begin()) --p;
    for (; p != m.end() && p->first < e; ++p) {
      u64 lo = std::max(p->first, s), hi = std::min(p->second.e, e);
      if (lo < hi) out.emplace_back(lo, hi, p->second.w);
    }
  }
  void write(uint32_t buf, u64 s, u64 e, uint32_t w) {
    auto& m = reg_[buf];
    auto p = m.upper_bound(s);
    if (p != m.begin()) --p;
    std::vector<std::pair<u64, Piece>> keep;
    while (p != m.end() && p->first < e) {
      u64 a = p->first, b = p->second.e;
      uint32_t ow = p->second.w;
      if (b <= s) {
        ++p;
        continue;
      }
      p = m.erase(p);
      if (a < s) keep.push_back({a, {s, ow}});
      if (b > e) keep.push_back({e, {b, ow}});
    }
    for (auto& kv : keep) m[kv.first] = kv.second;
    m[s] = {e, w};
  }

 private:
  std::map<uint32_t, std::map<u64, Piece>> reg_;
};

}  // namespace kd

using namespace kd;

extern "C" {

const char* kd_status_str(kd_status s) {
  switch (s) {
    case KD_OK: return "KD_OK";
    case KD_ERR_INVALID_ARG: return "KD_ERR_INVALID_ARG";
    case KD_ERR_RANGE: return "KD_ERR_RANGE";
    case KD_ERR_STATE: return "KD_ERR_STATE";
    case KD_ERR_PIN_CONFLICT: return "KD_ERR_PIN_CONFLICT";
    case KD_ERR_INFEASIBLE: return "KD_ERR_INFEASIBLE";
    case KD_ERR_UNSUPPORTED: return "KD_ERR_UNSUPPORTED";
    case KD_ERR_CUDA: return "KD_ERR_CUDA";
    case KD_ERR_NCCL: return "KD_ERR_NCCL";
    case KD_ERR_TIMEOUT: return "KD_ERR_TIMEOUT";
    case KD_ERR_OOM: return "KD_ERR_OOM";
  }
  return "KD_ERR_?";
}

const char* kd_last_error(void) { return kd::g_last_error.c_str(); }
uint32_t kd_version(void) { return (0u << 16) | 1u; }

kd_status kd_graph_create(kd_graph** out) {
  if (!out) return fail(KD_ERR_INVALID_ARG, "kd_graph_create: out is NULL");
  *out = new kd_graph();
  return KD_OK;
}

void kd_graph_destroy(kd_graph* g) { delete g; }

kd_status kd_graph_add_buffer(kd_graph* g, uint64_t bytes, uint32_t flags, uint32_t* id) {
  if (!g || !id) return fail(KD_ERR_INVALID_ARG, "kd_graph_add_buffer: NULL argument");
  if (g->finalized) return fail(KD_ERR_STATE, "kd_graph_add_buffer: graph already finalized");
  if (bytes == 0) return fail(KD_ERR_INVALID_ARG, "kd_graph_add_buffer: zero-size buffer");
  if (flags & ~0x3Fu) return fail(KD_ERR_INVALID_ARG, "kd_graph_add_buffer: unknown flag bits");
  if ((flags & KD_BUF_REPLICATED) && !(flags & KD_BUF_PERSISTENT))
    return fail(KD_ERR_INVALID_ARG, "kd_graph_add_buffer: REPLICATED applies to PERSISTENT buffers");
  g->buffers.push_back({bytes, flags});
  *id = (uint32_t)g->buffers.size() - 1;
  return KD_OK;
}

static kd_status copy_spans(const kd_graph* g, const kd_span* in, uint32_t n, std::vector<Span>& out,
                            const char* what) {
  if (n && !in) return fail(KD_ERR_INVALID_ARG, std::string("kd_graph_add_kernel: NULL ") + what);
  for (uint32_t i = 0; i < n; ++i) {
    const kd_span& s = in[i];
    if (s.buf >= g->buffers.size())
      return fail(KD_ERR_INVALID_ARG, std::string("kd_graph_add_kernel: unknown buffer in ") + what);
    if (s.len == 0) return fail(KD_ERR_INVALID_ARG, std::string("kd_graph_add_kernel: zero-length span in ") + what);
    if (s.offset > g->buffers[s.buf].bytes || s.len > g->buffers[s.buf].bytes - s.offset)
      return fail(KD_ERR_RANGE, std::string("kd_graph_add_kernel: span outside buffer in ") + what);
    out.push_back({s.buf, s.offset, s.len});
  }
  return KD_OK;
}

kd_status kd_graph_add_kernel(kd_graph* g, const kd_kernel_desc* d, uint32_t* id) {
  if (!g || !d || !id) return fail(KD_ERR_INVALID_ARG, "kd_graph_add_kernel: NULL argument");
  if (g->finalized) return fail(KD_ERR_STATE, "kd_graph_add_kernel: graph already finalized");
  if (d->op > KD_OP_PREFILL_ATTENTION) return fail(KD_ERR_INVALID_ARG, "kd_graph_add_kernel: unknown op");
  Kernel k;
  k.op = d->op;
  k.pin = d->pin_device;
  k.tmpl = d->template_id;
  k.flops = d->flops;
  kd_status s = copy_spans(g, d->reads, d->n_reads, k.reads, "reads");
  if (s) return s;
  s = copy_spans(g, d->writes, d->n_writes, k.writes, "writes");
  if (s) return s;
  for (const auto& w : k.writes)
    if (g->buffers[w.buf].flags & KD_BUF_WEIGHT)
      return fail(KD_ERR_INVALID_ARG, "kd_graph_add_kernel: kernel writes a WEIGHT buffer");
  if (d->attrs_size) {
    if (!d->attrs) return fail(KD_ERR_INVALID_ARG, "kd_graph_add_kernel: attrs_size without attrs");
    const uint8_t* a = (const uint8_t*)d->attrs;
    k.attrs.assign(a, a + d->attrs_size);
  }
  g->kernels.push_back(std::move(k));
  *id = (uint32_t)g->kernels.size() - 1;
  return KD_OK;
}

kd_status kd_graph_finalize(kd_graph* g) {
  if (!g) return fail(KD_ERR_INVALID_ARG, "kd_graph_finalize: NULL graph");
  if (g->finalized) return fail(KD_ERR_STATE, "kd_graph_finalize: already finalized");
  Registry reg;
  std::vector<kd_edge> edges;
  std::vector<std::tuple<u64, u64, uint32_t>> hits;
  for (uint32_t k = 0; k < g->kernels.size(); ++k) {
    const Kernel& K = g->kernels[k];
    // 1) resolve every read before applying k's own writes (R2)
    for (const auto& kv : span_union(K.reads)) {
      uint32_t buf = kv.first;
      for (const auto& iv : kv.second) {
        hits.clear();
        reg.lookup(buf, iv.s, iv.e, hits);
        // merge address-adjacent pieces with the same writer -> maximal spans (R3)
        bool open = false;
        u64 rs = 0, re = 0;
        uint32_t rw = 0;
        for (const auto& h : hits) {
          u64 lo = std::get<0>(h), hi = std::get<1>(h);
          uint32_t w = std::get<2>(h);
          if (w == k) continue;  // cannot happen (writes applied later); kept for clarity
          if (open && rw == w && re == lo) {
            re = hi;
          } else {
            if (open) edges.push_back({rw, k, buf, 0, rs, re - rs});
            open = true;
            rs = lo;
            re = hi;
            rw = w;
          }
        }
        if (open) edges.push_back({rw, k, buf, 0, rs, re - rs});
      }
    }
    // 2) k becomes the last writer of its write spans
    for (const auto& kv : span_union(K.writes))
      for (const auto& iv : kv.second) reg.write(kv.first, iv.s, iv.e, k);
  }
  std::sort(edges.begin(), edges.end(), [](const kd_edge& a, const kd_edge& b) {
    if (a.dst != b.dst) return a.dst < b.dst;
    if (a.src != b.src) return a.src < b.src;
    if (a.buf != b.buf) return a.buf < b.buf;
    return a.offset < b.offset;
  });
  g->edges.swap(edges);
  g->finalized = true;
  return KD_OK;
}

kd_status kd_graph_num_kernels(const kd_graph* g, uint32_t* n) {
  if (!g || !n) return fail(KD_ERR_INVALID_ARG, "kd_graph_num_kernels: NULL argument");
  *n = (uint32_t)g->kernels.size();
  return KD_OK;
}

kd_status kd_graph_num_buffers(const kd_graph* g, uint32_t* n) {
  if (!g || !n) return fail(KD_ERR_INVALID_ARG, "kd_graph_num_buffers: NULL argument");
  *n = (uint32_t)g->buffers.size();
  return KD_OK;
}

kd_status kd_graph_edges(const kd_graph* g, kd_edge* out, uint32_t cap, uint32_t* n) {
  if (!g || !n) return fail(KD_ERR_INVALID_ARG, "kd_graph_edges: NULL argument");
  if (!g->finalized) return fail(KD_ERR_STATE, "kd_graph_edges: graph not finalized");
  uint32_t need = (uint32_t)g->edges.size();
  if (cap < need || (need && !out)) {
    *n = need;
    return fail(KD_ERR_RANGE, "kd_graph_edges: capacity too small");
  }
  std::copy(g->edges.begin(), g->edges.end(), out);
  *n = need;
  return KD_OK;
}

}  // extern "C"
