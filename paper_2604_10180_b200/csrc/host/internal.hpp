// internal.hpp — host-side internal types of libkd (not part of the ABI).
#pragma once
#include <cstdint>
#include <cstring>
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "kd.h"

namespace kd {

// thread-local last error (kd_last_error)
void set_error(const std::string& msg);
kd_status fail(kd_status s, const std::string& msg);

using u64 = uint64_t;
using i64 = int64_t;
using u128 = unsigned __int128;

inline u64 ceil_div_u128(u128 a, u128 b) { return (u64)((a + b - 1) / b); }
inline u64 ceil_div(u64 a, u64 b) { return (a + b - 1) / b; }
constexpr u64 kPs = 1000000000000ull;

struct Span {
  uint32_t buf;
  u64 off, len;
};

struct Kernel {
  uint32_t op = 0;
  std::vector<Span> reads, writes;
  int32_t pin = -1;
  int32_t tmpl = -1;
  u64 flops = 0;
  std::vector<uint8_t> attrs;
};

struct Buffer {
  u64 bytes = 0;
  uint32_t flags = 0;
};

struct Interval {
  u64 s, e;
};
// per-buffer sorted disjoint union of spans
std::map<uint32_t, std::vector<Interval>> span_union(const std::vector<Span>& spans);
u64 union_bytes(const std::vector<Span>& spans);

}  // namespace kd

struct kd_graph {
  std::vector<kd::Buffer> buffers;
  std::vector<kd::Kernel> kernels;
  std::vector<kd_edge> edges;
  bool finalized = false;
};

namespace kd {
// cost (A10) of kernel k on device d in ps
i64 kernel_time(const kd_graph& g, const kd_machine& m, uint32_t k, uint32_t d);
bool machine_valid(const kd_machine* m);
// d_ij aggregated per (src,dst) pair
std::vector<std::pair<std::pair<uint32_t, uint32_t>, u64>> edge_pairs(const kd_graph& g);
i64 edge_cost(const kd_machine& m, u64 bytes, uint32_t u, uint32_t v);
}  // namespace kd

struct kd_plan {
  const kd_graph* g = nullptr;  // borrowed; graph must outlive the plan
  uint32_t n_dev = 0, n_micro = 1;
  std::vector<int32_t> assign;
  std::vector<kd_sched_entry> sched;   // global order
  std::vector<kd_transfer> transfers;  // sorted by (micro, producer, dst_dev)
  kd::i64 makespan = 0;
  // workspace layout per device
  struct Layout {
    kd::u64 ctrl_off = 0, ctrl_bytes = 0;      // epoch + barrier words
    kd::u64 flags_off = 0, flags_bytes = 0;    // one u32 per incoming transfer (padded)
    kd::u64 scratch_off = 0, scratch_bytes = 0;
    kd::u64 total = 0;
    // (buf, micro) -> offset of the local activation instance
    std::map<std::pair<uint32_t, uint32_t>, kd::u64> act;
    // transfer index -> (landing offset, flag offset)
    std::map<uint32_t, std::pair<kd::u64, kd::u64>> landing;
  };
  std::vector<Layout> layout;
  // external binding need [buf][dev]
  std::vector<std::vector<uint8_t>> needs_bind;
};
