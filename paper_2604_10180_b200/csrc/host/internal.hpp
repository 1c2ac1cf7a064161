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
constexpr uint32_t kMaxPlanChunks = 8;  // chunks per transfer (= kMaxChunks of the device code)

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
// a13 op knowledge (plan.cpp): the primary output of a COUNT-release producer
// as rows × row_bytes (false: CTA release — irregular or dynamic outputs)
bool op_count_geometry(const Kernel& k, u64* rows, u64* row_bytes);
// chunk unit (bytes along a row) the consumer k needs on read span ri when it
// acquires that input chunk by chunk inside the kernel; 0 = not chunk-aware
// (the runtime then waits for the whole transfer before launching it)
u64 op_consumer_unit(const Kernel& k, uint32_t ri, u64 row_bytes);
// delta replication (KD_BUF_REPLICATED): bytes kernel k actually
// writes into write span wi of a replicated buffer per step (RoPE/append: the
// appended K or V slot of every row and kv head), else the span length
u64 op_delta_bytes(const Kernel& k, uint32_t wi);
// producers whose peer stores can be filtered to the rows a device reads
// (the GEMM epilogues): a scatter transfer then carries only those rows
bool op_row_filter(const Kernel& k);
// bytes an edge record charges the cost model and the transfer: the delta for
// a replicated buffer (once per (src, buf): records after the first cost 0),
// else the span length
bool buf_replicated(const kd_graph& g, uint32_t buf);
u64 delta_of(const kd_graph& g, uint32_t src, uint32_t buf);
}  // namespace kd

struct kd_plan {
  const kd_graph* g = nullptr;  // borrowed; graph must outlive the plan
  uint32_t n_dev = 0, n_micro = 1;
  std::vector<int32_t> assign;
  std::vector<kd_sched_entry> sched;   // global order
  std::vector<kd_transfer> transfers;  // sorted by (micro, producer, dst_dev)
  // chunk table per transfer (R10): the producer's primary output as
  // [rows][row_bytes], each row cut into column chunks [begin, end) along the
  // chunk-aware consumers' streamable axis (unit = lcm of their units)
  struct XChunks {
    bool count = false;       // COUNT release (bytes per chunk) vs CTA release (1 chunk)
    kd::u64 row0 = 0;         // first row the transfer carries (row-filtered scatter, R24)
    kd::u64 rows = 1, row_bytes = 0, unit = 0;
    std::vector<std::pair<kd::u64, kd::u64>> ch;
  };
  std::vector<XChunks> xchunks;
  uint32_t n_chunks = 1;
  kd::i64 makespan = 0;
  // workspace layout per device
  struct Layout {
    kd::u64 ctrl_off = 0, ctrl_bytes = 0;      // epoch + error word + barrier words
    kd::u64 flags_off = 0, flags_bytes = 0;    // per incoming transfer: u64 flag per chunk + u64 residency counter
    kd::u64 log_off = 0, log_bytes = 0;        // per incoming transfer: kLogWords u64 per chunk (KD_MODE_LOG)
    kd::u64 scratch_off = 0, scratch_bytes = 0;
    kd::u64 total = 0;
    // (buf, micro) -> offset of the local activation instance
    std::map<std::pair<uint32_t, uint32_t>, kd::u64> act;
    // transfer index -> (landing offset, flag offset); the residency counter
    // follows the chunk flags; log records at xlog[t]
    std::map<uint32_t, std::pair<kd::u64, kd::u64>> landing;
    std::map<uint32_t, kd::u64> xlog;
  };
  std::vector<Layout> layout;
  // external binding need [buf][dev]
  std::vector<std::vector<uint8_t>> needs_bind;
};
