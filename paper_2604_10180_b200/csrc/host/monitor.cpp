// monitor.cpp — the online monitor's queueing-aware policy switch (PAPER.md
// §3.4 "Online Monitor"; defaults W = 300 ms, β = 1.5).
//
// Requests are attributed to the fixed window ⌊t_end / W⌋ in which they
// finish. At every window boundary the monitor compares the mean request
// latency L̄_req with the mean pure execution latency L̄_exec (computation +
// communication, queueing excluded): ratio > β → the throughput-oriented
// policy (queueing dominates), otherwise the latency-oriented one.
// Integer nanoseconds and a rational β make every decision exact
// (Σreq·β_den > β_num·Σexec ⇔ L̄_req / L̄_exec > β; the counts cancel). An
// empty window keeps the current policy (the paper is silent; R21).
#include "internal.hpp"

struct kd_monitor {
  uint64_t window_ns = 0;
  uint32_t beta_num = 0, beta_den = 1;
  uint32_t policy = KD_OBJ_LATENCY;
  uint32_t switches = 0;
  uint64_t next_window = 0;  // index of the first window not yet evaluated
  // per pending window: Σ req, Σ exec, count
  std::map<uint64_t, std::pair<kd::u128, kd::u128>> acc;
  std::map<uint64_t, uint64_t> cnt;
};

using namespace kd;

extern "C" {

kd_status kd_monitor_create(uint64_t window_ns, uint32_t beta_num, uint32_t beta_den, uint32_t initial_policy,
                            kd_monitor** out) {
  if (!out || window_ns == 0 || beta_den == 0) return fail(KD_ERR_INVALID_ARG, "kd_monitor_create: bad argument");
  if (initial_policy != KD_OBJ_LATENCY && initial_policy != KD_OBJ_THROUGHPUT)
    return fail(KD_ERR_INVALID_ARG, "kd_monitor_create: policy must be KD_OBJ_LATENCY or KD_OBJ_THROUGHPUT");
  auto* m = new kd_monitor();
  m->window_ns = window_ns;
  m->beta_num = beta_num;
  m->beta_den = beta_den;
  m->policy = initial_policy;
  *out = m;
  return KD_OK;
}

kd_status kd_monitor_destroy(kd_monitor* m) {
  delete m;
  return KD_OK;
}

kd_status kd_monitor_record(kd_monitor* m, uint64_t t_end_ns, uint64_t req_latency_ns, uint64_t exec_latency_ns) {
  if (!m) return fail(KD_ERR_INVALID_ARG, "kd_monitor_record: NULL monitor");
  const uint64_t w = t_end_ns / m->window_ns;
  if (w < m->next_window) return fail(KD_ERR_STATE, "kd_monitor_record: request finishes in an already evaluated window");
  auto& a = m->acc[w];
  a.first += req_latency_ns;
  a.second += exec_latency_ns;
  ++m->cnt[w];
  return KD_OK;
}

kd_status kd_monitor_poll(kd_monitor* m, uint64_t now_ns, uint32_t* policy, uint32_t* switches) {
  if (!m || !policy) return fail(KD_ERR_INVALID_ARG, "kd_monitor_poll: bad argument");
  const uint64_t done = now_ns / m->window_ns;  // windows [next_window, done) have ended
  for (uint64_t w = m->next_window; w < done; ++w) {
    auto it = m->acc.find(w);
    if (it == m->acc.end()) continue;  // empty window: keep the policy
    const u128 lhs = it->second.first * (u128)m->beta_den, rhs = it->second.second * (u128)m->beta_num;
    const uint32_t p = lhs > rhs ? (uint32_t)KD_OBJ_THROUGHPUT : (uint32_t)KD_OBJ_LATENCY;
    if (p != m->policy) {
      m->policy = p;
      ++m->switches;
    }
    m->acc.erase(it);
    m->cnt.erase(w);
  }
  if (done > m->next_window) m->next_window = done;
  *policy = m->policy;
  if (switches) *switches = m->switches;
  return KD_OK;
}

}  // extern "C"
