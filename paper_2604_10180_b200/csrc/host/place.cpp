// place.cpp — roofline cost model and placement search (§3.2,
// P:304-363, equations E1-E7; MILP replaced by exact branch and bound over
// template classes, A11/A14/A15; integer picoseconds, R7; N micro-batches, R8).
#include <algorithm>
#include <functional>
#include <limits>
#include <set>
#include <tuple>

#include "internal.hpp"

namespace kd {

bool machine_valid(const kd_machine* m) {
  if (!m || m->n_dev == 0 || !m->hbm_Bps || !m->tc_flops || !m->link_Bps || !m->link_lat_ps) return false;
  for (uint32_t d = 0; d < m->n_dev; ++d) {
    if (m->hbm_Bps[d] == 0 || m->tc_flops[d] == 0) return false;
    for (uint32_t g = 0; g < m->n_dev; ++g)
      if (g != d && m->link_Bps[d * m->n_dev + g] == 0) return false;
  }
  return true;
}

// t_{k,g} = max(⌈bytes·10¹²/HBM⌉, ⌈flops·10¹²/TC⌉) + launch (A10)
i64 kernel_time(const kd_graph& g, const kd_machine& m, uint32_t k, uint32_t d) {
  const Kernel& K = g.kernels[k];
  u64 bytes = union_bytes(K.reads) + union_bytes(K.writes);
  u64 tb = ceil_div_u128((u128)bytes * kPs, m.hbm_Bps[d]);
  u64 tf = ceil_div_u128((u128)K.flops * kPs, m.tc_flops[d]);
  return (i64)(std::max(tb, tf) + m.launch_ps);
}

// c^{u,g}_{ij} = ℓ_{u,g} + ⌈d_ij·10¹²/bw_{u,g}⌉ (E4)
i64 edge_cost(const kd_machine& m, u64 bytes, uint32_t u, uint32_t v) {
  uint32_t n = m.n_dev;
  return (i64)(m.link_lat_ps[u * n + v] + ceil_div_u128((u128)bytes * kPs, m.link_Bps[u * n + v]));
}

// d_ij = Σ record lengths per (src, dst) (Table 2, R3); records on a
// REPLICATED buffer charge the producer's delta once per (src, dst, buffer)
std::vector<std::pair<std::pair<uint32_t, uint32_t>, u64>> edge_pairs(const kd_graph& g) {
  std::map<std::pair<uint32_t, uint32_t>, u64> acc;
  std::set<std::tuple<uint32_t, uint32_t, uint32_t>> seen;
  for (const auto& e : g.edges) {
    if (buf_replicated(g, e.buf)) {
      if (seen.insert({e.src, e.dst, e.buf}).second) acc[{e.src, e.dst}] += delta_of(g, e.src, e.buf);
      else acc[{e.src, e.dst}] += 0;
      continue;
    }
    acc[{e.src, e.dst}] += e.len;
  }
  return {acc.begin(), acc.end()};
}

static i64 combine(const std::vector<i64>& T, const std::vector<i64>& M, uint32_t N, uint32_t obj) {
  // E5/E6 (throughput) or E7 (latency); both per step = N x per micro-batch (R8)
  i64 r = 0;
  if (obj == KD_OBJ_LATENCY) {
    for (size_t d = 0; d < T.size(); ++d) r += T[d] + M[d];
    return r * (i64)N;
  }
  for (size_t d = 0; d < T.size(); ++d) r = std::max(r, std::max(T[d], M[d]));
  return r * (i64)N;
}

static uint32_t resolve_obj(uint32_t obj, uint32_t N) {
  if (obj == KD_OBJ_AUTO) return N == 1 ? KD_OBJ_LATENCY : KD_OBJ_THROUGHPUT;
  return obj;
}

}  // namespace kd

using namespace kd;

extern "C" {

kd_status kd_cost(const kd_graph* g, const kd_machine* m, int64_t* t_ps) {
  if (!g || !t_ps) return fail(KD_ERR_INVALID_ARG, "kd_cost: NULL argument");
  if (!machine_valid(m)) return fail(KD_ERR_INVALID_ARG, "kd_cost: invalid machine");
  for (uint32_t k = 0; k < g->kernels.size(); ++k)
    for (uint32_t d = 0; d < m->n_dev; ++d) t_ps[k * m->n_dev + d] = kernel_time(*g, *m, k, d);
  return KD_OK;
}

kd_status kd_objective(const kd_graph* g, const kd_machine* m, const int32_t* assign, uint32_t n_micro,
                       uint32_t objective, int64_t* obj_ps, int64_t* T_ps, int64_t* M_ps) {
  if (!g || !assign || !obj_ps) return fail(KD_ERR_INVALID_ARG, "kd_objective: NULL argument");
  if (!g->finalized) return fail(KD_ERR_STATE, "kd_objective: graph not finalized");
  if (!machine_valid(m) || n_micro == 0 || objective > KD_OBJ_LATENCY)
    return fail(KD_ERR_INVALID_ARG, "kd_objective: invalid machine/n_micro/objective");
  uint32_t n = m->n_dev;
  std::vector<i64> T(n, 0), M(n, 0);
  for (uint32_t k = 0; k < g->kernels.size(); ++k) {
    if (assign[k] < 0 || (uint32_t)assign[k] >= n) return fail(KD_ERR_INVALID_ARG, "kd_objective: bad device");
    T[assign[k]] += kernel_time(*g, *m, k, assign[k]);
  }
  for (const auto& e : edge_pairs(*g)) {
    uint32_t u = assign[e.first.first], v = assign[e.first.second];
    if (u != v) M[v] += edge_cost(*m, e.second, u, v);  // y^{u,v}_{ij} = 1
  }
  *obj_ps = combine(T, M, n_micro, resolve_obj(objective, n_micro));
  for (uint32_t d = 0; d < n; ++d) {
    if (T_ps) T_ps[d] = T[d] * (i64)n_micro;
    if (M_ps) M_ps[d] = M[d] * (i64)n_micro;
  }
  return KD_OK;
}

kd_status kd_place(const kd_graph* g, const kd_machine* m, const kd_place_opts* opts, int32_t* assign,
                   int64_t* objective_ps, uint64_t* nodes_visited) {
  if (!g || !opts || !assign || !objective_ps) return fail(KD_ERR_INVALID_ARG, "kd_place: NULL argument");
  if (!g->finalized) return fail(KD_ERR_STATE, "kd_place: graph not finalized");
  if (!machine_valid(m) || opts->n_micro == 0 || opts->objective > KD_OBJ_LATENCY)
    return fail(KD_ERR_INVALID_ARG, "kd_place: invalid machine/n_micro/objective");
  const uint32_t n = m->n_dev, K = (uint32_t)g->kernels.size();
  const uint32_t N = opts->n_micro, obj = resolve_obj(opts->objective, N);

  // template classes in first-occurrence order; pins fix a class (A4, A15)
  std::vector<uint32_t> cls_of(K);
  std::map<std::pair<int, int64_t>, uint32_t> key2cls;
  for (uint32_t k = 0; k < K; ++k) {
    int tid = g->kernels[k].tmpl;
    auto key = tid >= 0 ? std::make_pair(0, (int64_t)tid) : std::make_pair(1, (int64_t)k);
    auto it = key2cls.find(key);
    if (it == key2cls.end()) it = key2cls.emplace(key, (uint32_t)key2cls.size()).first;
    cls_of[k] = it->second;
  }
  const uint32_t C = (uint32_t)key2cls.size();
  std::vector<int32_t> fixed(C, -1);
  for (uint32_t k = 0; k < K; ++k) {
    int32_t p = g->kernels[k].pin;
    if (p < 0) continue;
    if ((uint32_t)p >= n) return fail(KD_ERR_INVALID_ARG, "kd_place: pin outside the machine");
    int32_t& f = fixed[cls_of[k]];
    if (f >= 0 && f != p) return fail(KD_ERR_PIN_CONFLICT, "kd_place: conflicting pins in one template class");
    f = p;
  }
  std::vector<uint32_t> free_cls;
  std::vector<int32_t> pos_of(C, -1);
  for (uint32_t c = 0; c < C; ++c)
    if (fixed[c] < 0) {
      pos_of[c] = (int32_t)free_cls.size();
      free_cls.push_back(c);
    }
  const uint32_t P = (uint32_t)free_cls.size();

  // per-kernel, per-device times; edges bucketed by the position completing them
  std::vector<i64> t((size_t)K * n);
  for (uint32_t k = 0; k < K; ++k)
    for (uint32_t d = 0; d < n; ++d) t[(size_t)k * n + d] = kernel_time(*g, *m, k, d);
  std::vector<std::vector<uint32_t>> kern_at(P);
  std::vector<i64> T0(n, 0), M0(n, 0);
  std::vector<int32_t> dev_of_cls(C, -1);
  for (uint32_t c = 0; c < C; ++c) dev_of_cls[c] = fixed[c];
  for (uint32_t k = 0; k < K; ++k) {
    int32_t p = pos_of[cls_of[k]];
    if (p >= 0)
      kern_at[p].push_back(k);
    else
      T0[fixed[cls_of[k]]] += t[(size_t)k * n + fixed[cls_of[k]]];
  }
  struct EP {
    uint32_t i, j;
    u64 d;
  };
  std::vector<std::vector<EP>> edge_at(P);
  for (const auto& e : edge_pairs(*g)) {
    uint32_t i = e.first.first, j = e.first.second;
    int32_t p = std::max(pos_of[cls_of[i]], pos_of[cls_of[j]]);
    if (p >= 0)
      edge_at[p].push_back({i, j, e.second});
    else {
      uint32_t u = fixed[cls_of[i]], v = fixed[cls_of[j]];
      if (u != v) M0[v] += edge_cost(*m, e.second, u, v);
    }
  }

  // symmetry: all devices interchangeable (equal HBM/TC, uniform links) → devices
  // that are neither pinned nor used yet are equivalent; try only the lowest one
  bool homog = true;
  for (uint32_t d = 0; d < n && homog; ++d) {
    if (m->hbm_Bps[d] != m->hbm_Bps[0] || m->tc_flops[d] != m->tc_flops[0]) homog = false;
    for (uint32_t v = 0; v < n && homog; ++v)
      if (v != d && (m->link_Bps[d * n + v] != m->link_Bps[n > 1 ? 1 : 0] ||
                     m->link_lat_ps[d * n + v] != m->link_lat_ps[n > 1 ? 1 : 0]))
        homog = false;
  }
  std::vector<uint8_t> pinned(n, 0);
  for (uint32_t c = 0; c < C; ++c)
    if (fixed[c] >= 0) pinned[fixed[c]] = 1;

  std::vector<i64> T = T0, M = M0;
  std::vector<int32_t> choice(P, -1), best_choice;
  std::vector<uint32_t> use_cnt(n, 0);
  i64 best = std::numeric_limits<i64>::max();
  uint64_t nodes = 0;
  bool budget_hit = false;

  // iterative DFS; devices tried in ascending order → first optimum is lexicographically smallest
  std::vector<std::vector<i64>> saveT(P + 1), saveM(P + 1);
  std::function<void(uint32_t)> dfs = [&](uint32_t p) {
    if (budget_hit) return;
    ++nodes;
    if (opts->max_nodes && nodes > opts->max_nodes) {
      budget_hit = true;
      return;
    }
    i64 lb = combine(T, M, N, obj);  // partial sums only grow: a lower bound
    if (lb >= best) return;
    if (p == P) {
      best = lb;
      best_choice = choice;
      return;
    }
    bool new_tried = false;
    for (uint32_t d = 0; d < n; ++d) {
      if (homog && !pinned[d] && use_cnt[d] == 0) {
        if (new_tried) continue;
        new_tried = true;
      }
      choice[p] = (int32_t)d;
      dev_of_cls[free_cls[p]] = (int32_t)d;
      std::vector<i64> T_save = T, M_save = M;
      for (uint32_t k : kern_at[p]) T[d] += t[(size_t)k * n + d];
      for (const auto& e : edge_at[p]) {
        uint32_t u = dev_of_cls[cls_of[e.i]], v = dev_of_cls[cls_of[e.j]];
        if (u != v) M[v] += edge_cost(*m, e.d, u, v);
      }
      use_cnt[d]++;
      dfs(p + 1);
      use_cnt[d]--;
      T.swap(T_save);
      M.swap(M_save);
      dev_of_cls[free_cls[p]] = -1;
      choice[p] = -1;
    }
  };
  dfs(0);
  if (budget_hit) return fail(KD_ERR_INFEASIBLE, "kd_place: search budget exhausted");
  if (best_choice.size() != P) return fail(KD_ERR_INFEASIBLE, "kd_place: no candidate");
  for (uint32_t c = 0; c < C; ++c) dev_of_cls[c] = fixed[c];
  for (uint32_t p = 0; p < P; ++p) dev_of_cls[free_cls[p]] = best_choice[p];
  for (uint32_t k = 0; k < K; ++k) assign[k] = dev_of_cls[cls_of[k]];
  *objective_ps = best;
  if (nodes_visited) *nodes_visited = nodes;
  return KD_OK;
}

kd_status kd_place_roles(const kd_graph* g, const kd_machine* m, uint32_t rows, uint32_t max_gpus, uint32_t micro_mask,
                         kd_role_layout* best, int32_t* roles, uint32_t cap, uint32_t* n_out) {
  if (!g || !best || !roles || !n_out) return fail(KD_ERR_INVALID_ARG, "kd_place_roles: NULL argument");
  if (!g->finalized) return fail(KD_ERR_STATE, "kd_place_roles: graph not finalized");
  if (!machine_valid(m) || rows == 0 || max_gpus == 0 || (micro_mask & 7u) == 0)
    return fail(KD_ERR_INVALID_ARG, "kd_place_roles: invalid machine/rows/max_gpus/micro_mask");
  const uint32_t K = (uint32_t)g->kernels.size();
  // classes in first-use order; pins fix the role (0 memory, 1 GEMM)
  std::vector<uint32_t> cls_of(K);
  std::map<std::pair<int, int64_t>, uint32_t> key2cls;
  for (uint32_t k = 0; k < K; ++k) {
    int tid = g->kernels[k].tmpl;
    auto key = tid >= 0 ? std::make_pair(0, (int64_t)tid) : std::make_pair(1, (int64_t)k);
    auto it = key2cls.find(key);
    if (it == key2cls.end()) it = key2cls.emplace(key, (uint32_t)key2cls.size()).first;
    cls_of[k] = it->second;
  }
  const uint32_t C = (uint32_t)key2cls.size();
  std::vector<int32_t> fixed(C, -1);
  for (uint32_t k = 0; k < K; ++k) {
    const int32_t p = g->kernels[k].pin;
    if (p < 0) continue;
    if (p > 1) return fail(KD_ERR_INVALID_ARG, "kd_place_roles: a pin must name a role (0 memory, 1 GEMM)");
    if (fixed[cls_of[k]] >= 0 && fixed[cls_of[k]] != p) return fail(KD_ERR_PIN_CONFLICT, "kd_place_roles: conflicting pins");
    fixed[cls_of[k]] = p;
  }
  std::vector<uint32_t> free_cls;
  for (uint32_t c = 0; c < C; ++c)
    if (fixed[c] < 0) free_cls.push_back(c);
  if (free_cls.size() > 20) return fail(KD_ERR_UNSUPPORTED, "kd_place_roles: more than 20 free template classes");
  const u64 hbm = m->hbm_Bps[0], tc = m->tc_flops[0];
  const bool has_link = m->n_dev > 1;
  const u64 bw = has_link ? m->link_Bps[1] : 1, lat = has_link ? m->link_lat_ps[1] : 0;
  // per kernel: weight bytes, other bytes, flops
  std::vector<u64> wb(K), ab(K), fl(K);
  for (uint32_t k = 0; k < K; ++k) {
    const Kernel& Kk = g->kernels[k];
    std::vector<Span> wr, rd, wo;
    for (const auto& sp : Kk.reads) (g->buffers[sp.buf].flags & KD_BUF_WEIGHT ? wr : rd).push_back(sp);
    for (const auto& sp : Kk.writes) (g->buffers[sp.buf].flags & KD_BUF_WEIGHT ? wr : wo).push_back(sp);
    wb[k] = union_bytes(wr);
    ab[k] = union_bytes(rd) + union_bytes(wo);
    fl[k] = Kk.flops;
  }
  auto t_of = [&](u64 bytes, u64 flops) -> i64 {
    return (i64)(std::max(ceil_div_u128((u128)bytes * kPs, hbm), ceil_div_u128((u128)flops * kPs, tc)) + m->launch_ps);
  };
  const auto pairs = edge_pairs(*g);
  const uint32_t counts[4] = {1, 2, 4, 8};
  uint32_t nout = 0;
  for (uint32_t gpus : counts) {
    if (gpus > max_gpus || (gpus > 1 && !has_link)) continue;
    if (nout == cap) {
      *n_out = nout;
      return fail(KD_ERR_RANGE, "kd_place_roles: capacity too small");
    }
    kd_role_layout bl{};
    bool have = false;
    std::vector<int32_t> brole(K, 0);
    const uint32_t a_lo = gpus == 1 ? 1 : 1, a_hi = gpus == 1 ? 1 : gpus - 1;
    for (uint32_t a = a_lo; a <= a_hi; ++a) {
      const uint32_t gr = gpus - a;
      for (uint32_t j = 0; j < 3; ++j) {
        if (!(micro_mask & (1u << j))) continue;
        const i64 N = (i64)1 << j;
        const uint64_t n_masks = gpus == 1 ? 1 : (1ull << free_cls.size());
        for (uint64_t mask = 0; mask < n_masks; ++mask) {
          std::vector<uint8_t> role_c(C, 0);
          for (uint32_t c = 0; c < C; ++c) role_c[c] = fixed[c] > 0 ? 1 : 0;
          if (gpus > 1)
            for (size_t b = 0; b < free_cls.size(); ++b) role_c[free_cls[b]] = (mask >> b) & 1;
          else
            std::fill(role_c.begin(), role_c.end(), 0);
          i64 Tm = 0, Tg = 0, Mm = 0, Mg = 0;
          for (uint32_t k = 0; k < K; ++k) {
            if (!role_c[cls_of[k]]) {
              Tm += t_of(wb[k] + ab[k], fl[k]);
            } else {
              Tg += t_of(ceil_div(wb[k], gr) + (u64)a * ab[k], ceil_div((u64)a * fl[k], gr));
            }
          }
          for (const auto& e : pairs) {
            const uint8_t ri = role_c[cls_of[e.first.first]], rj = role_c[cls_of[e.first.second]];
            if (ri == rj) continue;
            if (rj == 1)  // memory -> GEMM: every GEMM GPU gathers all a shards' rows
              Mg += (i64)a * (i64)(lat + ceil_div_u128((u128)e.second * kPs, bw));
            else          // GEMM -> memory: every memory GPU receives from the gr GEMM GPUs
              Mm += (i64)gr * (i64)(lat + ceil_div_u128((u128)ceil_div(e.second, gr) * kPs, bw));
          }
          Tm *= N, Tg *= N, Mm *= N, Mg *= N;
          const i64 period = N == 1 ? Tm + Tg + Mm + Mg : std::max(std::max(Tm, Tg), std::max(Mm, Mg));
          const u64 tok = (u64)a * (u64)N * rows;
          // better: tok/period larger (same gpus) — compare tok·period_best > tok_best·period
          const bool better = !have || (u128)tok * (u128)bl.period_ps > (u128)bl.tokens_per_step * (u128)period;
          if (better) {
            have = true;
            bl = {gpus, a, gr, (uint32_t)N, period, Tm, Tg, Mm, Mg, tok, mask};
            for (uint32_t k = 0; k < K; ++k) brole[k] = role_c[cls_of[k]];
          }
        }
      }
    }
    best[nout] = bl;
    std::copy(brole.begin(), brole.end(), roles + (size_t)nout * K);
    ++nout;
  }
  *n_out = nout;
  return KD_OK;
}

kd_status kd_chunks(uint64_t len, uint64_t unit, uint32_t n, uint64_t* begin_end, uint32_t cap, uint32_t* n_out) {
  if (!n_out || unit == 0 || n == 0 || len == 0) return fail(KD_ERR_INVALID_ARG, "kd_chunks: bad argument");
  u64 q = ceil_div(ceil_div(len, unit), n) * unit;
  std::vector<u64> out;
  for (uint32_t c = 0; c < n; ++c) {
    u64 a = (u64)c * q, b = std::min((u64)(c + 1) * q, (u64)len);
    if (a < b) {
      out.push_back(a);
      out.push_back(b);
    }
  }
  uint32_t cnt = (uint32_t)(out.size() / 2);
  if (cap < cnt || !begin_end) {
    *n_out = cnt;
    return fail(KD_ERR_RANGE, "kd_chunks: capacity too small");
  }
  std::copy(out.begin(), out.end(), begin_end);
  *n_out = cnt;
  return KD_OK;
}

}  // extern "C"
