// runtime.cu — per-device execution of a plan (§3.3 GPU workers:
// "each GPU worker only executes the kernels assigned to it" P:378; recv
// before k / send after k P:380; per-GPU CUDA-graph subgraphs P:398, P:456;
// pipelined requests P:401-402). B200 redesign:
//  * the send is fused into the producer kernel (peer stores of its primary
//    output into the consumer GPU's landing slot + a system-scope release of
//    a per-(micro-batch, producer, device) flag), see common.cuh `Epi`;
//  * the recv is a 1-warp wait kernel on the consumer's stream that acquires
//    the flag (target = epoch × signals; epochs advance once per step, so
//    flags are never reset);
//  * each device replays its static schedule (a subsequence of one global
//    topological order → deadlock free) from a CUDA graph;
//  * a step-begin barrier keeps a device from overwriting landing slots of a
//    step its peers are still reading (WAR, R4).
#include <algorithm>
#include <map>
#include <set>
#include <cstdlib>

#include "launch.hpp"

namespace kd {

struct Launch {
  enum Kind { KERNEL, WAIT, STEP_BEGIN } kind = KERNEL;
  uint32_t micro = 0, kernel = 0, op = 0;
  std::vector<void*> rd, wr;
  LaunchCtx ctx;
  WaitList wait;
  GemmPlan* gemm = nullptr;  // owned
  // step-begin barrier words
  std::vector<unsigned*> bar_mine, bar_slots;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
};

struct DevState {
  uint32_t logical = 0;
  int cuda = 0;
  uint8_t* ws = nullptr;
  uint64_t ws_bytes = 0;
  std::vector<Launch> launches;
  cudaGraphExec_t exec = nullptr;
  bool captured = false;
  cudaEvent_t st0 = nullptr, st1 = nullptr;  // kd_step_stats
  MegaPlan* mega = nullptr;                  // KD_EXEC_MEGAKERNEL
  uint64_t mega_bytes = 0;
  void* mega_ws = nullptr;                   // caller-owned (kd_runtime_set_exec_workspace)
  uint64_t mega_ws_bytes = 0;
  // profiled op timing inside a captured graph: the event-record nodes hang
  // off a side stream (fork after the previous node, join at the end), so the
  // profiled kernel keeps its programmatic (PDL) edges to its neighbours
  cudaStream_t pside = nullptr;
  cudaEvent_t pfork = nullptr, pjoin = nullptr;
  bool pside_used = false;
};

}  // namespace kd

struct kd_runtime {
  const kd_plan* plan = nullptr;
  std::vector<kd::DevState> devs;              // local devices
  std::vector<uint8_t*> ws_of;                 // workspace base per logical device (local or peer-mapped)
  std::map<std::tuple<uint32_t, uint32_t, uint32_t>, void*> bind;  // (buf, micro, dev)
  std::map<std::tuple<uint32_t, uint32_t, uint32_t>, void*> peer_bind;  // replicas of remote devices (IPC-mapped)
  uint32_t mode = KD_MODE_DISAGG;
  uint32_t exec = KD_EXEC_GRAPH;
  bool use_graph = true;
  bool prepared = false;
  uint32_t profile_op = 0;
  // steps run in KD_MODE_NO_TRANSFER: their epochs advanced without any flag
  // release, so the DISAGG wait target is (epoch − nt_steps) × signals
  uint32_t nt_steps = 0;
  uint64_t steps = 0;  // kd_step calls so far (the next step_id)
  ~kd_runtime() {
    for (auto& d : devs) {
      cudaSetDevice(d.cuda);
      if (d.exec) cudaGraphExecDestroy(d.exec);
      if (d.st0) cudaEventDestroy(d.st0);
      if (d.st1) cudaEventDestroy(d.st1);
      if (d.pside) cudaStreamDestroy(d.pside);
      if (d.pfork) cudaEventDestroy(d.pfork);
      if (d.pjoin) cudaEventDestroy(d.pjoin);
      mega_destroy(d.mega);
      for (auto& l : d.launches) {
        delete l.gemm;
        if (l.ev0) cudaEventDestroy(l.ev0);
        if (l.ev1) cudaEventDestroy(l.ev1);
      }
    }
  }
};

using namespace kd;

namespace {

template <typename T>
T attrs_get(const Kernel& k) {
  T a;
  std::memcpy(&a, k.attrs.data(), sizeof(T));
  return a;
}

kd_status check_attrs(const Kernel& k) {
  size_t need = 0;
  switch (k.op) {
    case KD_OP_NONE: return KD_OK;
    case KD_OP_ADD_RMSNORM: need = sizeof(kd_attr_add_rmsnorm); break;
    case KD_OP_GEMM:
    case KD_OP_GEMM_SILU: need = sizeof(kd_attr_gemm); break;
    case KD_OP_QKV_ROPE: need = sizeof(kd_attr_qkv_rope); break;
    case KD_OP_GEMM_RMSNORM: need = sizeof(kd_attr_gemm_rmsnorm); break;
    case KD_OP_ATTN_MERGE: need = sizeof(kd_attr_attn_merge); break;
    case KD_OP_ROPE_APPEND: need = sizeof(kd_attr_rope_append); break;
    case KD_OP_ATTENTION: need = sizeof(kd_attr_attention); break;
    case KD_OP_SILU_MUL: need = sizeof(kd_attr_silu_mul); break;
    case KD_OP_RESIDUAL_ADD: need = sizeof(kd_attr_residual_add); break;
    case KD_OP_MOE_ROUTE: need = sizeof(kd_attr_moe_route); break;
    case KD_OP_MOE_DISPATCH: need = sizeof(kd_attr_moe_dispatch); break;
    case KD_OP_GROUPED_GEMM: need = sizeof(kd_attr_grouped_gemm); break;
    case KD_OP_MOE_COMBINE: need = sizeof(kd_attr_moe_combine); break;
    case KD_OP_SSM_CONV:
    case KD_OP_SSM_UPDATE:
    case KD_OP_GATED_NORM: need = sizeof(kd_attr_ssm); break;
    case KD_OP_ROPE_PREFILL: need = sizeof(kd_attr_rope_prefill); break;
    case KD_OP_PREFILL_ATTENTION: need = sizeof(kd_attr_prefill_attention); break;
    default: return fail(KD_ERR_UNSUPPORTED, "runtime: unknown op");
  }
  if (k.attrs.size() != need) return fail(KD_ERR_INVALID_ARG, "runtime: op attrs have the wrong size");
  // read/write arity per op (kd.h op table)
  size_t nr = k.reads.size(), nw = k.writes.size();
  bool ok = true;
  switch (k.op) {
    case KD_OP_ADD_RMSNORM: {
      kd_attr_add_rmsnorm a;
      std::memcpy(&a, k.attrs.data(), sizeof a);
      ok = a.n_delta <= (uint32_t)kMaxDeltas && nr == 2 + a.n_delta && nw == 2;
      break;
    }
    case KD_OP_GEMM: ok = nr == 2 && nw == 1; break;
    case KD_OP_GEMM_SILU: ok = (nr == 2 || nr == 3) && nw == 1; break;  // (+ deferred-norm partial sums)
    case KD_OP_QKV_ROPE: ok = (nr == 4 || nr == 5) && nw == 3; break;  // reads [X, W', bt, sl (, ssq)] writes [q, Kc, Vc]
    case KD_OP_GEMM_RMSNORM: {  // reads [X, W, r, gamma] writes [h, r] (deferred: [xs, r, ssq])
      kd_attr_gemm_rmsnorm a;
      std::memcpy(&a, k.attrs.data(), sizeof a);
      ok = nr == 4 && nw == ((a.flags & KD_NORM_DEFER) ? 3u : 2u);
      break;
    }
    case KD_OP_ATTN_MERGE: {
      kd_attr_attn_merge a;
      std::memcpy(&a, k.attrs.data(), sizeof a);
      ok = a.n_parts >= 1 && a.n_parts <= 8 && nr == a.n_parts && nw == 1;
      break;
    }
    case KD_OP_ROPE_APPEND: ok = nr == 3 && nw == 3; break;
    case KD_OP_ATTENTION: ok = nr == 5 && nw == 1; break;
    case KD_OP_SILU_MUL: ok = nr == 1 && nw == 1; break;
    case KD_OP_RESIDUAL_ADD: {
      kd_attr_residual_add a;
      std::memcpy(&a, k.attrs.data(), sizeof a);
      ok = a.n_delta >= 1 && a.n_delta <= (uint32_t)kMaxDeltas && nr == 1 + a.n_delta && nw == 1;
      break;
    }
    case KD_OP_MOE_ROUTE: ok = nr == 2 && nw == 1; break;
    case KD_OP_MOE_DISPATCH: ok = nr == 2 && nw == 1; break;  // writes [meta | xg]
    case KD_OP_GROUPED_GEMM: ok = nr == 3 && nw == 1; break;  // reads [xg, W, meta]
    case KD_OP_MOE_COMBINE: {  // reads [yg_0 .. yg_{n_parts-1}, route, meta]
      kd_attr_moe_combine a;
      std::memcpy(&a, k.attrs.data(), sizeof a);
      ok = nr == std::max(1u, a.n_parts) + 2 && nw == 1;
      break;
    }
    case KD_OP_SSM_CONV: ok = nr == 4 && nw == 2; break;      // reads [zx, w, b, state] writes [xbc, state]
    case KD_OP_SSM_UPDATE: ok = nr == 6 && nw == 2; break;    // reads [xbc, zx, dt_b, A_log, D, S] writes [y, S]
    case KD_OP_GATED_NORM: ok = nr == 3 && nw == 1; break;    // reads [y, zx, w]
    case KD_OP_ROPE_PREFILL: ok = nr == 2 && nw == 3; break;  // reads [qkv, bt] writes [q, Kc, Vc]
    case KD_OP_PREFILL_ATTENTION: ok = nr == 4 && nw == 1; break;  // reads [q, Kc, Vc, bt]
  }
  if (!ok) return fail(KD_ERR_INVALID_ARG, "runtime: wrong number of read/write spans for the op");
  return KD_OK;
}

inline cudaError_t record(cudaEvent_t e, cudaStream_t s, bool capturing) {
  return capturing ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal) : cudaEventRecord(e, s);
}
// timing event of a profiled launch: while capturing, recorded on the side
// stream after a fork from s (a full edge from the node s last added), which
// leaves s's own kernel-to-kernel edges programmatic. ev0 then completes when
// the kernel before the profiled one completes, ev1 when the profiled one does.
inline cudaError_t record_prof(DevState& d, cudaEvent_t e, cudaStream_t s, bool capturing) {
  if (!capturing || !d.pside) return record(e, s, capturing);
  cudaError_t ce = cudaEventRecord(d.pfork, s);
  if (ce == cudaSuccess) ce = cudaStreamWaitEvent(d.pside, d.pfork, 0);
  if (ce == cudaSuccess) ce = record(e, d.pside, true);
  d.pside_used = true;
  return ce;
}

kd_status enqueue(kd_runtime* rt, DevState& d, Launch& l, cudaStream_t s, bool capturing) {
  uint8_t* ws = d.ws;
  const auto& L = rt->plan->layout[d.logical];
  unsigned* epoch = (unsigned*)(ws + L.ctrl_off);
  unsigned* err = epoch + 1;
  if (l.kind == Launch::STEP_BEGIN)
    return launch_step_begin(epoch, l.bar_mine.data(), l.bar_slots.data(), (int)l.bar_mine.size(), s);
  if (l.kind == Launch::WAIT) return launch_wait(l.wait, epoch, rt->nt_steps, err, s);
  LaunchCtx c = l.ctx;
  c.stream = s;
  if (rt->mode == KD_MODE_NO_TRANSFER) {
    c.epi.n = 0;
    c.acq.n = 0;
  }
  const bool prof = rt->profile_op && l.op == rt->profile_op;
  if (prof) KD_CUDA_CHECK(record_prof(d, l.ev0, s, capturing), "event record");
  kd_status st = KD_OK;
  const Kernel& K = rt->plan->g->kernels[l.kernel];
  uint32_t sig = 0;
  switch (l.op) {
    case KD_OP_NONE: break;
    case KD_OP_ADD_RMSNORM: {
      auto a = attrs_get<kd_attr_add_rmsnorm>(K);
      Deltas d;
      d.n = (int)a.n_delta;
      for (int i = 0; i < d.n; ++i) d.p[i] = (const __nv_bfloat16*)l.rd[1 + i];
      st = launch_add_rmsnorm(a, (float*)l.wr[1], d, l.rd[1 + a.n_delta], l.wr[0], c, &sig);
      break;
    }
    case KD_OP_GEMM:
    case KD_OP_GEMM_SILU:
    case KD_OP_QKV_ROPE:
    case KD_OP_GEMM_RMSNORM: st = launch_gemm(*l.gemm, l.wr[0], c, &sig); break;
    case KD_OP_ROPE_APPEND: {
      auto a = attrs_get<kd_attr_rope_append>(K);
      st = launch_rope_append(a, l.rd[0], (const int32_t*)l.rd[1], (const int32_t*)l.rd[2], l.wr[0], l.wr[1],
                              l.wr[2], c, &sig);
      break;
    }
    case KD_OP_ATTENTION: {
      auto a = attrs_get<kd_attr_attention>(K);
      st = launch_attention(a, l.rd[0], l.rd[1], l.rd[2], (const int32_t*)l.rd[3], (const int32_t*)l.rd[4], l.wr[0],
                            c, &sig);
      break;
    }
    case KD_OP_SILU_MUL: {
      auto a = attrs_get<kd_attr_silu_mul>(K);
      st = launch_silu_mul(a, l.rd[0], l.wr[0], c, &sig);
      break;
    }
    case KD_OP_ATTN_MERGE: {
      auto a = attrs_get<kd_attr_attn_merge>(K);
      st = launch_attn_merge(a, (const void* const*)l.rd.data(), l.wr[0], c, &sig);
      break;
    }
    case KD_OP_RESIDUAL_ADD: {
      auto a = attrs_get<kd_attr_residual_add>(K);
      Deltas d;
      d.n = (int)a.n_delta;
      for (int i = 0; i < d.n; ++i) d.p[i] = (const __nv_bfloat16*)l.rd[1 + i];
      st = launch_residual_add(a, (float*)l.wr[0], d, c, &sig);
      break;
    }
    case KD_OP_MOE_ROUTE: {
      auto a = attrs_get<kd_attr_moe_route>(K);
      st = launch_moe_route(a, l.rd[0], (const float*)l.rd[1], l.wr[0], c, &sig);
      break;
    }
    case KD_OP_MOE_DISPATCH: {
      auto a = attrs_get<kd_attr_moe_dispatch>(K);
      uint64_t mb = 0;
      kd_moe_meta_bytes(a.rows, a.experts, a.top_k, &mb);
      st = launch_moe_dispatch(a, l.rd[0], l.rd[1], (uint8_t*)l.wr[0] + mb, l.wr[0], c, &sig);
      break;
    }
    case KD_OP_GROUPED_GEMM: st = launch_gemm(*l.gemm, l.wr[0], c, &sig); break;
    case KD_OP_SSM_CONV: {
      auto a = attrs_get<kd_attr_ssm>(K);
      st = launch_ssm_conv(a, l.rd[0], l.rd[1], l.rd[2], l.wr[1], l.wr[0], c, &sig);
      break;
    }
    case KD_OP_SSM_UPDATE: {
      auto a = attrs_get<kd_attr_ssm>(K);
      st = launch_ssm_update(a, l.rd[0], l.rd[1], (const float*)l.rd[2], (const float*)l.rd[3], (const float*)l.rd[4],
                             (float*)l.wr[1], l.wr[0], c, &sig);
      break;
    }
    case KD_OP_GATED_NORM: {
      auto a = attrs_get<kd_attr_ssm>(K);
      st = launch_gated_norm(a, l.rd[0], l.rd[1], l.rd[2], l.wr[0], c, &sig);
      break;
    }
    case KD_OP_MOE_COMBINE: {
      auto a = attrs_get<kd_attr_moe_combine>(K);
      const uint32_t np = std::max(1u, a.n_parts);
      st = launch_moe_combine(a, (const void* const*)l.rd.data(), l.rd[np], l.rd[np + 1], l.wr[0], c, &sig);
      break;
    }
    case KD_OP_ROPE_PREFILL: {
      auto a = attrs_get<kd_attr_rope_prefill>(K);
      st = launch_rope_prefill(a, l.rd[0], (const int32_t*)l.rd[1], l.wr[0], l.wr[1], l.wr[2], c, &sig);
      break;
    }
    case KD_OP_PREFILL_ATTENTION: {
      auto a = attrs_get<kd_attr_prefill_attention>(K);
      st = launch_prefill_attention(a, l.rd[0], l.rd[1], l.rd[2], (const int32_t*)l.rd[3], l.wr[0], c, &sig);
      break;
    }
  }
  if (st) return st;
  if (prof) KD_CUDA_CHECK(record_prof(d, l.ev1, s, capturing), "event record");
  if (!capturing && getenv("KD_DEBUG_SYNC")) {
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess)
      return fail(KD_ERR_CUDA, std::string("kernel ") + std::to_string(l.kernel) + " (op " + std::to_string(l.op) +
                                   ", micro " + std::to_string(l.micro) + ") failed: " + cudaGetErrorString(e));
  }
  return KD_OK;
}

}  // namespace

extern "C" {

kd_status kd_runtime_create(const kd_plan* p, const uint32_t* local_devs, const int32_t* cuda_ordinal, uint32_t n_local,
                            kd_runtime** out) {
  if (!p || !local_devs || !cuda_ordinal || !out || n_local == 0)
    return fail(KD_ERR_INVALID_ARG, "kd_runtime_create: bad argument");
  auto* rt = new kd_runtime();
  rt->plan = p;
  rt->ws_of.assign(p->n_dev, nullptr);
  std::set<uint32_t> seen;
  for (uint32_t j = 0; j < n_local; ++j) {
    if (local_devs[j] >= p->n_dev || !seen.insert(local_devs[j]).second) {
      delete rt;
      return fail(KD_ERR_INVALID_ARG, "kd_runtime_create: bad or duplicate logical device");
    }
    DevState d;
    d.logical = local_devs[j];
    d.cuda = cuda_ordinal[j];
    rt->devs.push_back(d);
  }
  *out = rt;
  return KD_OK;
}

void kd_runtime_destroy(kd_runtime* rt) { delete rt; }

kd_status kd_runtime_bind(kd_runtime* rt, uint32_t buf, uint32_t micro, uint32_t dev, void* dev_ptr) {
  if (!rt || !dev_ptr) return fail(KD_ERR_INVALID_ARG, "kd_runtime_bind: NULL argument");
  const kd_graph* g = rt->plan->g;
  if (buf >= g->buffers.size() || dev >= rt->plan->n_dev) return fail(KD_ERR_INVALID_ARG, "kd_runtime_bind: bad id");
  const uint32_t EXT = KD_BUF_WEIGHT | KD_BUF_INPUT | KD_BUF_OUTPUT | KD_BUF_PERSISTENT;
  if (!(g->buffers[buf].flags & EXT)) return fail(KD_ERR_INVALID_ARG, "kd_runtime_bind: internal buffers live in the workspace");
  bool per = g->buffers[buf].flags & KD_BUF_PER_MICROBATCH;
  if (per ? micro >= rt->plan->n_micro : micro != 0) return fail(KD_ERR_INVALID_ARG, "kd_runtime_bind: bad micro-batch");
  rt->bind[{buf, micro, dev}] = dev_ptr;
  rt->prepared = false;
  return KD_OK;
}

kd_status kd_runtime_set_workspace(kd_runtime* rt, uint32_t dev, void* dev_ptr, uint64_t bytes) {
  if (!rt || !dev_ptr) return fail(KD_ERR_INVALID_ARG, "kd_runtime_set_workspace: NULL argument");
  for (auto& d : rt->devs)
    if (d.logical == dev) {
      if (bytes < rt->plan->layout[dev].total) return fail(KD_ERR_OOM, "kd_runtime_set_workspace: workspace too small");
      if ((uintptr_t)dev_ptr & 255) return fail(KD_ERR_INVALID_ARG, "kd_runtime_set_workspace: need 256-byte alignment");
      d.ws = (uint8_t*)dev_ptr;
      d.ws_bytes = bytes;
      rt->ws_of[dev] = (uint8_t*)dev_ptr;
      rt->prepared = false;
      return KD_OK;
    }
  return fail(KD_ERR_INVALID_ARG, "kd_runtime_set_workspace: device is not local");
}

kd_status kd_runtime_set_peer_workspace(kd_runtime* rt, uint32_t dev, void* mapped_ptr) {
  if (!rt || !mapped_ptr || dev >= rt->plan->n_dev) return fail(KD_ERR_INVALID_ARG, "kd_runtime_set_peer_workspace: bad argument");
  for (auto& d : rt->devs)
    if (d.logical == dev) return fail(KD_ERR_INVALID_ARG, "kd_runtime_set_peer_workspace: device is local");
  rt->ws_of[dev] = (uint8_t*)mapped_ptr;
  rt->prepared = false;
  return KD_OK;
}

kd_status kd_runtime_set_peer_buffer(kd_runtime* rt, uint32_t buf, uint32_t micro, uint32_t dev, void* mapped_ptr) {
  if (!rt || !mapped_ptr || dev >= rt->plan->n_dev || buf >= rt->plan->g->buffers.size())
    return fail(KD_ERR_INVALID_ARG, "kd_runtime_set_peer_buffer: bad argument");
  if (!buf_replicated(*rt->plan->g, buf)) return fail(KD_ERR_INVALID_ARG, "kd_runtime_set_peer_buffer: not a REPLICATED buffer");
  for (auto& d : rt->devs)
    if (d.logical == dev) return fail(KD_ERR_INVALID_ARG, "kd_runtime_set_peer_buffer: device is local");
  rt->peer_bind[{buf, micro, dev}] = mapped_ptr;
  rt->prepared = false;
  return KD_OK;
}

kd_status kd_runtime_set_mode(kd_runtime* rt, uint32_t mode) {
  if (!rt || mode > KD_MODE_LOG) return fail(KD_ERR_INVALID_ARG, "kd_runtime_set_mode: bad argument");
  // (LOG = DISAGG plus per-chunk %globaltimer records; its epochs carry releases)
  rt->mode = mode;
  rt->prepared = false;
  for (auto& d : rt->devs) d.captured = false;
  return KD_OK;
}

kd_status kd_runtime_set_graph(kd_runtime* rt, int32_t enable) {
  if (!rt) return fail(KD_ERR_INVALID_ARG, "kd_runtime_set_graph: NULL runtime");
  rt->use_graph = enable != 0;
  for (auto& d : rt->devs) d.captured = false;
  return KD_OK;
}

kd_status kd_runtime_profile_op(kd_runtime* rt, uint32_t op) {
  if (!rt) return fail(KD_ERR_INVALID_ARG, "kd_runtime_profile_op: NULL runtime");
  rt->profile_op = op;
  rt->prepared = false;  // re-prepare (events) and re-capture with event nodes
  return KD_OK;
}

kd_status kd_runtime_prepare(kd_runtime* rt) {
  if (!rt) return fail(KD_ERR_INVALID_ARG, "kd_runtime_prepare: NULL runtime");
  const kd_plan* P = rt->plan;
  const kd_graph* g = P->g;
  const uint32_t n = P->n_dev;
  const uint32_t EXT = KD_BUF_WEIGHT | KD_BUF_INPUT | KD_BUF_OUTPUT | KD_BUF_PERSISTENT;
  for (uint32_t v = 0; v < n; ++v)
    if (!rt->ws_of[v]) return fail(KD_ERR_STATE, "kd_runtime_prepare: workspace of device " + std::to_string(v) + " not set");
  for (const auto& K : g->kernels) {
    kd_status s = check_attrs(K);
    if (s) return s;
  }
  // transfer lookup: (micro, producer, dst) -> transfer index
  std::map<std::tuple<uint32_t, uint32_t, uint32_t>, uint32_t> xidx;
  for (uint32_t t = 0; t < P->transfers.size(); ++t) {
    const auto& x = P->transfers[t];
    xidx[{x.micro, x.producer, x.dst_dev}] = t;
  }
  // incoming remote producers per (consumer kernel, buffer)
  std::map<std::pair<uint32_t, uint32_t>, std::set<uint32_t>> remote_src;
  for (const auto& e : g->edges)
    if (P->assign[e.src] != P->assign[e.dst]) remote_src[{e.dst, e.buf}].insert(e.src);

  for (auto& d : rt->devs) {
    KD_CUDA_CHECK(cudaSetDevice(d.cuda), "cudaSetDevice");
    kd_status s = kernels_init();
    if (s) return s;
    // peer access to every other physical device we store into
    for (uint32_t v = 0; v < n; ++v) {
      if (v == d.logical) continue;
      for (auto& o : rt->devs)
        if (o.logical == v && o.cuda != d.cuda) {
          int can = 0;
          cudaDeviceCanAccessPeer(&can, d.cuda, o.cuda);
          if (can) {
            cudaError_t e = cudaDeviceEnablePeerAccess(o.cuda, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return set_cuda_error(e, "peer access");
            cudaGetLastError();
          }
        }
    }
    for (auto& l : d.launches) {
      delete l.gemm;
      if (l.ev0) cudaEventDestroy(l.ev0);
      if (l.ev1) cudaEventDestroy(l.ev1);
    }
    d.launches.clear();
    if (d.exec) {
      cudaGraphExecDestroy(d.exec);
      d.exec = nullptr;
    }
    d.captured = false;
    const auto& L = P->layout[d.logical];
    auto local_ptr = [&](uint32_t buf, uint32_t i, uint64_t off) -> void* {
      const auto& B = g->buffers[buf];
      uint32_t inst = (B.flags & KD_BUF_PER_MICROBATCH) ? i : 0;
      if (B.flags & EXT) {
        auto it = rt->bind.find({buf, inst, d.logical});
        if (it == rt->bind.end()) return nullptr;
        return (uint8_t*)it->second + off;
      }
      auto it = L.act.find({buf, inst});
      if (it == L.act.end()) return nullptr;
      return d.ws + it->second + off;
    };
    const bool multi = n > 1;
    const bool transfers_on = rt->mode != KD_MODE_NO_TRANSFER;
    if (multi) {
      Launch sb;
      sb.kind = Launch::STEP_BEGIN;
      for (uint32_t v = 0; v < n; ++v) {
        if (v == d.logical) continue;
        sb.bar_mine.push_back((unsigned*)(d.ws + L.ctrl_off + 64 + 4 * v));
        sb.bar_slots.push_back((unsigned*)(rt->ws_of[v] + P->layout[v].ctrl_off + 64 + 4 * d.logical));
      }
      d.launches.push_back(sb);
    }
    const bool log_on = rt->mode == KD_MODE_LOG;
    const unsigned* my_epoch = (const unsigned*)(d.ws + L.ctrl_off);
    // logical devices driven by this process on the same GPU as d (loopback)
    auto loopback = [&](uint32_t v) {
      for (auto& o : rt->devs)
        if (o.logical == v) return o.cuda == d.cuda;
      return false;  // another process: time-sliced, never co-scheduled with d's kernels
    };
    std::set<uint32_t> waited;
    for (const auto& e : P->sched) {
      if (e.dev != d.logical) continue;
      const uint32_t i = e.micro, k = e.kernel;
      const Kernel& K = g->kernels[k];
      Launch l;
      l.kind = Launch::KERNEL;
      l.micro = i;
      l.kernel = k;
      l.op = K.op;
      WaitList wl;
      auto push_wait = [&](const unsigned long long* flag, unsigned long long mult, unsigned long long* log) {
        if (wl.n == kMaxWait) {
          Launch w;
          w.kind = Launch::WAIT;
          w.wait = wl;
          d.launches.push_back(w);
          wl.n = 0;
        }
        wl.flag[wl.n] = flag;
        wl.mult[wl.n] = mult;
        wl.log[wl.n] = log;
        ++wl.n;
      };
      l.ctx.acq.epoch = my_epoch;
      l.ctx.acq.base = rt->nt_steps;
      l.ctx.acq.err = (unsigned*)(d.ws + L.ctrl_off + 4);
      for (uint32_t ri = 0; ri < K.reads.size(); ++ri) {
        const auto& sp = K.reads[ri];
        auto rs = remote_src.find({k, sp.buf});
        if (rs == remote_src.end()) {
          void* ptr = local_ptr(sp.buf, i, sp.off);
          if (!ptr) return fail(KD_ERR_STATE, "kd_runtime_prepare: buffer " + std::to_string(sp.buf) + " not bound on device " + std::to_string(d.logical));
          l.rd.push_back(ptr);
          continue;
        }
        // remote producers whose writes this span reads (bipartite gather: one
        // per source device's row span; local writers are ordered by the stream)
        std::vector<uint32_t> srcs_here;
        for (uint32_t src : rs->second) {
          bool hit = false;
          for (const auto& e2 : g->edges)
            if (e2.dst == k && e2.src == src && e2.buf == sp.buf && e2.offset < sp.off + sp.len &&
                sp.off < e2.offset + e2.len)
              hit = true;
          if (!hit) continue;
          const Kernel& S = g->kernels[src];
          if (!buf_replicated(*g, sp.buf))  // (replicated state arrives as the producer's mirrored deltas)
            for (const auto& e2 : g->edges)
              if (e2.dst == k && e2.src == src && e2.buf == sp.buf &&
                  (S.writes.empty() || S.writes[0].buf != sp.buf || e2.offset < S.writes[0].off ||
                   e2.offset + e2.len > S.writes[0].off + S.writes[0].len))
                return fail(KD_ERR_UNSUPPORTED, "kd_runtime_prepare: a cut edge must read the producer's primary output");
          srcs_here.push_back(src);
        }
        if (srcs_here.empty()) {
          void* ptr = local_ptr(sp.buf, i, sp.off);
          if (!ptr) return fail(KD_ERR_STATE, "kd_runtime_prepare: buffer " + std::to_string(sp.buf) + " not bound on device " + std::to_string(d.logical));
          l.rd.push_back(ptr);
          continue;
        }
        const bool ext = g->buffers[sp.buf].flags & EXT;
        if (buf_replicated(*g, sp.buf)) {  // this device's own replica (deltas mirrored into it)
          void* ptr = local_ptr(sp.buf, i, sp.off);
          if (!ptr) return fail(KD_ERR_STATE, "kd_runtime_prepare: replica of buffer " + std::to_string(sp.buf) + " not bound on device " + std::to_string(d.logical));
          l.rd.push_back(ptr);
        } else if (ext) {  // external buffer: one remote producer, its private landing slot
          if (srcs_here.size() != 1)
            return fail(KD_ERR_UNSUPPORTED, "kd_runtime_prepare: an external buffer read span with several remote producers");
          const Kernel& S = g->kernels[srcs_here[0]];
          for (const auto& e2 : g->edges)
            if (e2.dst == k && e2.buf == sp.buf && e2.src != srcs_here[0] && e2.offset < sp.off + sp.len &&
                sp.off < e2.offset + e2.len)
              return fail(KD_ERR_UNSUPPORTED, "kd_runtime_prepare: a cut read span of an external buffer mixes writers");
          const auto& land = L.landing.at(xidx.at({i, srcs_here[0], d.logical}));
          l.rd.push_back(d.ws + land.first + (sp.off - S.writes[0].off));
        } else {  // transfers land in this device's instance of the buffer
          void* ptr = local_ptr(sp.buf, i, sp.off);
          if (!ptr) return fail(KD_ERR_STATE, "kd_runtime_prepare: no local instance of buffer " + std::to_string(sp.buf));
          l.rd.push_back(ptr);
        }
        for (uint32_t src : srcs_here) {
        const Kernel& S = g->kernels[src];
        uint32_t t = xidx.at({i, src, d.logical});
        const auto& land = L.landing.at(t);
        if (transfers_on && !waited.count(t)) {
          waited.insert(t);
          const auto& X = P->xchunks[t];
          const uint32_t nch = (uint32_t)X.ch.size();
          const unsigned long long* flags = (const unsigned long long*)(d.ws + land.second);
          unsigned long long* logp = log_on ? (unsigned long long*)(d.ws + L.xlog.at(t)) : nullptr;
          std::vector<unsigned long long> mult(nch);
          if (X.count) {
            for (uint32_t c = 0; c < nch; ++c) mult[c] = X.rows * (X.ch[c].second - X.ch[c].first);
          } else {
            uint32_t sig = 0;
            kd_status s2 = op_signals(S.op, S.attrs, &sig);
            if (s2) return s2;
            mult[0] = sig;
          }
          // chunk-aware consumer of a COUNT transfer: acquire chunk by chunk
          // inside the kernel (no wait launch); else wait for every chunk first
          // whole rows of the producer's output (all, or a scattered GEMM output's row span)
          const bool whole = X.count && sp.off >= S.writes[0].off && sp.off + sp.len <= S.writes[0].off + S.writes[0].len &&
                             (sp.off - S.writes[0].off) % X.row_bytes == 0 && sp.len % X.row_bytes == 0;
          const bool in_kernel = srcs_here.size() == 1 && X.count && whole && op_consumer_unit(K, ri, X.row_bytes) > 0 &&
                                 l.ctx.acq.n < kMaxAcqIn && !getenv("KD_NO_INKERNEL_ACQ");
          if (in_kernel) {
            AcqIn& in = l.ctx.acq.in[l.ctx.acq.n++];
            in.flag = flags;
            in.log = logp;
            in.slot = (K.op == KD_OP_ADD_RMSNORM || K.op == KD_OP_RESIDUAL_ADD) ? (int)ri - 1 : (int)ri;
            in.nch = (int)nch;
            in.row_bytes = (uint32_t)X.row_bytes;
            for (uint32_t c = 0; c < nch; ++c) {
              in.cb[c] = (uint32_t)X.ch[c].first;
              in.mult[c] = mult[c];
            }
            in.cb[nch] = (uint32_t)X.row_bytes;
            if (loopback(P->assign[src])) {
              // loopback residency gate: launch the consumer only once every CTA
              // of the producer is resident (it then spins on chunks without
              // being able to starve the producer of SMs)
              uint32_t grid = 0;
              kd_status s2 = op_grid(S.op, S.attrs, &grid);
              if (s2) return s2;
              push_wait(flags + nch, grid, nullptr);
            }
          } else {
            for (uint32_t c = 0; c < nch; ++c) push_wait(flags + c, mult[c], logp ? logp + kLogWords * c : nullptr);
          }
        }
        }  // remote producers of this span
      }
      if (wl.n) {
        Launch w;
        w.kind = Launch::WAIT;
        w.wait = wl;
        d.launches.push_back(w);
      }
      for (const auto& sp : K.writes) {
        void* ptr = local_ptr(sp.buf, i, sp.off);
        if (!ptr) return fail(KD_ERR_STATE, "kd_runtime_prepare: output buffer " + std::to_string(sp.buf) + " not bound on device " + std::to_string(d.logical));
        l.wr.push_back(ptr);
      }
      // fused sends: every remote device reading this kernel's output (all its
      // transfers share one chunk table, plan.cpp)
      for (uint32_t v = 0; v < n; ++v) {
        auto it = xidx.find({i, k, v});
        if (it == xidx.end()) continue;
        if (l.ctx.epi.n == kMaxPeers) return fail(KD_ERR_UNSUPPORTED, "kd_runtime_prepare: more than 8 consumer devices");
        const auto& X = P->xchunks[it->second];
        const uint32_t nch = (uint32_t)X.ch.size();
        Epi& ep = l.ctx.epi;
        ep.nch = X.count ? (int)nch : 0;
        ep.row_bytes = (uint32_t)X.row_bytes;
        for (uint32_t c = 0; c < nch; ++c) ep.cb[c] = (uint32_t)X.ch[c].first;
        ep.cb[nch] = (uint32_t)X.row_bytes;
        const auto& Lv = P->layout[v];
        const auto& land = Lv.landing.at(it->second);
        ep.dst[ep.n] = rt->ws_of[v] + land.first;
        ep.flag[ep.n] = (unsigned long long*)(rt->ws_of[v] + land.second);
        ep.started[ep.n] = (X.count && loopback(v)) ? (unsigned long long*)(rt->ws_of[v] + land.second) + nch : nullptr;
        u64 prows = 0, prb = 0;  // row filter: this peer reads rows [row0, row0 + rows) only
        const bool filt = X.count && op_count_geometry(K, &prows, &prb) && X.rows < prows;
        ep.r0[ep.n] = filt ? (uint32_t)X.row0 : 0u;
        ep.rn[ep.n] = filt ? (uint32_t)X.rows : 0u;
        ep.logt[ep.n] = log_on ? (unsigned long long*)(rt->ws_of[v] + Lv.xlog.at(it->second)) : nullptr;
        // delta replication: the peer's replicas of this kernel's replicated outputs
        int j = 0;
        for (const auto& w : K.writes) {
          if (!buf_replicated(*g, w.buf)) continue;
          if (K.op != KD_OP_ROPE_APPEND || j >= 2)
            return fail(KD_ERR_UNSUPPORTED, "kd_runtime_prepare: only RoPE/append mirrors replicated (KV) writes");
          const uint32_t inst = (g->buffers[w.buf].flags & KD_BUF_PER_MICROBATCH) ? i : 0;
          void* base = nullptr;
          auto bi = rt->bind.find({w.buf, inst, v});
          if (bi != rt->bind.end()) base = bi->second;
          auto pi = rt->peer_bind.find({w.buf, inst, v});
          if (pi != rt->peer_bind.end()) base = pi->second;
          if (P->needs_bind[w.buf][v] && !base)
            return fail(KD_ERR_STATE, "kd_runtime_prepare: replica of buffer " + std::to_string(w.buf) + " on device " +
                                          std::to_string(v) + " unknown (kd_runtime_set_peer_buffer)");
          ep.mir[ep.n][j++] = base ? (uint8_t*)base + w.off : nullptr;
        }
        ++ep.n;
      }
      l.ctx.scratch = d.ws + L.scratch_off;
      l.ctx.err = (unsigned*)(d.ws + L.ctrl_off + 4);
      if (K.op == KD_OP_GROUPED_GEMM) {
        l.gemm = new GemmPlan();
        kd_status s3 = gemm_prepare(gemm_shape(attrs_get<kd_attr_grouped_gemm>(K)), l.rd[0], l.rd[1], l.rd[2], l.gemm);
        if (s3) return s3;
      }
      if (K.op == KD_OP_QKV_ROPE) {
        const auto a = attrs_get<kd_attr_qkv_rope>(K);
        l.gemm = new GemmPlan();
        kd_status s3 = gemm_prepare(gemm_shape(a), l.rd[0], l.rd[1], nullptr, l.gemm);
        if (s3) return s3;
        s3 = qkv_rope_bind(a, (const int32_t*)l.rd[2], (const int32_t*)l.rd[3], l.wr[0], l.wr[1], l.wr[2], l.gemm);
        if (s3) return s3;
        if (l.rd.size() == 5) l.gemm->dssq = (const float*)l.rd[4];
      }
      if (K.op == KD_OP_GEMM_RMSNORM) {
        const auto a = attrs_get<kd_attr_gemm_rmsnorm>(K);
        l.gemm = new GemmPlan();
        kd_status s3 = gemm_prepare(gemm_shape(a), l.rd[0], l.rd[1], nullptr, l.gemm);
        if (s3) return s3;
        s3 = gemm_rmsnorm_bind(a, (float*)l.wr[1], l.rd[3], l.gemm, l.wr.size() == 3 ? (float*)l.wr[2] : nullptr);
        if (s3) return s3;
      }
      if (K.op == KD_OP_GEMM || K.op == KD_OP_GEMM_SILU) {
        l.gemm = new GemmPlan();
        kd_status s3 = gemm_prepare(gemm_shape(attrs_get<kd_attr_gemm>(K), K.op == KD_OP_GEMM_SILU), l.rd[0], l.rd[1],
                                    nullptr, l.gemm);
        if (s3) return s3;
        if (K.op == KD_OP_GEMM_SILU && l.rd.size() == 3) l.gemm->dssq = (const float*)l.rd[2];
      }
      if (rt->profile_op) {
        KD_CUDA_CHECK(cudaEventCreate(&l.ev0), "event create");
        KD_CUDA_CHECK(cudaEventCreate(&l.ev1), "event create");
        if (!d.pside) {
          KD_CUDA_CHECK(cudaStreamCreateWithFlags(&d.pside, cudaStreamNonBlocking), "profile side stream");
          KD_CUDA_CHECK(cudaEventCreateWithFlags(&d.pfork, cudaEventDisableTiming), "event create");
          KD_CUDA_CHECK(cudaEventCreateWithFlags(&d.pjoin, cudaEventDisableTiming), "event create");
        }
      }
      d.launches.push_back(std::move(l));
    }
    mega_destroy(d.mega);
    d.mega = nullptr;
    d.mega_bytes = 0;
    if (rt->exec == KD_EXEC_MEGAKERNEL) {
      std::vector<MegaOpDesc> ops;
      for (const auto& l : d.launches) {
        if (l.kind == Launch::KERNEL && l.gemm && (l.gemm->defer || l.gemm->dssq))
          return fail(KD_ERR_UNSUPPORTED, "kd_runtime_prepare: the megakernel has no deferred-norm GEMM tasks");
        if (l.kind != Launch::KERNEL || l.ctx.epi.n || l.ctx.acq.n)
          return fail(KD_ERR_UNSUPPORTED, "kd_runtime_prepare: the megakernel runs single-device schedules only "
                                          "(device " + std::to_string(d.logical) + " has cross-device transfers)");
        if (l.op == KD_OP_NONE) continue;
        const Kernel& K = g->kernels[l.kernel];
        MegaOpDesc o;
        o.op = l.op;
        o.attrs = K.attrs;
        o.rd = l.rd;
        o.wr = l.wr;
        for (const auto& sp : K.reads) o.rd_len.push_back(sp.len);
        for (const auto& sp : K.writes) o.wr_len.push_back(sp.len);
        ops.push_back(std::move(o));
      }
      kd_status s = mega_create(ops, &d.mega, &d.mega_bytes);
      if (s) return s;
      if (d.mega_ws && d.mega_ws_bytes >= d.mega_bytes) {
        KD_CUDA_CHECK(cudaMemset(d.mega_ws, 0, d.mega_bytes), "zero megakernel workspace");
        s = mega_bind(d.mega, d.mega_ws, d.mega_ws_bytes, (unsigned*)(d.ws + L.ctrl_off + 4));
        if (s) return s;
      }
    }
  }
  rt->prepared = true;
  return KD_OK;
}

kd_status kd_runtime_set_exec(kd_runtime* rt, uint32_t exec) {
  if (!rt || exec > KD_EXEC_MEGAKERNEL) return fail(KD_ERR_INVALID_ARG, "kd_runtime_set_exec: bad argument");
  if (rt->exec != exec) {
    rt->exec = exec;
    rt->prepared = false;
    for (auto& d : rt->devs) d.captured = false;
  }
  return KD_OK;
}

kd_status kd_runtime_exec_workspace_bytes(kd_runtime* rt, uint32_t dev, uint64_t* bytes) {
  if (!rt || !bytes) return fail(KD_ERR_INVALID_ARG, "kd_runtime_exec_workspace_bytes: NULL argument");
  if (rt->exec != KD_EXEC_MEGAKERNEL) return fail(KD_ERR_STATE, "kd_runtime_exec_workspace_bytes: not in KD_EXEC_MEGAKERNEL");
  if (!rt->prepared) {
    kd_status s = kd_runtime_prepare(rt);
    if (s) return s;
  }
  for (auto& d : rt->devs)
    if (d.logical == dev) {
      *bytes = d.mega_bytes;
      return KD_OK;
    }
  return fail(KD_ERR_INVALID_ARG, "kd_runtime_exec_workspace_bytes: device is not local");
}

kd_status kd_runtime_set_exec_workspace(kd_runtime* rt, uint32_t dev, void* dev_ptr, uint64_t bytes) {
  if (!rt || !dev_ptr) return fail(KD_ERR_INVALID_ARG, "kd_runtime_set_exec_workspace: NULL argument");
  if ((uintptr_t)dev_ptr & 255) return fail(KD_ERR_INVALID_ARG, "kd_runtime_set_exec_workspace: need 256-byte alignment");
  for (auto& d : rt->devs)
    if (d.logical == dev) {
      d.mega_ws = dev_ptr;
      d.mega_ws_bytes = bytes;
      if (rt->prepared && d.mega) {
        if (bytes < d.mega_bytes) return fail(KD_ERR_OOM, "kd_runtime_set_exec_workspace: workspace too small");
        KD_CUDA_CHECK(cudaSetDevice(d.cuda), "cudaSetDevice");
        KD_CUDA_CHECK(cudaMemset(dev_ptr, 0, d.mega_bytes), "zero megakernel workspace");
        return mega_bind(d.mega, dev_ptr, bytes, (unsigned*)(d.ws + rt->plan->layout[d.logical].ctrl_off + 4));
      }
      return KD_OK;
    }
  return fail(KD_ERR_INVALID_ARG, "kd_runtime_set_exec_workspace: device is not local");
}

kd_status kd_debug_mega_trace(kd_runtime* rt, uint32_t j, void* dev_buf) {
  if (!rt || j >= rt->devs.size()) return fail(KD_ERR_INVALID_ARG, "kd_debug_mega_trace: bad argument");
  if (!rt->devs[j].mega) return fail(KD_ERR_STATE, "kd_debug_mega_trace: no prepared megakernel");
  mega_set_trace(rt->devs[j].mega, dev_buf);
  return KD_OK;
}

kd_status kd_runtime_exec_info(kd_runtime* rt, uint32_t j, uint32_t* n_tasks, uint32_t* smem_bytes, uint32_t* grid) {
  if (!rt || j >= rt->devs.size()) return fail(KD_ERR_INVALID_ARG, "kd_runtime_exec_info: bad argument");
  if (!rt->prepared || !rt->devs[j].mega) return fail(KD_ERR_STATE, "kd_runtime_exec_info: no prepared megakernel");
  return mega_info(rt->devs[j].mega, n_tasks, smem_bytes, grid);
}

kd_status kd_step(kd_runtime* rt, void* const* streams, uint64_t step_id, kd_step_stats* stats) {
  if (!rt || !streams) return fail(KD_ERR_INVALID_ARG, "kd_step: NULL argument");
  if (step_id != UINT64_MAX && step_id != rt->steps)
    return fail(KD_ERR_INVALID_ARG, "kd_step: step_id " + std::to_string(step_id) + " out of order (next is " +
                                        std::to_string(rt->steps) + ")");
  if (stats && rt->devs.size() > KD_STATS_MAX_DEV) return fail(KD_ERR_UNSUPPORTED, "kd_step: stats cover <= 8 local devices");
  if (!rt->prepared) {
    kd_status s = kd_runtime_prepare(rt);
    if (s) return s;
  }
  for (size_t j = 0; j < rt->devs.size(); ++j) {
    auto& d = rt->devs[j];
    cudaStream_t s = (cudaStream_t)streams[j];
    KD_CUDA_CHECK(cudaSetDevice(d.cuda), "cudaSetDevice");
    if (stats) {
      if (!d.st0) {
        KD_CUDA_CHECK(cudaEventCreate(&d.st0), "event create");
        KD_CUDA_CHECK(cudaEventCreate(&d.st1), "event create");
      }
      KD_CUDA_CHECK(cudaEventRecord(d.st0, s), "event record");
    }
    if (rt->exec == KD_EXEC_MEGAKERNEL) {
      if (!d.mega) return fail(KD_ERR_STATE, "kd_step: megakernel not prepared");
      kd_status st = mega_launch(d.mega, s);
      if (st) return st;
    } else if (!rt->use_graph) {
      for (auto& l : d.launches) {
        kd_status st = enqueue(rt, d, l, s, false);
        if (st) return st;
      }
    } else {
      if (!d.captured) {
        if (d.exec) {
          cudaGraphExecDestroy(d.exec);
          d.exec = nullptr;
        }
        KD_CUDA_CHECK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "begin capture");
        kd_status st = KD_OK;
        d.pside_used = false;
        for (auto& l : d.launches) {
          st = enqueue(rt, d, l, s, true);
          if (st) break;
        }
        if (d.pside_used) {  // join the timing side stream back before the capture ends
          cudaError_t je = cudaEventRecord(d.pjoin, d.pside);
          if (je == cudaSuccess) je = cudaStreamWaitEvent(s, d.pjoin, 0);
          if (je != cudaSuccess && !st) st = set_cuda_error(je, "profile join");
        }
        cudaGraph_t graph = nullptr;
        cudaError_t ce = cudaStreamEndCapture(s, &graph);
        if (st) {
          if (graph) cudaGraphDestroy(graph);
          return st;
        }
        if (ce != cudaSuccess) return set_cuda_error(ce, "end capture");
        ce = cudaGraphInstantiate(&d.exec, graph, 0);
        cudaGraphDestroy(graph);
        if (ce != cudaSuccess) return set_cuda_error(ce, "graph instantiate");
        d.captured = true;
      }
      KD_CUDA_CHECK(cudaGraphLaunch(d.exec, s), "graph launch");
    }
    if (stats) KD_CUDA_CHECK(cudaEventRecord(d.st1, s), "event record");
  }
  if (rt->mode == KD_MODE_NO_TRANSFER) ++rt->nt_steps;  // graphs re-capture on the next mode switch
  const uint64_t this_step = rt->steps++;
  if (!stats) return KD_OK;
  // ---- statistics (synchronising)
  const kd_plan* P = rt->plan;
  std::memset(stats, 0, sizeof(*stats));
  stats->step_id = this_step;
  stats->n_local = (uint32_t)rt->devs.size();
  stats->n_dev = P->n_dev;
  if (P->n_dev <= KD_STATS_MAX_DEV)
    for (const auto& x : P->transfers)
      stats->link_bytes[P->assign[x.producer] * P->n_dev + x.dst_dev] += x.bytes;
  for (size_t j = 0; j < rt->devs.size(); ++j) {
    auto& d = rt->devs[j];
    KD_CUDA_CHECK(cudaSetDevice(d.cuda), "cudaSetDevice");
    KD_CUDA_CHECK(cudaEventSynchronize(d.st1), "event sync");
    float ms = 0.f;
    KD_CUDA_CHECK(cudaEventElapsedTime(&ms, d.st0, d.st1), "event elapsed");
    stats->step_ns[j] = (uint64_t)((double)ms * 1e6);
  }
  if (rt->mode == KD_MODE_LOG) {
    std::vector<kd_log_record> recs;
    uint32_t nrec = 0;
    kd_runtime_log(rt, nullptr, 0, &nrec);
    recs.resize(nrec);
    kd_status s = kd_runtime_log(rt, recs.data(), nrec, &nrec);
    if (s) return s;
    // device epoch of this step: step_begin increments it once per step (multi-device plans)
    for (const auto& r : recs) {
      for (size_t j = 0; j < rt->devs.size(); ++j)
        if (rt->devs[j].logical == r.dev && r.epoch != 0 && r.t_acquire >= r.t_wait) {
          stats->wait_ns[j] += r.t_acquire - r.t_wait;
          ++stats->chunk_waits[j];
        }
    }
  }
  return KD_OK;
}

kd_status kd_runtime_log(kd_runtime* rt, kd_log_record* out, uint32_t cap, uint32_t* n) {
  if (!rt || !n) return fail(KD_ERR_INVALID_ARG, "kd_runtime_log: NULL argument");
  if (rt->mode != KD_MODE_LOG) return fail(KD_ERR_STATE, "kd_runtime_log: runtime is not in KD_MODE_LOG");
  const kd_plan* P = rt->plan;
  uint32_t need = 0;
  for (auto& d : rt->devs)
    for (const auto& kv : P->layout[d.logical].xlog) need += (uint32_t)P->xchunks[kv.first].ch.size();
  if (cap < need || (need && !out)) {
    *n = need;
    return fail(KD_ERR_RANGE, "kd_runtime_log: capacity too small");
  }
  uint32_t i = 0;
  for (auto& d : rt->devs) {
    const auto& L = P->layout[d.logical];
    if (!L.log_bytes || !d.ws) continue;
    KD_CUDA_CHECK(cudaSetDevice(d.cuda), "cudaSetDevice");
    std::vector<unsigned long long> h(L.log_bytes / 8);
    KD_CUDA_CHECK(cudaMemcpy(h.data(), d.ws + L.log_off, L.log_bytes, cudaMemcpyDeviceToHost), "read log");
    for (const auto& kv : L.xlog) {
      const size_t base = (kv.second - L.log_off) / 8;
      for (uint32_t c = 0; c < P->xchunks[kv.first].ch.size(); ++c) {
        kd_log_record& r = out[i++];
        r.dev = d.logical;
        r.transfer = kv.first;
        r.chunk = c;
        r.pad_ = 0;
        r.epoch = h[base + (size_t)kLogWords * c + 0];
        r.t_wait = h[base + (size_t)kLogWords * c + 1];
        r.t_acquire = h[base + (size_t)kLogWords * c + 2];
        r.t_release = h[base + (size_t)kLogWords * c + 3];
      }
    }
  }
  *n = i;
  return KD_OK;
}

kd_status kd_runtime_check(kd_runtime* rt) {
  if (!rt) return fail(KD_ERR_INVALID_ARG, "kd_runtime_check: NULL runtime");
  for (auto& d : rt->devs) {
    KD_CUDA_CHECK(cudaSetDevice(d.cuda), "cudaSetDevice");
    KD_CUDA_CHECK(cudaDeviceSynchronize(), "device synchronize");
    if (d.mega) {
      std::string what;
      kd_status s = mega_diag(d.mega, &what);
      if (s) return s;
      if (!what.empty()) return fail(KD_ERR_TIMEOUT, "kd_runtime_check: " + what + " on device " + std::to_string(d.logical));
    }
    unsigned err = 0;
    KD_CUDA_CHECK(cudaMemcpy(&err, d.ws + rt->plan->layout[d.logical].ctrl_off + 4, 4, cudaMemcpyDeviceToHost),
                  "read error word");
    if (err) {
      const char* what = err == 2   ? "an in-kernel grid barrier"
                         : err == 3 ? "the step-begin barrier"
                         : err == 4 ? "a megakernel dependency wait"
                         : err == 5 ? "a megakernel pipeline wait"
                         : err == 6 ? "a megakernel split merge"
                                    : "a flag wait";
      return fail(KD_ERR_TIMEOUT, std::string("kd_runtime_check: ") + what + " timed out on device " +
                                      std::to_string(d.logical));
    }
  }
  return KD_OK;
}

kd_status kd_runtime_launch_count(const kd_runtime* rt, uint32_t j, uint32_t* n) {
  if (!rt || !n || j >= rt->devs.size()) return fail(KD_ERR_INVALID_ARG, "kd_runtime_launch_count: bad argument");
  if (!rt->prepared) return fail(KD_ERR_STATE, "kd_runtime_launch_count: runtime not prepared");
  *n = rt->exec == KD_EXEC_MEGAKERNEL ? 1u : (uint32_t)rt->devs[j].launches.size();
  return KD_OK;
}

kd_status kd_runtime_op_time(kd_runtime* rt, double* ms, uint64_t* launches) {
  if (!rt || !ms || !launches) return fail(KD_ERR_INVALID_ARG, "kd_runtime_op_time: NULL argument");
  double tot = 0;
  uint64_t cnt = 0;
  for (auto& d : rt->devs) {
    KD_CUDA_CHECK(cudaSetDevice(d.cuda), "cudaSetDevice");
    for (auto& l : d.launches)
      if (l.ev0 && l.kind == Launch::KERNEL && l.op == rt->profile_op) {
        KD_CUDA_CHECK(cudaEventSynchronize(l.ev1), "event sync");
        float t = 0;
        KD_CUDA_CHECK(cudaEventElapsedTime(&t, l.ev0, l.ev1), "event elapsed");
        tot += t;
        ++cnt;
      }
  }
  *ms = tot;
  *launches = cnt;
  return KD_OK;
}

}  // extern "C"
