"""Pythonic wrappers over the C ABI (include/kd.h). Argument marshalling only:
every computation (DAG, cost, placement, schedule, kernels) runs in libkd."""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence, Tuple

from . import _kd as K
from ._kd import check

Span = Tuple[int, int, int]  # (buf, offset, len)


def _spans(spans: Sequence[Span]):
    arr = (K.kd_span * max(1, len(spans)))()
    for i, (b, o, n) in enumerate(spans):
        arr[i].buf, arr[i].offset, arr[i].len = b, o, n
    return arr


class Graph:
    """kd_graph: buffers and kernels in program order, RAW DDG on finalize."""

    def __init__(self):
        h = C.c_void_p()
        check(K.kd_graph_create(C.byref(h)), "kd_graph_create")
        self.h = h
        self._keep = []
        # the declarations as given (op, reads, writes, attrs): introspection
        # for tests that restate the plan's rules independently
        self.decl = []
        self._desc = []       # (flops, template, pin) per kernel
        self._buf_flags = []  # flags per buffer

    def __del__(self):
        if getattr(self, "h", None):
            K.kd_graph_destroy(self.h)
            self.h = None

    def add_buffer(self, nbytes: int, flags: int = 0) -> int:
        i = C.c_uint32()
        check(K.kd_graph_add_buffer(self.h, int(nbytes), int(flags), C.byref(i)), "kd_graph_add_buffer")
        self._buf_flags.append(int(flags))
        return i.value

    def add_kernel(self, op: int, reads: Sequence[Span], writes: Sequence[Span], attrs=None, flops: int = 0,
                   pin: int = -1, template: int = -1) -> int:
        d = K.kd_kernel_desc()
        d.op, d.n_reads, d.n_writes = op, len(reads), len(writes)
        d.pin_device, d.template_id, d.flops = pin, template, int(flops)
        r, w = _spans(reads), _spans(writes)
        d.reads = C.cast(r, C.POINTER(K.kd_span))
        d.writes = C.cast(w, C.POINTER(K.kd_span))
        if attrs is not None:
            d.attrs = C.cast(C.byref(attrs), C.c_void_p)
            d.attrs_size = C.sizeof(attrs)
        i = C.c_uint32()
        check(K.kd_graph_add_kernel(self.h, C.byref(d), C.byref(i)), "kd_graph_add_kernel")
        self.decl.append((op, [tuple(x) for x in reads], [tuple(x) for x in writes], attrs))
        self._desc.append((int(flops), int(template), int(pin)))
        return i.value

    def finalize(self):
        check(K.kd_graph_finalize(self.h), "kd_graph_finalize")

    @property
    def num_kernels(self) -> int:
        n = C.c_uint32()
        check(K.kd_graph_num_kernels(self.h, C.byref(n)))
        return n.value

    def edges(self) -> List[Tuple[int, int, int, int, int]]:
        n = C.c_uint32()
        st = K.kd_graph_edges(self.h, None, 0, C.byref(n))
        if st not in (K.KD_OK, K.KD_ERR_RANGE):
            check(st, "kd_graph_edges")
        arr = (K.kd_edge * max(1, n.value))()
        check(K.kd_graph_edges(self.h, arr, n.value, C.byref(n)), "kd_graph_edges")
        return [(e.src, e.dst, e.buf, e.offset, e.len) for e in arr[:n.value]]


class Machine:
    """kd_machine from integer per-device / per-link parameters (R7)."""

    def __init__(self, hbm_Bps, tc_flops, link_Bps, link_lat_ps, launch_ps: int):
        n = len(hbm_Bps)
        self.n_dev = n
        self._hbm = (C.c_uint64 * n)(*[int(x) for x in hbm_Bps])
        self._tc = (C.c_uint64 * n)(*[int(x) for x in tc_flops])
        self._bw = (C.c_uint64 * (n * n))(*[int(link_Bps[u][g]) for u in range(n) for g in range(n)])
        self._lat = (C.c_uint64 * (n * n))(*[int(link_lat_ps[u][g]) for u in range(n) for g in range(n)])
        self.m = K.kd_machine(n, 0, self._hbm, self._tc, self._bw, self._lat, int(launch_ps))
        self.hbm_Bps, self.tc_flops = list(hbm_Bps), list(tc_flops)
        self.link_Bps, self.link_lat_ps, self.launch_ps = link_Bps, link_lat_ps, launch_ps
        # the constants kd_place_roles reads (device 0, link 0 → 1)
        self.py = {"hbm": int(hbm_Bps[0]), "tc": int(tc_flops[0]), "bw": int(link_Bps[0][1]) if n > 1 else 1,
                   "lat": int(link_lat_ps[0][1]) if n > 1 else 0, "launch": int(launch_ps)}

    @classmethod
    def uniform(cls, n, hbm_Bps, tc_flops, link_Bps, link_lat_ps, launch_ps):
        return cls([hbm_Bps] * n, [tc_flops] * n, [[link_Bps] * n for _ in range(n)],
                   [[link_lat_ps] * n for _ in range(n)], launch_ps)


def cost(g: Graph, m: Machine) -> List[List[int]]:
    K_ = g.num_kernels
    arr = (C.c_int64 * (K_ * m.n_dev))()
    check(K.kd_cost(g.h, C.byref(m.m), arr), "kd_cost")
    return [[arr[k * m.n_dev + d] for d in range(m.n_dev)] for k in range(K_)]


def objective(g: Graph, m: Machine, assign: Sequence[int], n_micro: int, obj: int = K.KD_OBJ_AUTO):
    a = (C.c_int32 * len(assign))(*assign)
    o = C.c_int64()
    T = (C.c_int64 * m.n_dev)()
    M = (C.c_int64 * m.n_dev)()
    check(K.kd_objective(g.h, C.byref(m.m), a, n_micro, obj, C.byref(o), T, M), "kd_objective")
    return o.value, list(T), list(M)


def place(g: Graph, m: Machine, n_micro: int, obj: int = K.KD_OBJ_AUTO, max_nodes: int = 0):
    opts = K.kd_place_opts(n_micro, obj, max_nodes)
    a = (C.c_int32 * g.num_kernels)()
    o = C.c_int64()
    nodes = C.c_uint64()
    check(K.kd_place(g.h, C.byref(m.m), C.byref(opts), a, C.byref(o), C.byref(nodes)), "kd_place")
    return list(a), o.value, nodes.value


def place_roles(g: Graph, m: Machine, rows_per_micro: int, max_gpus: int = 8, micro_mask: int = 0b111):
    """kd_place_roles: the best memory/GEMM role layout per GPU count
    (1, 2, 4, 8 ≤ max_gpus). Returns a list of dicts (gpus, a, gr, n_micro,
    period_ps, T/M per role, tokens_per_step, role_mask, roles[K])."""
    K_ = g.num_kernels
    best = (K.kd_role_layout * 4)()
    roles = (C.c_int32 * (4 * K_))()
    n = C.c_uint32()
    check(K.kd_place_roles(g.h, C.byref(m.m), rows_per_micro, max_gpus, micro_mask, best, roles, 4, C.byref(n)),
          "kd_place_roles")
    out = []
    for i in range(n.value):
        b = best[i]
        out.append({"gpus": b.gpus, "a": b.a, "gr": b.gr, "n_micro": b.n_micro, "period_ps": b.period_ps,
                    "T_mem_ps": b.T_mem_ps, "T_gemm_ps": b.T_gemm_ps, "M_mem_ps": b.M_mem_ps,
                    "M_gemm_ps": b.M_gemm_ps, "tokens_per_step": b.tokens_per_step, "role_mask": b.role_mask,
                    "roles": list(roles[i * K_:(i + 1) * K_])})
    return out


class Monitor:
    """Online monitor: record finished requests, poll at any time
    for the current policy (KD_OBJ_LATENCY / KD_OBJ_THROUGHPUT)."""

    def __init__(self, window_ns: int = 300_000_000, beta=(3, 2), initial_policy: int = K.KD_OBJ_LATENCY):
        h = C.c_void_p()
        check(K.kd_monitor_create(window_ns, beta[0], beta[1], initial_policy, C.byref(h)), "kd_monitor_create")
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            K.kd_monitor_destroy(self.h)
            self.h = None

    def record(self, t_end_ns: int, req_latency_ns: int, exec_latency_ns: int):
        check(K.kd_monitor_record(self.h, t_end_ns, req_latency_ns, exec_latency_ns), "kd_monitor_record")

    def poll(self, now_ns: int):
        p, n = C.c_uint32(), C.c_uint32()
        check(K.kd_monitor_poll(self.h, now_ns, C.byref(p), C.byref(n)), "kd_monitor_poll")
        return p.value, n.value


def chunks(length: int, unit: int, n: int):
    out = (C.c_uint64 * (2 * n))()
    cnt = C.c_uint32()
    check(K.kd_chunks(length, unit, n, out, n, C.byref(cnt)), "kd_chunks")
    return [(out[2 * i], out[2 * i + 1]) for i in range(cnt.value)]


class Plan:
    def __init__(self, g: Graph, m: Machine, assign: Sequence[int], n_micro: int, n_chunks: int = 4):
        self.g, self.m = g, m
        a = (C.c_int32 * len(assign))(*assign)
        h = C.c_void_p()
        check(K.kd_plan_create(g.h, C.byref(m.m), a, n_micro, n_chunks, C.byref(h)), "kd_plan_create")
        self.h = h
        self.assign = list(assign)
        self.n_micro = n_micro
        self.n_chunks = n_chunks

    def chunks(self):
        """Chunk table: [(transfer, chunk, count_mode, row0, rows, row_bytes, unit, begin, end)]."""
        n = C.c_uint32()
        K.kd_plan_chunks(self.h, None, 0, C.byref(n))
        arr = (K.kd_chunk * max(1, n.value))()
        check(K.kd_plan_chunks(self.h, arr, n.value, C.byref(n)), "kd_plan_chunks")
        return [(c.transfer, c.chunk, c.count_mode, c.row0, c.rows, c.row_bytes, c.unit, c.begin, c.end)
                for c in arr[:n.value]]

    def __del__(self):
        if getattr(self, "h", None):
            K.kd_plan_destroy(self.h)
            self.h = None

    def schedule(self):
        n = C.c_uint32()
        K.kd_plan_schedule(self.h, None, 0, C.byref(n))
        arr = (K.kd_sched_entry * max(1, n.value))()
        check(K.kd_plan_schedule(self.h, arr, n.value, C.byref(n)), "kd_plan_schedule")
        return [(e.dev, e.micro, e.kernel, e.start_ps, e.end_ps) for e in arr[:n.value]]

    def transfers(self):
        n = C.c_uint32()
        K.kd_plan_transfers(self.h, None, 0, C.byref(n))
        arr = (K.kd_transfer * max(1, n.value))()
        check(K.kd_plan_transfers(self.h, arr, n.value, C.byref(n)), "kd_plan_transfers")
        return [(t.micro, t.producer, t.dst_dev, t.bytes, t.issue_ps, t.arrival_ps) for t in arr[:n.value]]

    @property
    def makespan(self) -> int:
        v = C.c_int64()
        check(K.kd_plan_makespan(self.h, C.byref(v)))
        return v.value

    def workspace_bytes(self, dev: int) -> int:
        v = C.c_uint64()
        check(K.kd_plan_workspace_bytes(self.h, dev, C.byref(v)), "kd_plan_workspace_bytes")
        return v.value

    def workspace_layout(self, dev: int) -> dict:
        v = K.kd_ws_layout()
        check(K.kd_plan_workspace_layout(self.h, dev, C.byref(v)), "kd_plan_workspace_layout")
        return {f: getattr(v, f) for f, _ in K.kd_ws_layout._fields_}

    def needs_binding(self, buf: int, dev: int) -> bool:
        v = C.c_int32()
        check(K.kd_plan_needs_binding(self.h, buf, dev, C.byref(v)), "kd_plan_needs_binding")
        return bool(v.value)


class Runtime:
    def __init__(self, plan: Plan, local_devs: Sequence[int], cuda_ordinals: Sequence[int]):
        self.plan = plan
        n = len(local_devs)
        h = C.c_void_p()
        check(K.kd_runtime_create(plan.h, (C.c_uint32 * n)(*local_devs), (C.c_int32 * n)(*cuda_ordinals), n,
                                  C.byref(h)), "kd_runtime_create")
        self.h = h
        self.local_devs = list(local_devs)

    def __del__(self):
        if getattr(self, "h", None):
            K.kd_runtime_destroy(self.h)
            self.h = None

    def bind(self, buf: int, micro: int, dev: int, ptr: int):
        check(K.kd_runtime_bind(self.h, buf, micro, dev, C.c_void_p(int(ptr))), "kd_runtime_bind")

    def set_workspace(self, dev: int, ptr: int, nbytes: int):
        check(K.kd_runtime_set_workspace(self.h, dev, C.c_void_p(int(ptr)), int(nbytes)), "kd_runtime_set_workspace")

    def set_peer_workspace(self, dev: int, ptr: int):
        check(K.kd_runtime_set_peer_workspace(self.h, dev, C.c_void_p(int(ptr))), "kd_runtime_set_peer_workspace")

    def set_mode(self, mode: int):
        check(K.kd_runtime_set_mode(self.h, mode), "kd_runtime_set_mode")

    def set_graph(self, enable: bool):
        check(K.kd_runtime_set_graph(self.h, 1 if enable else 0), "kd_runtime_set_graph")

    def prepare(self):
        check(K.kd_runtime_prepare(self.h), "kd_runtime_prepare")

    def set_exec(self, exec_mode: int):
        """KD_EXEC_GRAPH (per-kernel CUDA graph) or KD_EXEC_MEGAKERNEL (f1)."""
        check(K.kd_runtime_set_exec(self.h, exec_mode), "kd_runtime_set_exec")

    def exec_workspace_bytes(self, dev: int) -> int:
        n = C.c_uint64()
        check(K.kd_runtime_exec_workspace_bytes(self.h, dev, C.byref(n)), "kd_runtime_exec_workspace_bytes")
        return n.value

    def set_exec_workspace(self, dev: int, ptr: int, nbytes: int):
        check(K.kd_runtime_set_exec_workspace(self.h, dev, C.c_void_p(int(ptr)), int(nbytes)),
              "kd_runtime_set_exec_workspace")

    def exec_info(self, j: int = 0) -> dict:
        t, s, g = C.c_uint32(), C.c_uint32(), C.c_uint32()
        check(K.kd_runtime_exec_info(self.h, j, C.byref(t), C.byref(s), C.byref(g)), "kd_runtime_exec_info")
        return {"tasks": t.value, "smem_bytes": s.value, "grid": g.value}

    def step(self, streams: Sequence[int], step_id: Optional[int] = None, stats: bool = False):
        """One decode step (async). stats=True synchronises and returns
        kd_step_stats as a dict (step_ns / wait_ns / chunk_waits per local
        device, link_bytes[u][v])."""
        arr = (C.c_void_p * len(streams))(*[C.c_void_p(int(s)) for s in streams])
        sid = (1 << 64) - 1 if step_id is None else int(step_id)
        st = K.kd_step_stats() if stats else None
        check(K.kd_step(self.h, arr, sid, C.byref(st) if stats else None), "kd_step")
        if not stats:
            return None
        nl, nd = st.n_local, st.n_dev
        return {"step_id": st.step_id, "step_ns": list(st.step_ns[:nl]), "wait_ns": list(st.wait_ns[:nl]),
                "chunk_waits": list(st.chunk_waits[:nl]),
                "link_bytes": [[st.link_bytes[u * nd + v] for v in range(nd)] for u in range(nd)]
                if nd <= K.KD_STATS_MAX_DEV else None}

    def log(self):
        """KD_MODE_LOG records of the last step: [(dev, transfer, chunk, epoch, t_wait, t_acquire, t_release)]."""
        n = C.c_uint32()
        K.kd_runtime_log(self.h, None, 0, C.byref(n))
        arr = (K.kd_log_record * max(1, n.value))()
        check(K.kd_runtime_log(self.h, arr, n.value, C.byref(n)), "kd_runtime_log")
        return [(r.dev, r.transfer, r.chunk, r.epoch, r.t_wait, r.t_acquire, r.t_release) for r in arr[:n.value]]

    def check(self):
        check(K.kd_runtime_check(self.h), "kd_runtime_check")

    def launch_count(self, j: int = 0) -> int:
        n = C.c_uint32()
        check(K.kd_runtime_launch_count(self.h, j, C.byref(n)), "kd_runtime_launch_count")
        return n.value

    def profile_op(self, op: int):
        check(K.kd_runtime_profile_op(self.h, op), "kd_runtime_profile_op")

    def op_time(self):
        ms = C.c_double()
        n = C.c_uint64()
        check(K.kd_runtime_op_time(self.h, C.byref(ms), C.byref(n)), "kd_runtime_op_time")
        return ms.value, n.value


# ------------------------------------------------------------------ single ops (torch tensors → pointers)
def _p(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream):
    if stream is None:
        import torch
        stream = torch.cuda.current_stream().cuda_stream
    return C.c_void_p(int(stream))


def op_scratch_bytes(op: int, attrs) -> int:
    v = C.c_uint64()
    check(K.kd_op_scratch_bytes(op, C.byref(attrs), C.byref(v)), "kd_op_scratch_bytes")
    return v.value


def _ptr_array(ts):
    ts = [] if ts is None else (list(ts) if isinstance(ts, (list, tuple)) else [ts])
    return (C.c_void_p * max(1, len(ts)))(*[C.c_void_p(t.data_ptr()) for t in ts]), len(ts)


def add_rmsnorm(attrs, r, deltas, gamma, h, stream=None):
    """deltas: None, one tensor, or a list of tensors (attrs.n_delta must match)."""
    arr, _ = _ptr_array(deltas)
    check(K.kd_op_add_rmsnorm(C.byref(attrs), _p(r), arr, _p(gamma), _p(h), _stream(stream)), "kd_op_add_rmsnorm")


def gemm(attrs, X, W, Y, scratch, stream=None):
    check(K.kd_op_gemm(C.byref(attrs), _p(X), _p(W), _p(Y), _p(scratch), _stream(stream)), "kd_op_gemm")


def gemm_silu(attrs, X, W, out, scratch, stream=None):
    """a9+a8 fused: out [M, N/2] = silu·mul of the 64-row gate/up blocks of X·Wᵀ."""
    check(K.kd_op_gemm_silu(C.byref(attrs), _p(X), _p(W), _p(out), _p(scratch), _stream(stream)), "kd_op_gemm_silu")


def gemm_rmsnorm(attrs, X, W, r, gamma, h, scratch, stream=None):
    """a7/a10 + a3 fused: r += bf16(X·Wᵀ) (fp32, in place); h = RMSNorm(r)·gamma."""
    check(K.kd_op_gemm_rmsnorm(C.byref(attrs), _p(X), _p(W), _p(r), _p(gamma), _p(h), _p(scratch),
                               _stream(stream)), "kd_op_gemm_rmsnorm")


def qkv_rope(attrs, X, W, block_table, seq_len, q_out, k_cache, v_cache, scratch, stream=None):
    """a4+a5 fused: QKV GEMM with the RoPE + KV-append epilogue (W rows pair-interleaved per head)."""
    check(K.kd_op_qkv_rope(C.byref(attrs), _p(X), _p(W), _p(block_table), _p(seq_len), _p(q_out), _p(k_cache),
                           _p(v_cache), _p(scratch), _stream(stream)), "kd_op_qkv_rope")


def rope_append(attrs, qkv, block_table, seq_len, q_out, k_cache, v_cache, stream=None):
    check(K.kd_op_rope_append(C.byref(attrs), _p(qkv), _p(block_table), _p(seq_len), _p(q_out), _p(k_cache),
                              _p(v_cache), _stream(stream)), "kd_op_rope_append")


def attention(attrs, q, k_cache, v_cache, block_table, seq_len, out, scratch, stream=None):
    check(K.kd_op_attention(C.byref(attrs), _p(q), _p(k_cache), _p(v_cache), _p(block_table), _p(seq_len), _p(out),
                            _p(scratch), _stream(stream)), "kd_op_attention")


def silu_mul(attrs, gu, out, stream=None):
    check(K.kd_op_silu_mul(C.byref(attrs), _p(gu), _p(out), _stream(stream)), "kd_op_silu_mul")


def residual_add(attrs, r, deltas, stream=None):
    arr, _ = _ptr_array(deltas)
    check(K.kd_op_residual_add(C.byref(attrs), _p(r), arr, _stream(stream)), "kd_op_residual_add")


def rope_prefill(attrs, qkv, block_table, q_out, k_cache, v_cache, stream=None):
    """f4: RoPE at every prompt position + paged-cache fill (KD_OP_ROPE_PREFILL)."""
    check(K.kd_op_rope_prefill(C.byref(attrs), _p(qkv), _p(block_table), _p(q_out), _p(k_cache), _p(v_cache),
                               _stream(stream)), "kd_op_rope_prefill")


def prefill_attention(attrs, q, k_cache, v_cache, block_table, out, stream=None):
    """f4: causal GQA attention over the prompt (KD_OP_PREFILL_ATTENTION)."""
    check(K.kd_op_prefill_attention(C.byref(attrs), _p(q), _p(k_cache), _p(v_cache), _p(block_table), _p(out),
                                    _stream(stream)), "kd_op_prefill_attention")
