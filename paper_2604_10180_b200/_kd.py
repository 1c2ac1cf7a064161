"""ctypes binding of include/kd.h — argument marshalling only, same names.

Loading fails loudly (ImportError) if libkd.so has not been built: there is
no CPU fallback anywhere in the product path.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KD_LIB") or os.path.join(_HERE, "libkd.so")  # KD_LIB: A/B experiments

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2604_10180_b200.build` "
                      "(there is no fallback implementation)")
lib = C.CDLL(LIB_PATH)

kd_status = C.c_int32
# status codes
KD_OK, KD_ERR_INVALID_ARG, KD_ERR_RANGE, KD_ERR_STATE, KD_ERR_PIN_CONFLICT, KD_ERR_INFEASIBLE, \
    KD_ERR_UNSUPPORTED, KD_ERR_CUDA, KD_ERR_NCCL, KD_ERR_TIMEOUT, KD_ERR_OOM = range(11)
# buffer flags
KD_BUF_WEIGHT, KD_BUF_INPUT, KD_BUF_OUTPUT, KD_BUF_PERSISTENT, KD_BUF_PER_MICROBATCH = 1, 2, 4, 8, 16
KD_BUF_REPLICATED = 32
# ops
KD_OP_NONE, KD_OP_ADD_RMSNORM, KD_OP_GEMM, KD_OP_ROPE_APPEND, KD_OP_ATTENTION, KD_OP_SILU_MUL, \
    KD_OP_RESIDUAL_ADD, KD_OP_MOE_ROUTE, KD_OP_MOE_DISPATCH, KD_OP_GROUPED_GEMM, KD_OP_MOE_COMBINE, \
    KD_OP_SSM_CONV, KD_OP_SSM_UPDATE, KD_OP_GATED_NORM, KD_OP_GEMM_SILU, KD_OP_QKV_ROPE, KD_OP_ATTN_MERGE, \
    KD_OP_GEMM_RMSNORM = range(18)
KD_OP_ROPE_PREFILL, KD_OP_PREFILL_ATTENTION = 18, 19
KD_BF16, KD_F32 = 0, 1
KD_OBJ_AUTO, KD_OBJ_THROUGHPUT, KD_OBJ_LATENCY = 0, 1, 2
KD_MODE_DISAGG, KD_MODE_NO_TRANSFER, KD_MODE_LOG = 0, 1, 2
KD_EXEC_GRAPH, KD_EXEC_MEGAKERNEL = 0, 1


class KdError(RuntimeError):
    def __init__(self, status, where):
        self.status = status
        msg = lib.kd_last_error().decode()
        super().__init__(f"{where}: {lib.kd_status_str(status).decode()}: {msg}")


def check(status, where=""):
    if status != KD_OK:
        raise KdError(status, where)
    return status


class kd_span(C.Structure):
    _fields_ = [("buf", C.c_uint32), ("pad_", C.c_uint32), ("offset", C.c_uint64), ("len", C.c_uint64)]


class kd_attr_add_rmsnorm(C.Structure):
    _fields_ = [("rows", C.c_uint32), ("hidden", C.c_uint32), ("n_delta", C.c_uint32), ("dtype", C.c_uint32),
                ("eps", C.c_float), ("pad_", C.c_uint32)]


class kd_attr_gemm(C.Structure):
    _fields_ = [("M", C.c_uint32), ("N", C.c_uint32), ("K", C.c_uint32), ("dtype", C.c_uint32)]


class kd_attr_rope_append(C.Structure):
    _fields_ = [("rows", C.c_uint32), ("n_heads", C.c_uint32), ("n_kv_heads", C.c_uint32), ("head_dim", C.c_uint32),
                ("page", C.c_uint32), ("pages_per_seq", C.c_uint32), ("dtype", C.c_uint32), ("slot_offset", C.c_uint32),
                ("theta", C.c_double)]


class kd_attr_rope_prefill(C.Structure):
    _fields_ = [("seqs", C.c_uint32), ("seq_len", C.c_uint32), ("n_heads", C.c_uint32), ("n_kv_heads", C.c_uint32),
                ("head_dim", C.c_uint32), ("page", C.c_uint32), ("pages_per_seq", C.c_uint32), ("dtype", C.c_uint32),
                ("theta", C.c_double)]


class kd_attr_prefill_attention(C.Structure):
    _fields_ = [("seqs", C.c_uint32), ("seq_len", C.c_uint32), ("n_heads", C.c_uint32), ("n_kv_heads", C.c_uint32),
                ("head_dim", C.c_uint32), ("page", C.c_uint32), ("pages_per_seq", C.c_uint32), ("dtype", C.c_uint32)]


class kd_attr_attention(C.Structure):
    _fields_ = [("rows", C.c_uint32), ("n_heads", C.c_uint32), ("n_kv_heads", C.c_uint32), ("head_dim", C.c_uint32),
                ("page", C.c_uint32), ("pages_per_seq", C.c_uint32), ("dtype", C.c_uint32), ("flags", C.c_uint32)]


class kd_attr_silu_mul(C.Structure):
    _fields_ = [("rows", C.c_uint32), ("ffn", C.c_uint32), ("dtype", C.c_uint32), ("pad_", C.c_uint32)]


class kd_attr_qkv_rope(C.Structure):
    _fields_ = [("rows", C.c_uint32), ("hidden", C.c_uint32), ("n_heads", C.c_uint32), ("n_kv_heads", C.c_uint32),
                ("head_dim", C.c_uint32), ("page", C.c_uint32), ("pages_per_seq", C.c_uint32), ("dtype", C.c_uint32),
                ("theta", C.c_double)]


class kd_attr_gemm_rmsnorm(C.Structure):
    _fields_ = [("M", C.c_uint32), ("N", C.c_uint32), ("K", C.c_uint32), ("dtype", C.c_uint32),
                ("eps", C.c_float), ("flags", C.c_uint32)]


KD_NORM_DEFER = 1
KD_DNORM_HDR, KD_DNORM_PARTS = 16, 160


def KD_DNORM_BYTES(M):
    return 4 * (KD_DNORM_HDR + M * KD_DNORM_PARTS)


class kd_attr_attn_merge(C.Structure):
    _fields_ = [("rows", C.c_uint32), ("n_heads", C.c_uint32), ("head_dim", C.c_uint32), ("n_parts", C.c_uint32)]


KD_ATTN_LSE = 1


class kd_attr_residual_add(C.Structure):
    _fields_ = [("rows", C.c_uint32), ("hidden", C.c_uint32), ("n_delta", C.c_uint32), ("dtype", C.c_uint32)]


class kd_attr_moe(C.Structure):  # kd_attr_moe_route / _dispatch / _combine
    _fields_ = [("rows", C.c_uint32), ("hidden", C.c_uint32), ("experts", C.c_uint32), ("top_k", C.c_uint32)]


kd_attr_moe_route = kd_attr_moe_dispatch = kd_attr_moe


class kd_attr_grouped_gemm(C.Structure):
    _fields_ = [("rows_total", C.c_uint32), ("N", C.c_uint32), ("K", C.c_uint32), ("experts", C.c_uint32),
                ("rows_cap", C.c_uint32), ("dtype", C.c_uint32), ("expert0", C.c_uint32),
                ("meta_experts", C.c_uint32)]


class kd_attr_moe_combine(C.Structure):
    _fields_ = [("rows", C.c_uint32), ("hidden", C.c_uint32), ("experts", C.c_uint32), ("top_k", C.c_uint32),
                ("n_parts", C.c_uint32), ("pad_", C.c_uint32)]


class kd_attr_ssm(C.Structure):
    _fields_ = [("rows", C.c_uint32), ("nheads", C.c_uint32), ("head_dim", C.c_uint32), ("d_state", C.c_uint32),
                ("ngroups", C.c_uint32), ("d_conv", C.c_uint32), ("dtype", C.c_uint32), ("eps", C.c_float)]


class kd_kernel_desc(C.Structure):
    _fields_ = [("op", C.c_uint32), ("n_reads", C.c_uint32), ("n_writes", C.c_uint32), ("pin_device", C.c_int32),
                ("template_id", C.c_int32), ("pad_", C.c_uint32), ("flops", C.c_uint64),
                ("reads", C.POINTER(kd_span)), ("writes", C.POINTER(kd_span)), ("attrs", C.c_void_p),
                ("attrs_size", C.c_uint32), ("pad2_", C.c_uint32)]


class kd_edge(C.Structure):
    _fields_ = [("src", C.c_uint32), ("dst", C.c_uint32), ("buf", C.c_uint32), ("pad_", C.c_uint32),
                ("offset", C.c_uint64), ("len", C.c_uint64)]


class kd_machine(C.Structure):
    _fields_ = [("n_dev", C.c_uint32), ("pad_", C.c_uint32), ("hbm_Bps", C.POINTER(C.c_uint64)),
                ("tc_flops", C.POINTER(C.c_uint64)), ("link_Bps", C.POINTER(C.c_uint64)),
                ("link_lat_ps", C.POINTER(C.c_uint64)), ("launch_ps", C.c_uint64)]


class kd_place_opts(C.Structure):
    _fields_ = [("n_micro", C.c_uint32), ("objective", C.c_uint32), ("max_nodes", C.c_uint64)]


class kd_sched_entry(C.Structure):
    _fields_ = [("dev", C.c_uint32), ("micro", C.c_uint32), ("kernel", C.c_uint32), ("pad_", C.c_uint32),
                ("start_ps", C.c_int64), ("end_ps", C.c_int64)]


class kd_transfer(C.Structure):
    _fields_ = [("micro", C.c_uint32), ("producer", C.c_uint32), ("dst_dev", C.c_uint32), ("pad_", C.c_uint32),
                ("bytes", C.c_uint64), ("issue_ps", C.c_int64), ("arrival_ps", C.c_int64)]


class kd_chunk(C.Structure):
    _fields_ = [("transfer", C.c_uint32), ("chunk", C.c_uint32), ("count_mode", C.c_uint32), ("pad_", C.c_uint32),
                ("row0", C.c_uint64), ("rows", C.c_uint64), ("row_bytes", C.c_uint64), ("unit", C.c_uint64),
                ("begin", C.c_uint64), ("end", C.c_uint64)]


class kd_ws_layout(C.Structure):
    _fields_ = [(f, C.c_uint64) for f in ("ctrl_off", "ctrl_bytes", "flags_off", "flags_bytes", "log_off", "log_bytes",
                                          "scratch_off", "scratch_bytes", "act_off", "total")]


KD_STATS_MAX_DEV = 8


class kd_step_stats(C.Structure):
    _fields_ = [("step_id", C.c_uint64), ("n_local", C.c_uint32), ("n_dev", C.c_uint32),
                ("step_ns", C.c_uint64 * KD_STATS_MAX_DEV), ("wait_ns", C.c_uint64 * KD_STATS_MAX_DEV),
                ("chunk_waits", C.c_uint32 * KD_STATS_MAX_DEV),
                ("link_bytes", C.c_uint64 * (KD_STATS_MAX_DEV * KD_STATS_MAX_DEV))]


class kd_log_record(C.Structure):
    _fields_ = [("dev", C.c_uint32), ("transfer", C.c_uint32), ("chunk", C.c_uint32), ("pad_", C.c_uint32),
                ("epoch", C.c_uint64), ("t_wait", C.c_uint64), ("t_acquire", C.c_uint64), ("t_release", C.c_uint64)]


class kd_role_layout(C.Structure):
    _fields_ = [("gpus", C.c_uint32), ("a", C.c_uint32), ("gr", C.c_uint32), ("n_micro", C.c_uint32),
                ("period_ps", C.c_int64), ("T_mem_ps", C.c_int64), ("T_gemm_ps", C.c_int64), ("M_mem_ps", C.c_int64),
                ("M_gemm_ps", C.c_int64), ("tokens_per_step", C.c_uint64), ("role_mask", C.c_uint64)]


P = C.c_void_p
u32, i32, u64, i64 = C.c_uint32, C.c_int32, C.c_uint64, C.c_int64
PU32, PI32, PU64, PI64 = C.POINTER(u32), C.POINTER(i32), C.POINTER(u64), C.POINTER(i64)

_PROTOS = {
    "kd_status_str": (C.c_char_p, [kd_status]),
    "kd_last_error": (C.c_char_p, []),
    "kd_version": (u32, []),
    "kd_graph_create": (kd_status, [C.POINTER(P)]),
    "kd_graph_destroy": (None, [P]),
    "kd_graph_add_buffer": (kd_status, [P, u64, u32, PU32]),
    "kd_graph_add_kernel": (kd_status, [P, C.POINTER(kd_kernel_desc), PU32]),
    "kd_graph_finalize": (kd_status, [P]),
    "kd_graph_num_kernels": (kd_status, [P, PU32]),
    "kd_graph_num_buffers": (kd_status, [P, PU32]),
    "kd_graph_edges": (kd_status, [P, C.POINTER(kd_edge), u32, PU32]),
    "kd_cost": (kd_status, [P, C.POINTER(kd_machine), PI64]),
    "kd_objective": (kd_status, [P, C.POINTER(kd_machine), PI32, u32, u32, PI64, PI64, PI64]),
    "kd_place": (kd_status, [P, C.POINTER(kd_machine), C.POINTER(kd_place_opts), PI32, PI64, PU64]),
    "kd_chunks": (kd_status, [u64, u64, u32, PU64, u32, PU32]),
    "kd_place_roles": (kd_status, [P, C.POINTER(kd_machine), u32, u32, u32, C.POINTER(kd_role_layout), PI32, u32,
                                   PU32]),
    "kd_plan_create": (kd_status, [P, C.POINTER(kd_machine), PI32, u32, u32, C.POINTER(P)]),
    "kd_plan_chunks": (kd_status, [P, C.POINTER(kd_chunk), u32, PU32]),
    "kd_plan_destroy": (None, [P]),
    "kd_plan_schedule": (kd_status, [P, C.POINTER(kd_sched_entry), u32, PU32]),
    "kd_plan_transfers": (kd_status, [P, C.POINTER(kd_transfer), u32, PU32]),
    "kd_plan_makespan": (kd_status, [P, PI64]),
    "kd_plan_workspace_bytes": (kd_status, [P, u32, PU64]),
    "kd_plan_workspace_layout": (kd_status, [P, u32, C.POINTER(kd_ws_layout)]),
    "kd_plan_needs_binding": (kd_status, [P, u32, u32, PI32]),
    "kd_runtime_create": (kd_status, [P, PU32, PI32, u32, C.POINTER(P)]),
    "kd_runtime_destroy": (None, [P]),
    "kd_runtime_bind": (kd_status, [P, u32, u32, u32, P]),
    "kd_runtime_set_workspace": (kd_status, [P, u32, P, u64]),
    "kd_runtime_set_peer_workspace": (kd_status, [P, u32, P]),
    "kd_runtime_set_peer_buffer": (kd_status, [P, u32, u32, u32, P]),
    "kd_runtime_set_mode": (kd_status, [P, u32]),
    "kd_runtime_set_graph": (kd_status, [P, i32]),
    "kd_runtime_prepare": (kd_status, [P]),
    "kd_runtime_set_exec": (kd_status, [P, u32]),
    "kd_runtime_exec_workspace_bytes": (kd_status, [P, u32, PU64]),
    "kd_runtime_set_exec_workspace": (kd_status, [P, u32, P, u64]),
    "kd_runtime_exec_info": (kd_status, [P, u32, PU32, PU32, PU32]),
    "kd_step": (kd_status, [P, C.POINTER(P), u64, C.POINTER(kd_step_stats)]),
    "kd_runtime_log": (kd_status, [P, C.POINTER(kd_log_record), u32, PU32]),
    "kd_runtime_check": (kd_status, [P]),
    "kd_runtime_launch_count": (kd_status, [P, u32, PU32]),
    "kd_runtime_profile_op": (kd_status, [P, u32]),
    "kd_runtime_op_time": (kd_status, [P, C.POINTER(C.c_double), PU64]),
    "kd_ipc_get_handle": (kd_status, [P, P, PU64]),
    "kd_ipc_open": (kd_status, [P, u64, C.POINTER(P)]),
    "kd_ipc_close": (kd_status, [P]),
    "kd_debug_gemm_trace": (kd_status, [P]),
    "kd_debug_timeline": (kd_status, [P, u64]),
    "kd_debug_timeline_kinds": (kd_status, [PI32, u32, PU32]),
    "kd_debug_mega_trace": (kd_status, [P, u32, P]),
    "kd_monitor_create": (kd_status, [u64, u32, u32, u32, C.POINTER(P)]),
    "kd_monitor_destroy": (kd_status, [P]),
    "kd_monitor_record": (kd_status, [P, u64, u64, u64]),
    "kd_monitor_poll": (kd_status, [P, u64, PU32, PU32]),
    "kd_gemm_tiling": (kd_status, [u32, u32, u32, C.POINTER(C.c_int32)]),
    "kd_set_pdl": (kd_status, [i32]),
    "kd_op_scratch_bytes": (kd_status, [u32, P, PU64]),
    "kd_moe_meta_bytes": (kd_status, [u32, u32, u32, PU64]),
    "kd_op_moe_route": (kd_status, [C.POINTER(kd_attr_moe), P, P, P, P]),
    "kd_op_moe_dispatch": (kd_status, [C.POINTER(kd_attr_moe), P, P, P, P, P]),
    "kd_op_grouped_gemm": (kd_status, [C.POINTER(kd_attr_grouped_gemm), P, P, P, P, P, P]),
    "kd_op_moe_combine": (kd_status, [C.POINTER(kd_attr_moe_combine), P, P, P, P, P]),
    "kd_op_ssm_conv": (kd_status, [C.POINTER(kd_attr_ssm), P, P, P, P, P, P]),
    "kd_op_ssm_update": (kd_status, [C.POINTER(kd_attr_ssm), P, P, P, P, P, P, P, P]),
    "kd_op_gated_norm": (kd_status, [C.POINTER(kd_attr_ssm), P, P, P, P, P]),
    "kd_op_add_rmsnorm": (kd_status, [C.POINTER(kd_attr_add_rmsnorm), P, P, P, P, P]),
    "kd_op_gemm": (kd_status, [C.POINTER(kd_attr_gemm), P, P, P, P, P]),
    "kd_op_gemm_silu": (kd_status, [C.POINTER(kd_attr_gemm), P, P, P, P, P]),
    "kd_op_gemm_rmsnorm": (kd_status, [C.POINTER(kd_attr_gemm_rmsnorm), P, P, P, P, P, P, P]),
    "kd_op_attn_merge": (kd_status, [C.POINTER(kd_attr_attn_merge), P, P, P]),
    "kd_op_qkv_rope": (kd_status, [C.POINTER(kd_attr_qkv_rope), P, P, P, P, P, P, P, P, P]),
    "kd_op_rope_append": (kd_status, [C.POINTER(kd_attr_rope_append), P, P, P, P, P, P, P]),
    "kd_op_attention": (kd_status, [C.POINTER(kd_attr_attention), P, P, P, P, P, P, P, P]),
    "kd_op_silu_mul": (kd_status, [C.POINTER(kd_attr_silu_mul), P, P, P]),
    "kd_op_rope_prefill": (kd_status, [C.POINTER(kd_attr_rope_prefill), P, P, P, P, P, P]),
    "kd_op_prefill_attention": (kd_status, [C.POINTER(kd_attr_prefill_attention), P, P, P, P, P, P]),
    "kd_op_residual_add": (kd_status, [C.POINTER(kd_attr_residual_add), P, P, P]),
}

EXPORTED = sorted(_PROTOS)

for _name, (_res, _args) in _PROTOS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args
    globals()[_name] = _f
