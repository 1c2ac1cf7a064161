#!/usr/bin/env python3
"""bench.py — decode tokens/s of the kernel-disaggregation hot path on B200.

Contract (task statement):
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
A "step" = one full L-layer decode step (every §8(a) kernel) over one batch.
N=1 workload: BASELINE.json configs[1], Llama-3-8B-shaped decode, B=64,
C=4096, L=32, bf16, monolithic on one B200 (1-GPU reference point of the
metric). N>1 (torchrun, one process per GPU): disaggregated replicas of the
same workload per rank group — see DESIGN.md §Multi-GPU.
Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode_tokens_per_s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=60)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="llama3-8b")
    p.add_argument("--layers", type=int, default=0, help="override L (default: the config's)")
    p.add_argument("--batch", type=int, default=0)
    p.add_argument("--no-graph", action="store_true")
    p.add_argument("--kernels", action="store_true", help="also time every op kind (extra passes)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--exec", dest="exec_mode", default="graph", choices=["graph", "mega"],
                   help="N=1: per-kernel CUDA graph (default) or the f1 megakernel (one launch per step)")
    p.add_argument("--layout", default="search", choices=["search", "pairs"],
                   help="N>1: the role layout kd_place_roles picks (default) or independent 1:1 pairs")
    return p.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d["hbm_gbs"], d["bf16_tflops"], d.get("bf16_tflops_sustained"), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.lines = []
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                       "-lms", "50", "-i", str(gpu_index)], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.p = None

    def _read(self):
        for line in self.p.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(2)
        except Exception:
            self.p.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- CPU baseline (the oracle)
def _oracle_cores():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        return os.cpu_count()


def cpu_baseline(cfg, full_batch=True):
    """Times the oracle as it stands (fp64 numpy) on the host cores: one
    full-width layer of the workload at its FULL batch B (every kernel of the
    layer, all B sequences at context C), extrapolated × L layers; tokens/s =
    B / (L · t_layer). Also a 1-thread figure on a 2-sequence sample
    (BASELINE.md §3). Input generation is outside the timed region."""
    import numpy as np  # noqa: F401
    import synth
    from oracle import layer as OL
    cores = _oracle_cores()
    B = cfg.batch if full_batch else 2
    sub = cfg.with_(n_layers=1, batch=B, n_micro=1)
    inp = synth.make_decoder_inputs(sub)
    t0 = time.perf_counter()
    OL.decoder_step(inp, act="bf16")
    t = time.perf_counter() - t0
    value = B / (cfg.n_layers * t)
    out = {"value": value, "unit": "tokens/s", "cores": cores, "kind": "oracle",
           "sample": f"{B} sequences x 1 full-width layer of {cfg.name} (C={cfg.context}), fp64 numpy oracle on "
                     f"{cores} BLAS threads, 1 rep ({t:.1f} s), extrapolated x{cfg.n_layers} layers",
           "host_cpus": os.cpu_count()}
    try:
        from threadpoolctl import threadpool_limits
        sub2 = cfg.with_(n_layers=1, batch=2, n_micro=1)
        inp2 = synth.make_decoder_inputs(sub2)
        with threadpool_limits(1):
            t0 = time.perf_counter()
            OL.decoder_step(inp2, act="bf16")
            t1 = time.perf_counter() - t0
        out["one_thread"] = {"value": 2 / (cfg.n_layers * t1), "unit": "tokens/s",
                             "sample": f"2 sequences x 1 layer, 1 thread ({t1:.1f} s), extrapolated x{cfg.n_layers}"}
    except Exception as ex:  # report, do not hide
        out["one_thread"] = {"error": str(ex)}
    return out


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # the reference arm is the oracle (PAPER.md has no code to install): each
    # step = one full-width layer of the workload for a bounded 2-sequence
    # sample, timed W + K times on the host cores, extrapolated × L layers
    import synth
    from oracle import layer as OL
    steps, warm = args.steps, args.warmup
    inp = synth.make_decoder_inputs(cfg.with_(n_layers=1, batch=2, n_micro=1))
    for _ in range(warm):
        OL.decoder_step(inp, act="bf16")
    t0 = time.perf_counter()
    for _ in range(steps):
        OL.decoder_step(inp, act="bf16")
    t = (time.perf_counter() - t0) / max(steps, 1)
    cores = _oracle_cores()
    base = {"value": 2 / (cfg.n_layers * t), "unit": "tokens/s", "cores": cores, "kind": "oracle",
            "sample": f"2 sequences x 1 full-width layer of {cfg.name} (C={cfg.context}) per step, fp64 numpy oracle on "
                      f"{cores} BLAS threads, {steps} timed steps after {warm} warm-up, extrapolated x{cfg.n_layers} layers"}
    line = {"impl": "reference", "metric": METRIC, "value": base["value"], "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": steps, "warmup": warm, "ms_per_step": round(t * cfg.n_layers * 1e3, 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_config(cfg, 1, "oracle (CPU)"),
            "cpu_baseline": base,
            "e2e": {"value": base["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def placement_search(cfg, DEC):
    """a1 on the host ("report search time", "solves
    each DDG in about 20 ms"): the device-role search kd_place_roles over one
    memory shard's unfused step graph (m = 32 rows per micro-batch, the 8B
    pair's micro-batch) — the best memory:GEMM ratio and N per GPU count with
    its modelled tokens/s per GPU — and kd_place's kernel-level search on the
    2-device pair; wall time of each exact search."""
    from paper_2604_10180_b200.api import place, place_roles
    if cfg.n_experts or cfg.attn_every:
        return None
    m = 32
    dg = DEC.DecoderGraph(cfg.with_(batch=m, n_micro=1))
    out = {"kernels": dg.g.num_kernels, "rows_per_micro": m, "model": "kd_place_roles (E6 over role layouts)"}
    t0 = time.perf_counter()
    lays = place_roles(dg.g, DEC.b200_machine(8), m, 8, 0b111)
    out["roles_search_ms"] = round((time.perf_counter() - t0) * 1e3, 2)
    for L in lays:
        tok_s = L["tokens_per_step"] / (L["period_ps"] * 1e-12)
        out[f"{L['gpus']}gpu"] = {"memory_gpus": L["a"], "gemm_gpus": L["gr"], "n_micro": L["n_micro"],
                                  "period_us": round(L["period_ps"] / 1e6, 1),
                                  "model_tokens_per_s_per_gpu": round(tok_s / L["gpus"], 1),
                                  "T_mem_us": round(L["T_mem_ps"] / 1e6, 1), "T_gemm_us": round(L["T_gemm_ps"] / 1e6, 1)}
    dg2 = DEC.DecoderGraph(cfg.with_(n_micro=2))
    t0 = time.perf_counter()
    a, obj, nodes = place(dg2.g, DEC.b200_machine(2), 2)
    out["pair_kernel_search"] = {"search_ms": round((time.perf_counter() - t0) * 1e3, 2),
                                 "objective_us": round(obj / 1e6, 1), "nodes": nodes, "devices_used": len(set(a))}
    return out


def role_layout(cfg, DEC, n_gpus):
    """(a, N) of kd_place_roles' best layout on n_gpus (8B shard, m = 32)."""
    from paper_2604_10180_b200.api import place_roles
    dg = DEC.DecoderGraph(cfg.with_(batch=32, n_micro=1))
    for L in place_roles(dg.g, DEC.b200_machine(8), 32, 8, 0b110):  # N ∈ {2, 4}
        if L["gpus"] == n_gpus:
            return L["a"], L["n_micro"]
    return n_gpus - 1, 2


def step_bytes(cfg):
    """Algorithmic HBM bytes of one monolithic decode step (dense attention
    layers, N=1) as the f1 megakernel runs it (QKV+RoPE and gate_up+SiLU
    fused, norms separate): every weight, every KV page, each remaining
    activation written once and read once, the fp32 residual read and
    written by each add."""
    m, H, F, L = cfg.batch, cfg.hidden, cfg.ffn, cfg.n_layers
    Hq, Hkv, D, pps = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim, cfg.pages_per_seq
    qkv = (Hq + 2 * Hkv) * D
    w = (qkv * H + H * Hq * D + 2 * F * H + H * F + 2 * H) * 2
    kv = m * pps * Hkv * 16 * D * 2 * 2 + m * pps * 4 + m * 4
    norm = m * H * (4 + 4 + 2 + 2)                  # r read + write, delta read, h write
    act = (m * H * 2                               # QKV reads h1
           + m * Hq * D * 2 * 2 + 2 * m * Hkv * D * 2  # q written + read by attention, K/V slot appends
           + m * Hq * D * 2 * 2                    # attention out, O reads it
           + m * H * 2 + m * H * 2                 # O out (read by norm2), gate_up reads h2
           + m * F * 2 * 2                         # a written by the gate_up fold, read by down
           + m * H * 2)                            # down out (read by the next norm)
    return L * (w + kv + 2 * norm + act) + m * H * (4 + 4 + 2)  # + the final residual add


def workload_config(cfg, n_gpus, placement):
    return {"workload": f"{cfg.name} decode B={cfg.batch} C={cfg.context} L={cfg.n_layers}",
            "model_shape": {"hidden": cfg.hidden, "heads": cfg.n_heads, "kv_heads": cfg.n_kv_heads,
                            "head_dim": cfg.head_dim, "ffn": cfg.ffn, "layers": cfg.n_layers},
            "batch": cfg.batch, "context": cfg.context, "n_micro": cfg.n_micro, "placement": placement,
            "n_gpus": n_gpus,
            "l2": "inputs larger than L2 (per step: KV cache + weights >> 126 MB), no flush needed"}


# ---------------------------------------------------------------- our arm
def main():
    args = parse()
    import synth
    cfg = synth.CONFIGS[args.config]
    if args.layers:
        cfg = cfg.with_(n_layers=args.layers)
    if args.batch:
        cfg = cfg.with_(batch=args.batch)
    cfg = cfg.with_(n_micro=1)
    if args.impl == "reference":
        run_reference(args, cfg)
        return
    import torch
    import numpy as np
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    # test hooks: exercise the N>1 code path on a 1-GPU box (all ranks on cuda:0,
    # gloo process group); never set by the driver
    if os.environ.get("KD_BENCH_ONE_GPU"):
        local = 0
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        if os.environ.get("KD_BENCH_ONE_GPU"):
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    from paper_2604_10180_b200 import decoder as DEC, _kd as K

    hbm_gbs, tc_tflops, tc_sus, peak_src = peaks()
    if world == 1:
        # 1 GPU: the monolithic reference point of the metric (all kernels on one B200);
        # gate_up and SiLU·mul share the device, so they are declared as one fused kernel
        # (KD_OP_GEMM_SILU, bit-identical to the pair); so are QKV + RoPE/append
        # (KD_OP_QKV_ROPE, bit-identical to the pair: 17.0 vs 15.0 + 3.7 µs, step 9.04 vs
        # 9.13 ms) and the O GEMM with norm2 / the down GEMM with the next layer's norm1
        # (KD_OP_GEMM_RMSNORM), with the RMSNorm's per-token 1/rms deferred to the
        # consumers (KD_NORM_DEFER: gate_up+SiLU and QKV+RoPE scale their fp32 sums; no
        # grid barrier in the O / down epilogues: 8.73 vs 8.84 ms same box). A/B:
        # KD_BENCH_NO_FUSE (all), KD_BENCH_NO_FUSE_ROPE, KD_BENCH_NO_FUSE_NORM,
        # KD_BENCH_FUSE_NORM=o (O+norm2 only), KD_BENCH_FUSE_NORM=1 (norm in the GEMM epilogue
        # after an in-kernel grid barrier).
        mega = args.exec_mode == "mega"
        fuse = not os.environ.get("KD_BENCH_NO_FUSE")
        # (the megakernel has no GEMM + RMSNorm task: the norms stay separate tasks)
        dg = DEC.DecoderGraph(cfg, fuse_silu=fuse, fuse_rope=fuse and not os.environ.get("KD_BENCH_NO_FUSE_ROPE"),
                              fuse_norm=(fuse and not mega and not os.environ.get("KD_BENCH_NO_FUSE_NORM")) and
                              (os.environ.get("KD_BENCH_FUSE_NORM") or "defer"))
        assign = [0] * dg.g.num_kernels
        rt = DEC.DecoderRuntime(dg, assign, 1, [local], seed=cfg.seed, use_graph=not args.no_graph, megakernel=mega)
        placement = "monolithic (all kernels on one B200)" + (
            ", f1 megakernel: the graph's 7 ops/layer (QKV+RoPE and gate_up+SiLU fused) as tasks of ONE persistent "
            "launch per step" if mega else "")
    elif cfg.name == "llama3-70b":
        # BASELINE config 3: GEMMs TP-sharded over N/2 GPUs, attention partners on the
        # other N/2 (head-sharded); row-parallel partials streamed to every partner by
        # the GEMM epilogue and reduced in the partners' norms (fused all-reduce, a14)
        T = world // 2
        cfg = cfg.with_(n_micro=2)
        dg = DEC.TPDecoderGraph(cfg, T)
        rt = DEC.DecoderRuntime(dg, dg.assign(), 2 * T, [local], seed=cfg.seed, use_graph=not args.no_graph,
                                local_devs=[rank], dist=dist)
        placement = (f"TP={T}: GEMM ranks {T}..{2 * T - 1}, attention partners 0..{T - 1} (head-sharded), "
                     f"fused peer-store all-reduce, N=2 micro-batches")
    elif cfg.n_experts:
        # BASELINE config 4 ("router/attention kernels disaggregated from expert
        # GEMMs over 8 GPUs"): N/2 attention/router shards, each
        # decoding B/(N/2) of the B sequences (norms, QKV/O GEMMs, RoPE/append,
        # attention, router, dispatch, combine), and N/2 expert ranks owning
        # E/(N/2) experts each (grouped gate_up, SiLU, grouped down); dispatch
        # and combine are P2P (expert parallelism), N=2 micro-batches
        if world % 2:
            raise SystemExit("bench.py: the MoE expert-parallel layout needs an even --gpus")
        a = e = world // 2
        if cfg.n_experts % e:
            raise SystemExit(f"bench.py: {cfg.n_experts} experts do not split over {e} expert ranks")
        shard = cfg.with_(batch=max(2, cfg.batch // a), n_micro=2)
        dg = DEC.MoEEPDecoderGraph(shard, a, e)
        rt = DEC.DecoderRuntime(dg, dg.assign(), a + e, [local], seed=cfg.seed, use_graph=not args.no_graph,
                                local_devs=[rank], dist=dist)
        placement = (f"MoE expert parallel {a}+{e}: ranks 0..{a - 1} attention/router shards ({shard.batch} "
                     f"sequences each), ranks {a}..{world - 1} own {cfg.n_experts // e} experts each; P2P "
                     f"dispatch/combine, chunked handoff, N=2 micro-batches")
        cfg = shard
        tokens_per_step = shard.batch * a
    else:
        # N GPUs: N/2 independent disaggregated pairs (BASELINE config 2: memory-bound
        # kernels on the even rank, GEMMs on the odd rank), each decoding its own batch
        # of B sequences with 2 micro-batches; cut edges are streamed by the producers'
        # fused peer stores into the partner's HBM (CUDA IPC over NVLink). No collective.
        if args.layout == "pairs" or cfg.attn_every:  # (the role-layout graph has no SSM layers)
            if world % 2:
                raise SystemExit("bench.py: --layout pairs needs an even --gpus")
            pair, role = rank // 2, rank % 2
            groups = [dist.new_group([2 * p, 2 * p + 1]) for p in range(world // 2)]
            cfg = cfg.with_(n_micro=2)
            dg = DEC.DecoderGraph(cfg)
            assign = dg.role_assign(0, 1)
            rt = DEC.DecoderRuntime(dg, assign, 2, [local], seed=cfg.seed + pair, use_graph=not args.no_graph,
                                    local_devs=[role], dist=dist, dist_group=groups[pair])
            placement = (f"{world // 2} disaggregated pair(s): memory-role kernels (norms, RoPE+append, attention, "
                         f"SiLU) on even ranks, GEMMs on odd ranks, N=2 micro-batches")
            tokens_per_step = cfg.batch * (world // 2)
        else:
            # the layout kd_place_roles picks for this GPU count:
            # a memory-role ranks (0..a-1), each decoding its own B sequences, and
            # world − a GEMM ranks; with one GEMM rank (a:1) every GEMM runs once
            # per micro-batch over all a·m rows (bipartite gather/scatter)
            a, N = role_layout(cfg, DEC, world)
            if world - a != 1:
                raise SystemExit(f"bench.py: the searched layout {a}:{world - a} needs TP GEMM ranks (use --layout pairs)")
            shard = cfg.with_(n_micro=N)
            if shard.m * a > 256:
                shard = shard.with_(batch=N * (256 // a))
            dg = DEC.RoleDecoderGraph(shard, a)
            rt = DEC.DecoderRuntime(dg, dg.assign(), a + 1, [local], seed=cfg.seed, use_graph=not args.no_graph,
                                    local_devs=[rank], dist=dist)
            cfg = shard
            placement = (f"searched role layout {a}:1 (kd_place_roles): ranks 0..{a - 1} memory role (norms, "
                         f"RoPE+append, attention, SiLU; {shard.batch} sequences each), rank {a} the GEMMs over "
                         f"{a}x{shard.m} rows per micro-batch, N={N} micro-batches, chunked P2P handoff")
            tokens_per_step = shard.batch * a
    stream = rt.streams[0]

    def barrier():
        if dist is not None:
            dist.barrier()

    for _ in range(args.warmup):
        rt.step()
    torch.cuda.synchronize()
    n_launch = rt.rt.launch_count(0)

    # ---- timed region (device resident inputs)
    clocks = ClockSampler(local)
    time.sleep(0.15)
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        rt.step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1)
    clk = clocks.stop()
    rt.rt.check()
    # exposed transfer (N>1): same plan and schedule with the peer stores and
    # flag waits removed (KD_MODE_NO_TRANSFER; consumers read their landing
    # slots as left by the previous steps) — exposed = T(DISAGG) − T(NO_TRANSFER)
    exposed = None
    if world > 1:
        rt.rt.set_mode(K.KD_MODE_NO_TRANSFER)
        rt.rt.prepare()
        for _ in range(2):
            rt.step()
        torch.cuda.synchronize()
        barrier()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.steps):
            rt.step()
        f1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ms_nt = f0.elapsed_time(f1)
        if dist is not None:
            t = torch.tensor([ms_nt], device="cpu" if os.environ.get("KD_BENCH_ONE_GPU") else "cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_nt = float(t.item())
        exposed = {"ms_per_step": round(ms / args.steps - ms_nt / args.steps, 4),
                   "no_transfer_ms_per_step": round(ms_nt / args.steps, 4),
                   "fraction_of_step": round(1 - ms_nt / ms, 4)}
        # and as the consumers saw it: KD_MODE_LOG per-chunk records, kd_step_stats
        # wait_ns = Σ over this rank's incoming chunks of the first acquirer's stall
        rt.rt.set_mode(K.KD_MODE_LOG)
        rt.rt.prepare()
        for _ in range(2):
            rt.step()
        barrier()
        st = rt.step(stats=True)
        exposed["log_wait_us_per_step_rank0"] = round(st["wait_ns"][0] / 1e3, 2)
        exposed["log_step_us_rank0"] = round(st["step_ns"][0] / 1e3, 2)
        exposed["log_chunk_waits_rank0"] = st["chunk_waits"][0]
        exposed["link_bytes_per_step_from_rank0"] = sum(st["link_bytes"][rt.local_devs[0]]) if st["link_bytes"] else None
        barrier()
        rt.rt.set_mode(K.KD_MODE_DISAGG)
        rt.rt.prepare()
    # per-kernel CUDA-event timing: a second pass of the same K steps whose
    # graph carries event-record nodes around every attention launch, on a
    # side branch so the kernel keeps its PDL edges (kept out of the headline)
    mega = world == 1 and args.exec_mode == "mega"
    attn_ms, attn_n = 0.0, 0
    if not mega:
        rt.rt.profile_op(K.KD_OP_ATTENTION)
        rt.rt.prepare()
        for _ in range(2):
            rt.step()
        torch.cuda.synchronize()
        attn_ms_tot, attn_n_tot = 0.0, 0
        for _ in range(args.steps):
            rt.step()
            torch.cuda.synchronize()
            t_ms, t_n = rt.rt.op_time()
            attn_ms_tot += t_ms
            attn_n_tot += t_n
        attn_ms, attn_n = attn_ms_tot / args.steps, attn_n_tot // args.steps
        rt.rt.profile_op(0)
        rt.rt.prepare()
    if dist is not None:
        t = torch.tensor([ms], device="cpu" if os.environ.get("KD_BENCH_ONE_GPU") else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    if world == 1 or cfg.name == "llama3-70b":
        tokens_per_step = cfg.batch
    value = tokens_per_step / (ms_step / 1e3)

    # ---- roofline of the dominant kernel (decode attention)
    m, C, Hkv, D, Hq = cfg.m, cfg.context, cfg.n_kv_heads, cfg.head_dim, cfg.n_heads
    pps = cfg.pages_per_seq
    attn_bytes = (m * pps * Hkv * 16 * D * 2 * 2      # K and V pools (every page of every sequence)
                  + 2 * m * Hq * D * 2                 # q in, out
                  + m * pps * 4 + m * 4)               # block table, seq_len
    avg_attn_s = (attn_ms / max(attn_n, 1)) / 1e3
    achieved = attn_bytes / avg_attn_s / 1e9 if attn_n else 0.0
    roof = {"kernel": "decode_attention_kernel<128>", "bound": "hbm", "achieved": round(achieved, 1),
            "peak": hbm_gbs, "unit": "GB/s", "frac": round(achieved / hbm_gbs, 4), "traffic": None,
            "bytes_per_launch": attn_bytes, "avg_launch_us": round(avg_attn_s * 1e6, 2),
            "launches_per_step": attn_n, "steps_profiled": args.steps,
            "share_of_step": round(attn_ms / ms_step, 4) if ms_step else None,
            "peak_source": peak_src,
            "timing": "CUDA events around every attention launch, averaged over K profiled steps run right after "
                      "the timed region; the event-record nodes hang off a side branch of the captured step graph "
                      "(ev0 completes with the kernel before attention, ev1 with attention), so the attention "
                      "launch keeps its programmatic (PDL) edges as in the timed steps"}
    if mega:
        # the megakernel is the step's only kernel: its algorithmic bytes are the
        # whole step's (KV cache, weights, activations), its
        # duration the timed step's (CUDA events on its stream)
        sb = step_bytes(cfg)
        achieved = sb / (ms_step / 1e3) / 1e9
        roof = {"kernel": f"mega_kernel<{D}> (f1: the whole step, one launch)", "bound": "hbm",
                "achieved": round(achieved, 1), "peak": hbm_gbs, "unit": "GB/s", "frac": round(achieved / hbm_gbs, 4),
                "traffic": None, "bytes_per_launch": sb, "avg_launch_us": round(ms_step * 1e3, 2),
                "launches_per_step": 1, "share_of_step": 1.0, "peak_source": peak_src,
                "timing": "CUDA events on the launching stream around the K timed steps (one launch each)"}
    tr_path = os.path.join(ROOT, "profiles", "mega_traffic.json" if mega else "attention_traffic.json")
    if mega and os.path.exists(tr_path):
        try:
            sys.path.insert(0, os.path.join(ROOT, "scripts"))
            from attention_traffic import source_sha256, MEGA_SOURCES
            tr = json.load(open(tr_path))
            if (tr.get("algorithmic_bytes_per_launch") == roof["bytes_per_launch"]
                    and tr.get("source_sha256") == source_sha256(MEGA_SOURCES)):
                roof["traffic"] = tr.get("bytes_per_launch")
                roof["traffic_source"] = tr.get("source")
        except Exception:
            pass
    elif os.path.exists(tr_path):
        # ncu dram bytes of the same launch shape (profiles/), ONLY if captured
        # from the kernel sources this build compiled (sha256 stamp), else null
        try:
            sys.path.insert(0, os.path.join(ROOT, "scripts"))
            from attention_traffic import source_sha256
            tr = json.load(open(tr_path))
            if tr.get("algorithmic_bytes_per_launch") == attn_bytes and tr.get("source_sha256") == source_sha256():
                roof["traffic"] = tr.get("bytes_per_launch")
                roof["traffic_source"] = tr.get("source")
        except Exception:
            pass

    # ---- e2e: host buffers, H2D of the step inputs and D2H of the result inside the region
    h2d = d2h = 0
    e2e_value = None
    try:
        me = rt.local_devs[0]
        def mine(base, dt):  # this rank's instance of r / bt / sl (suffixed per shard in the role graphs)
            for (nm, i, d), t in rt.tensors.items():
                if d == me and i == 0 and (nm == base or nm.startswith(base + ".")):
                    return t
            return torch.zeros(1, dtype=dt, device="cuda")  # GEMM-role rank: its inputs arrive from the peers
        r_dev = mine("r", torch.float32)
        bt_dev = mine("bt", torch.int32)
        sl_dev = mine("sl", torch.int32)
        r_host = torch.empty_like(r_dev, device="cpu").pin_memory()
        r_host.copy_(r_dev)
        bt_host = bt_dev.cpu().pin_memory()
        sl_host = sl_dev.cpu().pin_memory()
        out_host = torch.empty_like(r_host).pin_memory()
        h2d = r_host.numel() * 4 + bt_host.numel() * 4 + sl_host.numel() * 4
        d2h = out_host.numel() * 4
        n_e2e = max(5, args.steps // 2)
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        with torch.cuda.stream(stream):
            for _ in range(n_e2e):
                r_dev.copy_(r_host, non_blocking=True)
                bt_dev.copy_(bt_host, non_blocking=True)
                sl_dev.copy_(sl_host, non_blocking=True)
                rt.step()
                out_host.copy_(r_dev, non_blocking=True)
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        if dist is not None:
            t = torch.tensor([el], device="cpu" if os.environ.get("KD_BENCH_ONE_GPU") else "cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        e2e_value = tokens_per_step * n_e2e / el
    except Exception as ex:  # report, do not hide
        e2e_value = None
        print(f"e2e failed: {ex}", file=sys.stderr)

    kernels = None
    if args.kernels:
        kernels = {}
        for op, nm in ((K.KD_OP_GEMM, "gemm"), (K.KD_OP_GEMM_SILU, "gemm_silu"), (K.KD_OP_QKV_ROPE, "qkv_rope"),
                       (K.KD_OP_GEMM_RMSNORM, "gemm_rmsnorm"),
                       (K.KD_OP_ADD_RMSNORM, "add_rmsnorm"),
                       (K.KD_OP_ROPE_APPEND, "rope_append"), (K.KD_OP_SILU_MUL, "silu_mul")):
            rt.rt.profile_op(op)
            rt.rt.prepare()
            for _ in range(3):
                rt.step()
            torch.cuda.synchronize()
            t_ms, n = rt.rt.op_time()
            kernels[nm] = {"ms_per_step": round(t_ms, 4), "launches": n}

    line = {"metric": METRIC, "value": round(value, 1), "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded random-init weights, KV cache and residual inputs on device)",
            "config": workload_config(cfg, world, placement),
            "roofline": roof,
            "e2e": {"value": round(e2e_value, 1) if e2e_value else None, "unit": "tokens/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": n_launch * args.steps,
            "exposed_transfer": exposed,
            "clocks": clk}
    if kernels:
        line["kernels"] = kernels
    if rank == 0:
        line["placement_search"] = placement_search(cfg, DEC)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
