#!/usr/bin/env python3
"""f4 measurement: the prefill kernels and a full prefill step on one B200.

Per kernel (CUDA graph of 10 launches, CUDA events, after warm-up): the large-M
tcgen05 GEMM at the 8B prefill shapes (M = B·S tokens) in TFLOP/s against the
measured bf16 peak (MEASURED_PEAKS.json; torch.matmul = cuBLAS at the same
shape printed beside it as context), the causal prefill attention in TFLOP/s
(causal FLOPs: 2·D·S·(S+1) per (sequence, head) for QKᵀ and PV), RoPE + cache
fill in GB/s. Then the whole PrefillGraph step through kd_step: prompt
tokens/s and each op kind's share of the step.

    python scripts/bench_prefill.py [--layers 32] [--batch 8] [--seq 1024]
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2604_10180_b200 import _kd as K, api, decoder as DEC  # noqa: E402
import synth  # noqa: E402


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d["bf16_tflops"], d["hbm_gbs"]
    return 1590.0, 6650.0


def timeit(fn, iters=10, warm=3):
    s = torch.cuda.Stream()
    torch.cuda.synchronize()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(warm):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(iters):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record()
        g.replay()
        e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3  # µs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--seq", type=int, default=1024)
    ap.add_argument("--kernels-only", action="store_true")
    a = ap.parse_args()
    tf_peak, hbm = peaks()
    cfg = synth.LLAMA8B.with_(batch=a.batch, n_layers=a.layers, context=a.seq)
    B, S, H, F = a.batch, a.seq, cfg.hidden, cfg.ffn
    Hq, Hkv, D = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
    M = B * S
    out = {"config": f"llama3-8b prefill B={B} S={S} (M={M} tokens)", "bf16_peak_tflops": tf_peak,
           "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst)", "kernels": []}
    # ---- GEMMs
    for name, N, Kd in (("qkv", cfg.qkv_dim, H), ("o", H, Hq * D), ("gate_up", 2 * F, H), ("down", H, F)):
        X = torch.randn(M, Kd, device="cuda").to(torch.bfloat16)
        W = (torch.randn(N, Kd, device="cuda") / math.sqrt(Kd)).to(torch.bfloat16)
        Y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        at = K.kd_attr_gemm(M, N, Kd, K.KD_BF16)
        scr = torch.zeros(256, dtype=torch.uint8, device="cuda")
        us = timeit(lambda: api.gemm(at, X, W, Y, scr))
        us_cublas = timeit(lambda: torch.matmul(X, W.t(), out=Y))
        fl = 2.0 * M * N * Kd
        out["kernels"].append({"kernel": f"gemm_{name}", "M": M, "N": N, "K": Kd, "us": round(us, 1),
                               "tflops": round(fl / us / 1e6, 1), "frac": round(fl / us / 1e6 / tf_peak, 3),
                               "cublas_us": round(us_cublas, 1), "cublas_tflops": round(fl / us_cublas / 1e6, 1)})
        print(json.dumps(out["kernels"][-1]), flush=True)
        del X, W, Y
    # ---- attention
    pps = (S + 15) // 16
    kc = torch.randn(B * pps, Hkv, 16, D, device="cuda").to(torch.bfloat16)
    vc = torch.randn(B * pps, Hkv, 16, D, device="cuda").to(torch.bfloat16)
    bt = torch.randperm(B * pps, device="cuda").to(torch.int32).view(B, pps)
    q = torch.randn(M, Hq * D, device="cuda").to(torch.bfloat16)
    o = torch.empty_like(q)
    aa = K.kd_attr_prefill_attention(B, S, Hq, Hkv, D, 16, pps, K.KD_BF16)
    us = timeit(lambda: api.prefill_attention(aa, q, kc, vc, bt, o))
    fl = 2.0 * D * S * (S + 1) * B * Hq
    out["kernels"].append({"kernel": "prefill_attention", "B": B, "S": S, "heads": f"{Hq}/{Hkv}", "D": D,
                           "us": round(us, 1), "tflops": round(fl / us / 1e6, 1),
                           "frac": round(fl / us / 1e6 / tf_peak, 3)})
    print(json.dumps(out["kernels"][-1]), flush=True)
    # ---- RoPE + cache fill
    qkv = torch.randn(M, cfg.qkv_dim, device="cuda").to(torch.bfloat16)
    ra = K.kd_attr_rope_prefill(B, S, Hq, Hkv, D, 16, pps, K.KD_BF16, 5e5)
    us = timeit(lambda: api.rope_prefill(ra, qkv, bt, q, kc, vc))
    by = M * cfg.qkv_dim * 2 + M * Hq * D * 2 + 2 * M * Hkv * D * 2
    out["kernels"].append({"kernel": "rope_prefill", "us": round(us, 1), "GBps": round(by / us / 1e3, 1),
                           "frac_hbm": round(by / us / 1e3 / hbm, 3)})
    print(json.dumps(out["kernels"][-1]), flush=True)
    del kc, vc, q, o, qkv
    torch.cuda.empty_cache()
    if a.kernels_only:
        return
    # ---- the whole prefill step through kd_step
    pg = DEC.PrefillGraph(cfg, S)
    rt = DEC.DecoderRuntime(pg, [0] * pg.g.num_kernels, 1, [0], seed=cfg.seed)
    for _ in range(2):
        rt.step()
    torch.cuda.synchronize()
    steps = 5
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(rt.streams[0])
    for _ in range(steps):
        rt.step()
    e1.record(rt.streams[0])
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    rt.rt.check()
    flops = sum(2.0 * M * n * k for n, k in ((cfg.qkv_dim, H), (H, Hq * D), (2 * F, H), (H, F))) * cfg.n_layers \
        + 2.0 * D * S * (S + 1) * B * Hq * cfg.n_layers
    shares = {}
    for op, nm in ((K.KD_OP_GEMM, "gemm"), (K.KD_OP_PREFILL_ATTENTION, "prefill_attention"),
                   (K.KD_OP_ROPE_PREFILL, "rope_prefill"), (K.KD_OP_ADD_RMSNORM, "add_rmsnorm"),
                   (K.KD_OP_SILU_MUL, "silu_mul")):
        rt.rt.profile_op(op)
        rt.rt.prepare()
        rt.step()
        torch.cuda.synchronize()
        t_ms, n = rt.rt.op_time()
        shares[nm] = {"ms_per_step": round(t_ms, 3), "launches": n, "share": round(t_ms / ms, 3)}
    out["step"] = {"layers": cfg.n_layers, "ms_per_step": round(ms, 3), "prompt_tokens_per_s": round(M / ms * 1e3, 1),
                   "model_tflops": round(flops / ms / 1e9, 1), "frac_of_peak": round(flops / ms / 1e9 / tf_peak, 3),
                   "ops": shares}
    print(json.dumps(out["step"]), flush=True)


if __name__ == "__main__":
    main()
