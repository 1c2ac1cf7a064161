#!/usr/bin/env python3
"""Per-kernel microbenchmark through the C ABI (CUDA events, warm L2 flushed by
rotating through distinct weight copies larger than L2). Prints one JSON line
per kernel: algorithmic bytes, avg µs, GB/s and fraction of measured HBM peak."""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2604_10180_b200 import _kd as K, api  # noqa: E402


def peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    return json.load(open(p))["hbm_gbs"] if os.path.exists(p) else 6650.0


def timeit(fn, iters=20, warm=3):
    """Device time per launch: the launches are captured in a CUDA graph so the
    host (ctypes, descriptor encoding) never starves the GPU."""
    s = torch.cuda.Stream()
    torch.cuda.synchronize()  # inputs were produced on the default stream
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(warm):
            fn(0)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(iters):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record()
        g.replay()
        e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3  # µs


def gemm(M, N, Kd, copies):
    a = K.kd_attr_gemm(M, N, Kd, K.KD_BF16)
    X = torch.randn(M, Kd, device="cuda").to(torch.bfloat16)
    Ws = [torch.randn(N, Kd, device="cuda").to(torch.bfloat16) * (1 / math.sqrt(Kd)) for _ in range(copies)]
    Y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    scr = torch.zeros(api.op_scratch_bytes(K.KD_OP_GEMM, a), dtype=torch.uint8, device="cuda")
    us = timeit(lambda i: api.gemm(a, X, Ws[i % copies], Y, scr))
    b = N * Kd * 2 + M * Kd * 2 + M * N * 2
    return us, b


def gemm_cublas(M, N, Kd, copies):
    """The same decode GEMM through torch.matmul (cuBLAS / cuBLASLt), same
    rotating weight copies: the library baseline beside our kernels."""
    X = torch.randn(M, Kd, device="cuda").to(torch.bfloat16)
    Ws = [torch.randn(N, Kd, device="cuda").to(torch.bfloat16) * (1 / math.sqrt(Kd)) for _ in range(copies)]
    Y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    us = timeit(lambda i: torch.matmul(X, Ws[i % copies].t(), out=Y))
    return us, N * Kd * 2 + M * Kd * 2 + M * N * 2


def gemm_norm(M, N, Kd, copies):
    """O/down GEMM with the fused residual add + RMSNorm epilogue (KD_OP_GEMM_RMSNORM)."""
    a = K.kd_attr_gemm_rmsnorm(M, N, Kd, K.KD_BF16, 1e-5, 0)
    X = torch.randn(M, Kd, device="cuda").to(torch.bfloat16)
    Ws = [torch.randn(N, Kd, device="cuda").to(torch.bfloat16) * (1 / math.sqrt(Kd)) for _ in range(copies)]
    r = torch.randn(M, N, device="cuda")
    gam = torch.ones(N, device="cuda").to(torch.bfloat16)
    h = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    scr = torch.zeros(api.op_scratch_bytes(K.KD_OP_GEMM_RMSNORM, a), dtype=torch.uint8, device="cuda")
    us = timeit(lambda i: api.gemm_rmsnorm(a, X, Ws[i % copies], r, gam, h, scr))
    b = N * Kd * 2 + M * Kd * 2 + M * N * (4 + 4 + 2) + N * 2
    return us, b


def qkv_rope(M, H, Hq, Hkv, D, C, copies):
    """QKV GEMM with the fused RoPE + KV-append epilogue (KD_OP_QKV_ROPE)."""
    pps = (C + 15) // 16
    N = (Hq + 2 * Hkv) * D
    a = K.kd_attr_qkv_rope(M, H, Hq, Hkv, D, 16, pps, K.KD_BF16, 5e5)
    X = torch.randn(M, H, device="cuda").to(torch.bfloat16)
    Ws = [torch.randn(N, H, device="cuda").to(torch.bfloat16) * (1 / math.sqrt(H)) for _ in range(copies)]
    bt = torch.arange(M * pps, device="cuda", dtype=torch.int32).view(M, pps)
    sl = torch.full((M,), C, device="cuda", dtype=torch.int32)
    q = torch.empty(M, Hq * D, device="cuda", dtype=torch.bfloat16)
    kc = torch.zeros(M * pps, Hkv, 16, D, device="cuda", dtype=torch.bfloat16)
    vc = torch.zeros_like(kc)
    scr = torch.zeros(api.op_scratch_bytes(K.KD_OP_QKV_ROPE, a), dtype=torch.uint8, device="cuda")
    us = timeit(lambda i: api.qkv_rope(a, X, Ws[i % copies], bt, sl, q, kc, vc, scr))
    b = N * H * 2 + M * H * 2 + M * N * 2
    return us, b


def attention(rows, Hq, Hkv, D, C):
    pps = (C + 15) // 16
    a = K.kd_attr_attention(rows, Hq, Hkv, D, 16, pps, K.KD_BF16, 0)
    kc = torch.randn(rows * pps, Hkv, 16, D, device="cuda").to(torch.bfloat16)
    vc = torch.randn(rows * pps, Hkv, 16, D, device="cuda").to(torch.bfloat16)
    bt = torch.randperm(rows * pps, device="cuda").to(torch.int32).view(rows, pps)
    sl = torch.full((rows,), C, dtype=torch.int32, device="cuda")
    q = torch.randn(rows, Hq * D, device="cuda").to(torch.bfloat16)
    out = torch.empty_like(q)
    scr = torch.zeros(max(256, api.op_scratch_bytes(K.KD_OP_ATTENTION, a)), dtype=torch.uint8, device="cuda")
    us = timeit(lambda i: api.attention(a, q, kc, vc, bt, sl, out, scr))
    b = rows * pps * Hkv * 16 * D * 2 * 2 + 2 * rows * Hq * D * 2 + rows * pps * 4 + rows * 4
    return us, b


def small_ops(m):
    H, F, Hq, Hkv, D, C = 4096, 14336, 32, 8, 128, 4096
    pps = C // 16
    out = []
    r = torch.randn(m, H, device="cuda")
    d = torch.randn(m, H, device="cuda").to(torch.bfloat16)
    gm = torch.ones(H, device="cuda").to(torch.bfloat16)
    h = torch.empty(m, H, device="cuda", dtype=torch.bfloat16)
    a = K.kd_attr_add_rmsnorm(m, H, 1, K.KD_BF16, 1e-5, 0)
    out.append(("add_rmsnorm", timeit(lambda i: api.add_rmsnorm(a, r, d, gm, h)), m * H * (4 * 2 + 2 * 2) + H * 2))
    qkv = torch.randn(m, (Hq + 2 * Hkv) * D, device="cuda").to(torch.bfloat16)
    kc = torch.randn(m * pps, Hkv, 16, D, device="cuda").to(torch.bfloat16)
    vc = torch.randn(m * pps, Hkv, 16, D, device="cuda").to(torch.bfloat16)
    bt = torch.randperm(m * pps, device="cuda").to(torch.int32).view(m, pps)
    sl = torch.full((m,), C, dtype=torch.int32, device="cuda")
    q = torch.empty(m, Hq * D, device="cuda", dtype=torch.bfloat16)
    ra = K.kd_attr_rope_append(m, Hq, Hkv, D, 16, pps, K.KD_BF16, 0, 5e5)
    out.append(("rope_append", timeit(lambda i: api.rope_append(ra, qkv, bt, sl, q, kc, vc)),
                qkv.numel() * 2 + q.numel() * 2 + m * Hkv * D * 2 * 2))
    gu = torch.randn(m, 2 * F, device="cuda").to(torch.bfloat16)
    ao = torch.empty(m, F, device="cuda", dtype=torch.bfloat16)
    sa = K.kd_attr_silu_mul(m, F, K.KD_BF16, 0)
    out.append(("silu_mul", timeit(lambda i: api.silu_mul(sa, gu, ao)), m * F * 2 * 3))
    return out


def ssm_ops(rows=64, nh=128, P=64, N=128, G=8, W=4):
    """Mamba-2 decode kernels at the hybrid config (state fp32
    [64,128,64,128] = 256 MiB read + write)."""
    import ctypes as C
    di = nh * P
    ch = di + 2 * G * N
    pin = 2 * di + 2 * G * N + nh
    a = K.kd_attr_ssm(rows, nh, P, N, G, W, K.KD_BF16, 1e-5)
    zx = torch.randn(rows, pin, device="cuda").to(torch.bfloat16)
    cw = (torch.randn(ch, W, device="cuda") * 0.5).to(torch.bfloat16)
    cb = (torch.randn(ch, device="cuda") * 0.5).to(torch.bfloat16)
    cst = torch.randn(rows, ch, W - 1, device="cuda").to(torch.bfloat16)
    xbc = torch.empty(rows, ch, device="cuda", dtype=torch.bfloat16)
    dtb = torch.full((nh,), -2.0, device="cuda")
    alog = torch.zeros(nh, device="cuda")
    Dp = torch.ones(nh, device="cuda")
    S = torch.randn(rows, nh, P, N, device="cuda") * 0.1
    y = torch.empty(rows, di, device="cuda", dtype=torch.bfloat16)
    nw = torch.ones(di, device="cuda").to(torch.bfloat16)
    yn = torch.empty(rows, di, device="cuda", dtype=torch.bfloat16)
    st = lambda: torch.cuda.current_stream().cuda_stream
    out = []
    out.append(("ssm_conv", timeit(lambda i: K.check(K.kd_op_ssm_conv(a, zx.data_ptr(), cw.data_ptr(), cb.data_ptr(),
                                                                       cst.data_ptr(), xbc.data_ptr(), st()))),
                rows * ch * 2 + rows * ch * (W - 1) * 2 * 2 + ch * W * 2 + ch * 2 + rows * ch * 2))
    out.append(("ssm_update", timeit(lambda i: K.check(K.kd_op_ssm_update(a, xbc.data_ptr(), zx.data_ptr(), dtb.data_ptr(),
                                                                           alog.data_ptr(), Dp.data_ptr(), S.data_ptr(),
                                                                           y.data_ptr(), st()))),
                S.numel() * 4 * 2 + rows * ch * 2 + rows * nh * 2 + rows * di * 2 + nh * 12))
    out.append(("gated_norm", timeit(lambda i: K.check(K.kd_op_gated_norm(a, y.data_ptr(), zx.data_ptr(), nw.data_ptr(),
                                                                           yn.data_ptr(), st()))),
                rows * di * 2 * 3 + di * 2))
    return out


def moe_ops(rows=128, H=4096, F=14336, E=8, k=2):
    """Mixtral-shaped MoE decode (SURVEY a11, B = 128): router, dispatch, the two
    grouped expert GEMMs (every expert's weights streamed once: 1.88 + 0.94
    GB), SiLU·mul on the routed rows, combine."""
    import ctypes as C
    h = torch.randn(rows, H, device="cuda").to(torch.bfloat16)
    wr = torch.randn(E, H, device="cuda") / math.sqrt(H)
    route = torch.empty(2 * rows * k, dtype=torch.int32, device="cuda")
    am = K.kd_attr_moe(rows, H, E, k)
    st = lambda: torch.cuda.current_stream().cuda_stream
    K.check(K.kd_op_moe_route(am, h.data_ptr(), wr.data_ptr(), route.data_ptr(), st()))
    mb = C.c_uint64()
    K.check(K.kd_moe_meta_bytes(rows, E, k, C.byref(mb)))
    xgm = torch.zeros(mb.value + rows * k * H * 2, dtype=torch.uint8, device="cuda")
    K.check(K.kd_op_moe_dispatch(am, h.data_ptr(), route.data_ptr(), xgm.data_ptr() + mb.value, xgm.data_ptr(), st()))
    torch.cuda.synchronize()
    wgu = torch.randn(E, 2 * F, H, device="cuda").to(torch.bfloat16) * (1 / math.sqrt(H))
    wd = torch.randn(E, H, F, device="cuda").to(torch.bfloat16) * (1 / math.sqrt(F))
    a1 = K.kd_attr_grouped_gemm(rows * k, 2 * F, H, E, rows, K.KD_BF16, 0, E)
    a2 = K.kd_attr_grouped_gemm(rows * k, H, F, E, rows, K.KD_BF16, 0, E)
    scr = torch.zeros(max(api.op_scratch_bytes(K.KD_OP_GROUPED_GEMM, a1), api.op_scratch_bytes(K.KD_OP_GROUPED_GEMM, a2)),
                      dtype=torch.uint8, device="cuda")
    gu = torch.empty(rows * k, 2 * F, dtype=torch.bfloat16, device="cuda")
    act = torch.empty(rows * k, F, dtype=torch.bfloat16, device="cuda")
    yg = torch.empty(rows * k, H, dtype=torch.bfloat16, device="cuda")
    out_t = torch.empty(rows, H, dtype=torch.bfloat16, device="cuda")
    n = rows * k
    out = []
    out.append(("moe_route", timeit(lambda i: K.check(K.kd_op_moe_route(am, h.data_ptr(), wr.data_ptr(), route.data_ptr(),
                                                                         st()))), rows * H * 2 + E * H * 4 + n * 8))
    out.append(("moe_dispatch", timeit(lambda i: K.check(K.kd_op_moe_dispatch(am, h.data_ptr(), route.data_ptr(),
                                                                               xgm.data_ptr() + mb.value, xgm.data_ptr(),
                                                                               st()))), n * 8 + n * H * 2 * 2 + mb.value))
    out.append(("grouped_gemm_gate_up", timeit(lambda i: K.check(K.kd_op_grouped_gemm(
        a1, xgm.data_ptr() + mb.value, wgu.data_ptr(), xgm.data_ptr(), gu.data_ptr(), scr.data_ptr(), st())), iters=5),
        wgu.numel() * 2 + n * H * 2 + n * 2 * F * 2))
    sa = K.kd_attr_silu_mul(n, F, K.KD_BF16, 0)
    out.append(("moe_silu_mul", timeit(lambda i: api.silu_mul(sa, gu, act)), n * F * 2 * 3))
    out.append(("grouped_gemm_down", timeit(lambda i: K.check(K.kd_op_grouped_gemm(
        a2, act.data_ptr(), wd.data_ptr(), xgm.data_ptr(), yg.data_ptr(), scr.data_ptr(), st())), iters=5),
        wd.numel() * 2 + n * F * 2 + n * H * 2))
    ac = K.kd_attr_moe_combine(rows, H, E, k, 1, 0)
    out.append(("moe_combine", timeit(lambda i: K.check(K.kd_op_moe_combine(ac, yg.data_ptr(), route.data_ptr(),
                                                                             xgm.data_ptr(), out_t.data_ptr(), st()))),
                n * H * 2 + n * 8 + n * 4 + rows * H * 2))
    return out


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--m", type=int, default=64)
    p.add_argument("--only", default="")
    args = p.parse_args()
    pk = peak()
    m = args.m
    cases = [("gemm_qkv", lambda: gemm(m, 6144, 4096, 4)), ("gemm_o", lambda: gemm(m, 4096, 4096, 5)),
             ("gemm_gu", lambda: gemm(m, 28672, 4096, 2)), ("gemm_down", lambda: gemm(m, 4096, 14336, 2)),
             ("gemm_o_norm", lambda: gemm_norm(m, 4096, 4096, 5)),
             ("gemm_qkv_rope", lambda: qkv_rope(m, 4096, 32, 8, 128, 4096, 4)),
             ("gemm_down_norm", lambda: gemm_norm(m, 4096, 14336, 2)),
             ("attention", lambda: attention(m, 32, 8, 128, 4096)),
             ("gemm_overhead_1kb", lambda: gemm(m, 128 * 148, 64, 2)),
             ("cublas_qkv", lambda: gemm_cublas(m, 6144, 4096, 4)), ("cublas_o", lambda: gemm_cublas(m, 4096, 4096, 5)),
             ("cublas_gu", lambda: gemm_cublas(m, 28672, 4096, 2)), ("cublas_down", lambda: gemm_cublas(m, 4096, 14336, 2))]
    for grp, fn in (("ssm", ssm_ops), ("moe", moe_ops)):
        if args.only == grp or args.only == "all2":
            for name, us, b in fn():
                print(json.dumps({"kernel": name, "us": round(us, 2), "bytes": b, "GBps": round(b / us / 1e3, 1),
                                  "frac": round(b / us / 1e3 / pk, 3)}), flush=True)
    if args.only in ("ssm", "moe", "all2"):
        return
    if not args.only or args.only == "small":
        for name, us, b in small_ops(m):
            print(json.dumps({"kernel": name, "m": m, "us": round(us, 2), "bytes": b,
                              "GBps": round(b / us / 1e3, 1), "frac": round(b / us / 1e3 / pk, 3)}), flush=True)
        if args.only == "small":
            return
    for name, fn in cases:
        if args.only and args.only not in name:
            continue
        us, b = fn()
        gbs = b / us / 1e3
        print(json.dumps({"kernel": name, "m": m, "us": round(us, 2), "bytes": b, "GBps": round(gbs, 1),
                          "frac": round(gbs / pk, 3)}), flush=True)


if __name__ == "__main__":
    main()
