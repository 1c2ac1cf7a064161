#!/usr/bin/env python3
"""Per-CTA phase timeline of one GEMM launch (kd_debug_gemm_trace).

usage: trace_gemm.py [qkv|o|gu|down|o_norm|down_norm|qkv_rope|gu_silu ...]
(8B shapes, m=64; the traced launch streams cold weights). The fused-norm
variants print per-phase cycle counts of the norm epilogue instead."""
import ctypes as C, os, sys, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_10180_b200 import _kd as K, api
shapes = {"qkv": (64, 6144, 4096), "o": (64, 4096, 4096), "gu": (64, 28672, 4096), "down": (64, 4096, 14336),
          "o_norm": (64, 4096, 4096), "down_norm": (64, 4096, 14336), "qkv_rope": (64, 6144, 4096), "gu_silu": (64, 28672, 4096)}
plain_gemm = api.gemm
for name in (sys.argv[1:] or list(shapes)):
    M, N, Kd = shapes[name]
    norm = name.endswith("_norm")
    rope = name == "qkv_rope"
    api.gemm = plain_gemm
    a = K.kd_attr_gemm_rmsnorm(M, N, Kd, K.KD_BF16, 1e-5, 0) if norm else K.kd_attr_gemm(M, N, Kd, K.KD_BF16)
    if name == "gu_silu":
        api.gemm = lambda a_, X_, W_, Y_, s_: api.gemm_silu(a_, X_, W_, Y_, s_)
    if rope:
        a = K.kd_attr_qkv_rope(M, Kd, 32, 8, 128, 16, 256, K.KD_BF16, 5e5)
        bt = torch.arange(M * 256, device="cuda", dtype=torch.int32).view(M, 256)
        sl = torch.full((M,), 4096, device="cuda", dtype=torch.int32)
        q = torch.empty(M, 32 * 128, device="cuda", dtype=torch.bfloat16)
        kc = torch.zeros(M * 256, 8, 16, 128, device="cuda", dtype=torch.bfloat16)
        vc = torch.zeros_like(kc)
        api.gemm = lambda a_, X_, W_, Y_, s_: api.qkv_rope(a_, X_, W_, bt, sl, q, kc, vc, s_)
    X = torch.randn(M, Kd, device="cuda").to(torch.bfloat16)
    W = torch.randn(N, Kd, device="cuda").to(torch.bfloat16)
    W2 = torch.randn(N, Kd, device="cuda").to(torch.bfloat16)
    Y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    op = K.KD_OP_GEMM_RMSNORM if norm else (K.KD_OP_QKV_ROPE if rope else
                                            (K.KD_OP_GEMM_SILU if name == "gu_silu" else K.KD_OP_GEMM))
    scr = torch.zeros(max(256, api.op_scratch_bytes(op, a)), dtype=torch.uint8, device="cuda")
    r = torch.randn(M, N, device="cuda")
    gam = torch.ones(N, device="cuda").to(torch.bfloat16)
    if norm:
        api.gemm = lambda a_, X_, W_, Y_, s_: api.gemm_rmsnorm(a_, X_, W_, r, gam, Y_, s_)
    tr = torch.zeros(148 * 32, dtype=torch.int64, device="cuda")
    for _ in range(3):
        api.gemm(a, X, W, Y, scr)
    torch.cuda.synchronize()
    K.kd_debug_gemm_trace(C.c_void_p(tr.data_ptr()))
    api.gemm(a, X, W2, Y, scr)       # cold weights
    torch.cuda.synchronize()
    K.kd_debug_gemm_trace(None)
    t = tr.view(148, 32).cpu().numpy().astype("float64")
    t0 = t[:, 0][t[:, 0] > 0].min()  # rows past the grid are unused (0)
    rel = (t - t0) / 1000.0
    rel[t == 0] = float("nan")
    rel[:, 16:] = float("nan")  # slots 16.. hold clock64 cycle stamps
    import numpy as np
    labels = ["entry", "setup", "tma0", "tmaN", "full0", "commitN", "seg0.wait", "seg0.done", "seg1.wait", "seg1.done",
              "seg2.wait", "seg2.done", "-", "fold.end|n.A", "n.bar", "exit|n.end", "gbar.pass", "-", "gbar.arrive", "-"] + ["-"] * 12
    print(f"== {name} M={M} N={N} K={Kd}: span {np.nanmax(rel):.2f} us")
    raw = tr.view(148, 32).cpu().numpy()
    if os.environ.get("KD_GEMM_DBG", "0") != "0":
        print("  probe cycles (slots 16-18):", [int(np.median(raw[:, k])) for k in (16, 17, 18)],
              "max", [int(raw[:, k].max()) for k in (16, 17, 18)])
    if norm:
        d = lambda a, b: int(np.median(raw[:, b].astype(np.int64) - raw[:, a].astype(np.int64)))
        print("  norm cycles: A", d(22, 16), "sync", d(16, 17), "B", d(17, 18), "sync+fence..arrive", d(18, 24),
              "barrier", d(24, 23), "C", d(23, 19), "sync", d(19, 20), "D", d(20, 21))
        continue
    if name in ("gu", "gu_silu"):
        d = lambda a, b: int(np.median(raw[:, b].astype(np.int64) - raw[:, a].astype(np.int64)))
        print("  prologue cycles: first TMA issue", d(24, 25), "rest of the first ring", d(25, 26))
    own_rows = raw[raw[:, 21] > 0] if name in ("gu", "gu_silu") else raw[:0]
    if len(own_rows):
        print(f"  fold cycles: med {np.median(own_rows[:, 20]):.0f} max {own_rows[:, 20].max()}  nb {np.unique(own_rows[:, 21])} n4 {np.unique(own_rows[:, 22])}")
    for i, l in enumerate(labels):
        col = rel[:, i]
        if np.all(np.isnan(col)):
            continue
        print(f"  {i:2d} {l:10s} min {np.nanmin(col):7.2f} med {np.nanmedian(col):7.2f} max {np.nanmax(col):7.2f}  n={np.sum(~np.isnan(col))}")
