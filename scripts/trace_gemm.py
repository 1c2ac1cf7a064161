#!/usr/bin/env python3
"""Per-CTA phase timeline of one GEMM launch (kd_debug_gemm_trace)."""
import ctypes as C, os, sys, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_10180_b200 import _kd as K, api
shapes = {"qkv": (64, 6144, 4096), "o": (64, 4096, 4096), "gu": (64, 28672, 4096), "down": (64, 4096, 14336)}
for name in (sys.argv[1:] or list(shapes)):
    M, N, Kd = shapes[name]
    a = K.kd_attr_gemm(M, N, Kd, K.KD_BF16)
    X = torch.randn(M, Kd, device="cuda").to(torch.bfloat16)
    W = torch.randn(N, Kd, device="cuda").to(torch.bfloat16)
    W2 = torch.randn(N, Kd, device="cuda").to(torch.bfloat16)
    Y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    scr = torch.zeros(api.op_scratch_bytes(K.KD_OP_GEMM, a), dtype=torch.uint8, device="cuda")
    tr = torch.zeros(148 * 32, dtype=torch.int64, device="cuda")
    for _ in range(3):
        api.gemm(a, X, W, Y, scr)
    torch.cuda.synchronize()
    K.kd_debug_gemm_trace(C.c_void_p(tr.data_ptr()))
    api.gemm(a, X, W2, Y, scr)       # cold weights
    torch.cuda.synchronize()
    K.kd_debug_gemm_trace(None)
    t = tr.view(148, 32).cpu().numpy().astype("float64")
    t0 = t[:, 0].min()
    rel = (t - t0) / 1000.0
    rel[t == 0] = float("nan")
    rel[:, 20:] = float("nan")
    import numpy as np
    labels = ["entry", "setup", "tma0", "tmaN", "full0", "commitN", "seg0.wait", "seg0.done", "seg1.wait", "seg1.done",
              "seg2.wait", "seg2.done", "-", "fold.end", "-", "exit", "gbar.pass", "-", "gbar.arrive", "-"] + ["-"] * 12
    print(f"== {name} M={M} N={N} K={Kd}: span {np.nanmax(rel):.2f} us")
    raw = tr.view(148, 32).cpu().numpy()
    own_rows = raw[raw[:, 21] > 0]
    if len(own_rows):
        print(f"  fold cycles: med {np.median(own_rows[:, 20]):.0f} max {own_rows[:, 20].max()}  nb {np.unique(own_rows[:, 21])} n4 {np.unique(own_rows[:, 22])}")
    for i, l in enumerate(labels):
        col = rel[:, i]
        if np.all(np.isnan(col)):
            continue
        print(f"  {l:10s} min {np.nanmin(col):7.2f} med {np.nanmedian(col):7.2f} max {np.nanmax(col):7.2f}  n={np.sum(~np.isnan(col))}")
