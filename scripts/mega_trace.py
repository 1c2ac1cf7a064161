#!/usr/bin/env python3
"""Timeline of one KD_EXEC_MEGAKERNEL step (kd_debug_mega_trace): per task,
per role (loader / MMA / merge / workers), the earliest start, latest
dependency-satisfied and latest end over CTAs, relative to the step start.

    python scripts/mega_trace.py [--layers L] [--batch B] [--out file.json]
"""
import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2604_10180_b200 import decoder as DEC, _kd as K  # noqa: E402

ROLES = ("load", "mma", "merge", "work")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--config", default="llama3-8b")
    ap.add_argument("--out", default="")
    ap.add_argument("--unfused", action="store_true")
    a = ap.parse_args()
    cfg = synth.CONFIGS[a.config].with_(n_layers=a.layers, batch=a.batch, n_micro=1)
    dg = DEC.DecoderGraph(cfg, fuse_silu=not a.unfused, fuse_rope=not a.unfused)
    rt = DEC.DecoderRuntime(dg, [0] * dg.g.num_kernels, 1, [0], seed=cfg.seed, megakernel=True)
    info = rt.rt.exec_info(0)
    nt, grid = info["tasks"], info["grid"]
    buf = torch.zeros(nt * grid * 5 * 4, dtype=torch.int64, device="cuda")
    for _ in range(3):
        rt.step()
    torch.cuda.synchronize()
    K.check(K.kd_debug_mega_trace(rt.rt.h, 0, C.c_void_p(buf.data_ptr())), "trace on")
    rt.step()
    torch.cuda.synchronize()
    K.check(K.kd_debug_mega_trace(rt.rt.h, 0, None), "trace off")
    rt.rt.check()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(rt.streams[0])
    for _ in range(5):
        rt.step()
    e1.record(rt.streams[0])
    torch.cuda.synchronize()
    step_ms = e0.elapsed_time(e1) / 5
    tr = buf.cpu().numpy().astype(np.int64).reshape(nt, grid, 5, 4)
    t0 = tr[tr > 0].min()
    names = [k.name for k in dg.kernels]
    rows = []
    print(f"step {step_ms:.3f} ms (untraced), {nt} tasks, grid {grid}, smem {info['smem_bytes']}")
    print(f"{'task':>4} {'name':<10} " + " ".join(f"{r+'.beg':>9} {r+'.dep':>9} {r+'.end':>9}" for r in ROLES))
    for t in range(nt):
        row = {"task": t, "name": names[t] if t < len(names) else "?"}
        cols = []
        for r, rn in enumerate(ROLES):
            st = tr[t, :, r, 0]
            dp = tr[t, :, r, 1]
            en = tr[t, :, r, 2]
            beg = (st[st > 0].min() - t0) / 1e3 if (st > 0).any() else float("nan")
            dep = (dp[dp > 0].max() - t0) / 1e3 if (dp > 0).any() else float("nan")
            end = (en[en > 0].max() - t0) / 1e3 if (en > 0).any() else float("nan")
            row[rn] = [beg, dep, end]
            cols.append(f"{beg:9.1f} {dep:9.1f} {end:9.1f}")
        rows.append(row)
        print(f"{t:4d} {row['name']:<10} " + " ".join(cols))
    print("GEMM epilogue (last piece), max over CTAs, relative to that task's MMA end (us):")
    for t in range(nt):
        ep_ = tr[t, :, 4, :]
        if not (ep_[:, 0] > 0).any():
            continue
        mma_end = tr[t, :, 1, 2].max()
        def mx(k):
            v = ep_[:, k]
            return (v[v > 0].max() - mma_end) / 1e3 if (v > 0).any() else float("nan")
        def md(k, k0):
            v = ep_[:, k] - ep_[:, k0]
            ok = (ep_[:, k] > 0) & (ep_[:, k0] > 0)
            return float(np.median(v[ok])) / 1e3 if ok.any() else float("nan")
        lastdata = tr[t, :, 1, 1]
        mma_last = tr[t, :, 1, 2]
        okm = (lastdata > 0) & (mma_last > 0)
        stores = tr[t, :, 3, 1]
        oks = (stores > 0) & (ep_[:, 0] > 0)
        print(f"      median per CTA: last data -> mma commit {np.median((mma_last - lastdata)[okm]) / 1e3:5.2f}  "
              f"mma commit -> tmem seen {np.median((ep_[:, 0] - mma_last)[okm & (ep_[:, 0] > 0)]) / 1e3:5.2f}  "
              f"tmem -> own stores done {np.median((stores - ep_[:, 0])[oks]) / 1e3:5.2f}  "
              f"own stores -> published {np.median((ep_[:, 1] - stores)[oks & (ep_[:, 1] > 0)]) / 1e3:5.2f}")
        print(f"  {t:3d} {names[t] if t < len(names) else '?':<9} tmem {mx(0):6.1f} published {mx(1):6.1f} "
              f"all-present {mx(2):6.1f} folded {mx(3):6.1f} | median per CTA: store+arrive {md(1,0):5.1f} "
              f"wait {md(2,1):5.1f} fold {md(3,2):5.1f}")
    attn = [r for r in rows if r["name"] == "attn"]
    lay = [r for r in rows if r["name"] == "norm1"]
    if len(lay) >= 3:
        print(f"SUMMARY per-layer span (norm1 start to next norm1 start) us: "
              f"{(lay[2]['work'][0] - lay[1]['work'][0]):.1f}")
    if attn:
        import statistics
        spans = [r["load"][2] - r["load"][1] for r in attn[1:]] or [attn[0]["load"][2] - attn[0]["load"][1]]
        print(f"SUMMARY attention load span (dep -> end) us: median {statistics.median(spans):.1f}")
    if a.out:
        json.dump({"step_ms": step_ms, "tasks": rows, "grid": grid}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
