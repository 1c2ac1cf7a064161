#!/usr/bin/env python3
"""In-step timeline of the 8B decode step (kd_debug_timeline).

Runs the bench's 1-GPU monolithic step (fused graph, CUDA graph + PDL) with
every GEMM / attention launch writing per-CTA %globaltimer stamps, then prints,
per launch kind averaged over the layers, when the launch's CTAs start, pass
their dependency wait, finish streaming (last MMA / producer done) and exit,
relative to the previous launch's last CTA exit — i.e. where each kernel
boundary spends its time with HBM idle.

usage: step_timeline.py [--layers L] [--steps K] [--json out.json]"""
import argparse, ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=32)
ap.add_argument("--steps", type=int, default=6)
ap.add_argument("--json", default="")
args = ap.parse_args()

import synth
from paper_2604_10180_b200 import decoder as DEC, _kd as K

cfg = synth.CONFIGS["llama3-8b"].with_(n_micro=1, n_layers=args.layers)
dg = DEC.DecoderGraph(cfg, fuse_silu=True, fuse_rope=True, fuse_norm=os.environ.get("KD_TL_FUSE_NORM", "defer"))
rt = DEC.DecoderRuntime(dg, [0] * dg.g.num_kernels, 1, [0], seed=cfg.seed, use_graph=True)
REG = 512 * 32
n_max = 8 * args.layers + 16
buf = torch.zeros(n_max * REG, dtype=torch.int64, device="cuda")
K.kd_debug_timeline(C.c_void_p(buf.data_ptr()), C.c_uint64(buf.numel() * 8))
for _ in range(args.steps):
    rt.step()
torch.cuda.synchronize()
n = C.c_uint32()
K.kd_debug_timeline_kinds(None, 0, C.byref(n))
kinds = (C.c_int32 * n.value)()
K.kd_debug_timeline_kinds(kinds, n.value, C.byref(n))
K.kd_debug_timeline(None, 0)
kinds = list(kinds)
T = buf.view(n_max, 512, 32)[: len(kinds)].cpu().numpy().astype(np.float64)
name = {100: "qkv/o csk", 101: "qkv+rope", 102: "gemm+norm(csk)", 200: "gemm(sk)", 201: "gate_up+silu",
        202: "gemm+norm(sk)", 300: "attention"}

recs = []
slots = {}  # launch label -> list over layers of per-slot (median, max) over CTAs, µs after the previous end
prev_end = None
prev_kind = None
t0 = None
for i, k in enumerate(kinds):
    R = T[i]
    live = R[:, 0] > 0
    if not live.any():
        continue
    R = R[live]
    if t0 is None:
        t0 = R[:, 0].min()
    rel = lambda v: float(v - (prev_end if prev_end is not None else t0)) / 1e3  # µs after previous launch's end
    if k == 300:
        end = R[:, [3, 4]].max()
        rec = dict(kind=name[k], first_entry=rel(R[:, 0].min()), last_entry=rel(R[:, 0].max()),
                   wait_done=rel(R[:, 1][R[:, 1] > 0].min()), stream_done_first=rel(R[:, 2].min()),
                   stream_done_last=rel(R[:, 2].max()), end=rel(end))
    else:
        end = R[:, 15].max()
        lastmma = R[:, 5][R[:, 5] > 0]
        ep = R[:, 6][R[:, 6] > 0]
        rec = dict(kind=name.get(k, str(k)), first_entry=rel(R[:, 0].min()), last_entry=rel(R[:, 0].max()),
                   first_mma=rel(R[:, 4][R[:, 4] > 0].min()), first_mma_last=rel(R[:, 4][R[:, 4] > 0].max()),
                   last_mma_first=rel(lastmma.min()) if lastmma.size else None,
                   last_mma_last=rel(lastmma.max()) if lastmma.size else None,
                   epi_start_med=rel(np.median(ep)) if ep.size else None, exit_first=rel(R[:, 15][R[:, 15] > 0].min()),
                   end=rel(end))
    rec["span"] = rec["end"] - 0.0
    recs.append(rec)
    if prev_end is not None:
        label = rec["kind"] + ("" if k not in (102,) else (" [O+norm2]" if prev_kind == 300 else " [down+norm1]"))
        row = []
        for sl in range(16):
            v = R[:, sl][R[:, sl] > 0]
            row.append((rel(np.median(v)), rel(v.max())) if v.size else (None, None))
        slots.setdefault(label, []).append(row)
    prev_end = end
    prev_kind = k

# group by position in the layer pattern (kind sequence repeats per layer)
by = {}
for r in recs[1:]:  # drop the first launch (no previous end in this step)
    by.setdefault(r["kind"], []).append(r)
out = {}
print(f"{len(recs)} traced launches; µs relative to the previous launch's last CTA exit (mean over layers)")
for k, rs in by.items():
    keys = [x for x in rs[0] if x != "kind" and rs[0][x] is not None]
    avg = {x: float(np.mean([r[x] for r in rs if r.get(x) is not None])) for x in keys}
    out[k] = dict(n=len(rs), **{x: round(v, 2) for x, v in avg.items()})
    print(f"{k:16s} n={len(rs):3d} " + " ".join(f"{x}={v:7.2f}" for x, v in avg.items()))
print("per-slot stamps (median / max over CTAs, mean over layers; µs after the previous launch's end):")
slot_out = {}
for label, rows in slots.items():
    parts = []
    slot_out[label] = {}
    for sl in range(16):
        med = [r[sl][0] for r in rows if r[sl][0] is not None]
        mx = [r[sl][1] for r in rows if r[sl][1] is not None]
        if med:
            slot_out[label][sl] = (round(float(np.mean(med)), 2), round(float(np.mean(mx)), 2))
            parts.append(f"{sl}:{np.mean(med):.1f}/{np.mean(mx):.1f}")
    print(f"  {label:28s} " + " ".join(parts))
# attention tail: per CTA, epilogue lag behind its consumers and the last two items' epilogue spans
lag, last_items, worst = [], [], []
for i, k in enumerate(kinds):
    if k != 300 or i == 0:
        continue
    R = T[i]
    R = R[R[:, 0] > 0]
    lag.append(float(np.median(R[:, 3] - R[:, 4])) / 1e3)
    v = (R[:, 8] > 0) & (R[:, 7] > 0)
    last_items.append((float(np.median(R[v, 8] - R[v, 7])) / 1e3, float(np.median(R[v, 7] - R[v, 6])) / 1e3))
    w = int(np.argmax(R[:, 3]))
    worst.append([(R[w, sl] - R[w, 4]) / 1e3 for sl in (5, 6, 7, 8, 9, 3)])
if lag:
    print(f"attention epilogue lag behind consumers (median over CTAs) {np.mean(lag):.2f} us; last item epilogue "
          f"{np.mean([a for a, _ in last_items]):.2f} us, gap before it {np.mean([b for _, b in last_items]):.2f} us")
    print("  last CTA out, relative to its consumers' end (us): prev item acquired/done, last acquired/done, "
          "split atomic, exit: " + " ".join(f"{x:.2f}" for x in np.mean(np.array(worst), axis=0)))
# cluster split-K epilogue (non-norm: QKV+RoPE, plain): TMEM → DSMEM push (clock64 slots 21 → 22),
# owner sum + stores (24 → 25), in cycles
for kk, nm in ((101, "qkv+rope"), (100, "plain csk")):
    push, own = [], []
    for i, k in enumerate(kinds):
        if k != kk:
            continue
        R = T[i]
        R = R[(R[:, 0] > 0) & (R[:, 24] > 0) & (R[:, 25] > 0)]
        if len(R):
            push.append(float(np.median(R[:, 22] - R[:, 21])))
            own.append((float(np.median(R[:, 27] - R[:, 24])), float(np.median(R[:, 28] - R[:, 27])),
                        float(np.median(R[:, 25] - R[:, 28]))))
    if push:
        o = np.mean(np.array(own), axis=0)
        print(f"{nm} epilogue (cycles, median over CTAs): push={np.mean(push):.0f} owner sum={o[0]:.0f} "
              f"sync={o[1]:.0f} stores (RoPE)={o[2]:.0f}")
# fused-norm epilogue sub-phases (clock64 stamps, slots 16-24; cycles, median over CTAs, mean over launches)
chain = [(22, "waits"), (16, "sum+add"), (17, "sync"), (18, "ssq"), (24, "sync"), (23, "barrier"), (19, "x-CTA sums"),
         (20, "sync"), (21, "norm+stores")]
ph = {}
for i, k in enumerate(kinds):
    if k != 102:
        continue
    R = T[i]
    R = R[R[:, 0] > 0]
    for (a, _), (b, nm) in zip(chain, chain[1:]):
        d = R[:, b] - R[:, a]
        d = d[(R[:, a] > 0) & (R[:, b] > 0)]
        if d.size:
            ph.setdefault(nm, []).append(float(np.median(d)))
if ph:
    print("fused-norm epilogue phases (cycles, median over CTAs): " +
          " ".join(f"{nm}={np.mean(v):.0f}" for nm, v in ph.items()))
total = sum(r["span"] for r in recs[1:])
print(f"sum of spans {total / 1e3:.3f} ms over {len(recs) - 1} launches")
if args.json:
    json.dump(dict(per_kind=out, slots=slot_out, launches=recs), open(args.json, "w"), indent=1)
