#!/usr/bin/env python3
"""KD_MODE_LOG evidence of the chunked handoff: run the 8B-shaped
disaggregated pair (m = 32 rows per micro-batch, N = 2; memory role on logical
device 0, GEMMs on device 1, loopback on one GPU) for a few steps and
summarise, per cut edge kind, when the consumer first acquired each chunk
relative to the producer's per-chunk completion (%globaltimer, ns), plus the
kd_step_stats of the last step. Output: one JSON object on stdout."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import synth
    from paper_2604_10180_b200 import decoder as DEC, _kd as K
    layers = int(os.environ.get("KD_LOG_LAYERS", "2"))
    n_chunks = int(os.environ.get("KD_LOG_CHUNKS", "4"))
    cfg = synth.LLAMA8B.with_(n_layers=layers, batch=64, n_micro=2)
    dg = DEC.DecoderGraph(cfg)
    rt = DEC.DecoderRuntime(dg, dg.role_assign(0, 1), 2, [0, 0], seed=1, n_chunks=n_chunks, mode=K.KD_MODE_LOG)
    for _ in range(3):
        rt.step()
    st = rt.step(stats=True)
    rt.rt.check()
    recs = rt.rt.log()
    xs = rt.plan.transfers()
    name = {k.kid: k.name for k in dg.kernels}
    per = {}
    for dev, t, c, epoch, tw, ta, tr in recs:
        per.setdefault(t, []).append((c, tw, ta, tr))
    kinds = {}
    for t, v in per.items():
        v.sort()
        i, prod, dst, nbytes = xs[t][:4]
        first_acq = min(ta for _, _, ta, _ in v)
        last_rel = max(tr for *_, tr in v)
        first_rel = min(tr for *_, tr in v)
        k = kinds.setdefault(name[prod], {"transfers": 0, "chunks": len(v), "bytes": nbytes, "overlap_ns": [],
                                           "release_spread_ns": [], "stall_ns": []})
        k["transfers"] += 1
        k["overlap_ns"].append(last_rel - first_acq)       # > 0: consumer started before the last chunk was done
        k["release_spread_ns"].append(last_rel - first_rel)
        k["stall_ns"].append(sum(max(0, ta - tw) for _, tw, ta, _ in v))
    out = {"config": f"8B layer shapes, L={layers}, B=64, N=2 (m=32), n_chunks={n_chunks}, 2 logical devices on 1 GPU "
                     "(loopback), KD_MODE_LOG",
           "records": len(recs), "step_stats": st, "per_producer": {}}
    for nm, k in kinds.items():
        ov = k["overlap_ns"]
        out["per_producer"][nm] = {"transfers": k["transfers"], "chunks": k["chunks"], "bytes": k["bytes"],
                                   "overlapped_transfers": sum(1 for x in ov if x > 0),
                                   "median_overlap_ns": sorted(ov)[len(ov) // 2],
                                   "median_release_spread_ns": sorted(k["release_spread_ns"])[len(ov) // 2],
                                   "median_stall_ns": sorted(k["stall_ns"])[len(ov) // 2]}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
