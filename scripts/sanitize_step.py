#!/usr/bin/env python3
"""One small decode configuration per kernel family, eager launches (no CUDA
graph), for compute-sanitizer (memcheck / racecheck / synccheck):
  python scripts/sanitize_step.py [dense|fused|defer|moe|ssm|all]
dense: TINY 2-device loopback pair with 4-chunk handoff; fused: the 1-GPU
fused graph (QKV+RoPE, gate_up+SiLU, GEMM+RMSNorm); moe: Mixtral-shaped tiny
EP 1+2; ssm: the hybrid tiny graph. Exits non-zero on a runtime error."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import synth  # noqa: E402
from paper_2604_10180_b200 import decoder as DEC  # noqa: E402


def run(dg, assign, n_dev, inp, **kw):
    rt = DEC.DecoderRuntime(dg, assign, n_dev, [0] * n_dev, inputs=inp, use_graph=False, **kw)
    for _ in range(2):
        rt.step()
    rt.sync()
    rt.rt.check()
    r = rt.residual() if not hasattr(dg, "residual_global") else dg.residual_global(rt)
    assert np.isfinite(r).all()
    return r


def main(which):
    if which in ("dense", "all"):
        cfg = synth.TINY
        inp = synth.make_decoder_inputs(cfg)
        dg = DEC.DecoderGraph(cfg)
        run(dg, dg.role_assign(0, 1), 2, inp, n_chunks=4)
        print("dense pair ok", flush=True)
    if which in ("fused", "all"):
        cfg = synth.TINY
        inp = synth.make_decoder_inputs(cfg)
        dg = DEC.DecoderGraph(cfg, fuse_silu=True, fuse_rope=True, fuse_norm=True)
        run(dg, [0] * dg.g.num_kernels, 1, inp)
        print("fused ok", flush=True)
    if which in ("defer", "all"):  # the bench's 1-GPU graph: RMSNorm's 1/rms deferred to the consumers (R31)
        cfg = synth.TINY
        inp = synth.make_decoder_inputs(cfg)
        dg = DEC.DecoderGraph(cfg, fuse_silu=True, fuse_rope=True, fuse_norm="defer")
        run(dg, [0] * dg.g.num_kernels, 1, inp)
        print("deferred-norm fused ok", flush=True)
    if which in ("moe", "all"):
        a, e, m = 1, 2, 2
        cfg = synth.TINY.with_(n_experts=4, top_k=2, n_micro=2, batch=a * 2 * m)
        inp = synth.make_decoder_inputs(cfg)
        dg = DEC.MoEEPDecoderGraph(cfg.with_(batch=2 * m), a, e)
        run(dg, dg.assign(), a + e, inp)
        print("moe ok", flush=True)
    if which in ("ssm", "all"):
        cfg = synth.TINY_HYBRID if hasattr(synth, "TINY_HYBRID") else None
        if cfg is not None:
            inp = synth.make_decoder_inputs(cfg)
            dg = DEC.DecoderGraph(cfg)
            run(dg, [0] * dg.g.num_kernels, 1, inp)
            print("ssm ok", flush=True)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "all")
