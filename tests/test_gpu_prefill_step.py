"""f4: the PREFILL kernel graph through the same DAG / plan / runtime
(kd_step, C ABI) as decode. A prefill step over S prompt tokens per sequence
vs the prefill oracle (oracle/prefill.py), and the method-level invariant:
the disaggregated prefill graph (norms, RoPE + cache fill, attention, SiLU on
one logical device, the tensor-bound GEMMs on another, cut edges by fused
peer stores + flags in loopback) is BITWISE equal to the monolithic run."""
import numpy as np
import pytest

import synth
from oracle import layer as OL, prefill as PF
from parity import assert_elementwise

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mod(cuda_ok):
    from paper_2604_10180_b200 import decoder as DEC
    return DEC


def relerr(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


def prompt_inputs(cfg, S, seed=5):
    inp = synth.make_decoder_inputs(cfg, seed=seed)
    g = np.random.default_rng(seed + 1)
    inp.x = g.standard_normal((cfg.batch * S, cfg.hidden)).astype(np.float32)
    return inp


def run(DEC, cfg, S, inp, assign=None, n_dev=1):
    pg = DEC.PrefillGraph(cfg, S)
    a = [0] * pg.g.num_kernels if assign is None else assign(pg)
    rt = DEC.DecoderRuntime(pg, a, n_dev, [0] * n_dev, inputs=inp)
    rt.step()
    rt.sync()
    rt.rt.check()
    return rt


# (cfg, S): M = B·S = 512 rows → the large-M tensor-bound GEMM; GQA; 8B layer shapes
CASES = {
    "tiny_S256": (synth.TINY.with_(n_micro=1, batch=2, context=256), 256),
    "tiny_gqa_S320": (synth.TINY.with_(n_micro=1, batch=2, n_kv_heads=2, context=336), 320),
    "8b_2layers_S128": (synth.LLAMA8B.with_(n_layers=2, batch=4, context=256), 128),
}


@pytest.mark.parametrize("name", list(CASES))
def test_prefill_step_vs_oracle(mod, name):
    DEC = mod
    cfg, S = CASES[name]
    inp = prompt_inputs(cfg, S)
    rt = run(DEC, cfg, S, inp)
    r_ref, kcs, vcs = PF.prefill_step(inp, S)
    r = rt.residual()
    assert relerr(r, r_ref) < 1e-2
    assert_elementwise(r, r_ref, 4, 3e-2, "prefill residual")
    for l in range(cfg.n_layers):
        assert relerr(OL.bf16_to_f64(rt.cache("kc", l)), kcs[l]) < 1e-2
        assert_elementwise(OL.bf16_to_f64(rt.cache("vc", l)), vcs[l], 2, 2e-2, f"v cache {l}")


def test_prefill_disaggregated_bitwise_equals_monolithic(mod):
    DEC = mod
    cfg, S = CASES["tiny_gqa_S320"]
    inp = prompt_inputs(cfg, S)
    mono = run(DEC, cfg, S, inp)
    dis = run(DEC, cfg, S, inp, assign=lambda pg: pg.role_assign(0, 1), n_dev=2)
    assert len(dis.plan.transfers()) > 0
    assert np.array_equal(mono.residual(), dis.residual())
    for l in range(cfg.n_layers):
        assert np.array_equal(mono.cache("kc", l), dis.cache("kc", l))


def test_prefill_then_decode_matches_oracle(mod):
    """A prompt prefilled through kd_step, then one decode step of the next
    token on the SAME caches through the decode graph: vs the oracle's
    prefill(S) + decode_step(seq_len = S + 1)."""
    DEC = mod
    cfg = synth.TINY.with_(n_micro=1, batch=2, context=272)
    S = 256
    inp = prompt_inputs(cfg, S)
    pre = run(DEC, cfg, S, inp)
    kbits = [pre.cache("kc", l) for l in range(cfg.n_layers)]
    vbits = [pre.cache("vc", l) for l in range(cfg.n_layers)]
    g = np.random.default_rng(9)
    x_next = g.standard_normal((cfg.batch, cfg.hidden)).astype(np.float32)
    dec_inp = synth.DecoderInputs(cfg, inp.layers, x_next, kbits, vbits, inp.block_table,
                                  np.full(cfg.batch, S + 1, np.int32))
    dg = DEC.DecoderGraph(cfg)
    rt = DEC.DecoderRuntime(dg, [0] * dg.g.num_kernels, 1, [0], inputs=dec_inp)
    rt.step()
    rt.sync()
    rt.rt.check()
    # oracle: prefill then decode, all in fp64 (caches from the oracle's own prefill)
    _, kcs, vcs = PF.prefill_step(inp, S)
    to_bits = lambda v: synth.f32_to_bf16_bits(np.asarray(v, np.float32))
    ref_inp = synth.DecoderInputs(cfg, inp.layers, x_next, [to_bits(k) for k in kcs], [to_bits(v) for v in vcs],
                                  inp.block_table, np.full(cfg.batch, S + 1, np.int32))
    r_ref, _, _ = OL.decoder_step(ref_inp)
    assert relerr(rt.residual(), r_ref) < 1e-2
    assert_elementwise(rt.residual(), r_ref, 4, 3e-2, "decode after prefill")
