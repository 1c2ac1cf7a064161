"""f1 megakernel (KD_EXEC_MEGAKERNEL): one persistent launch per step runs the
device's whole schedule with in-kernel dependency waits (
launch-overhead motive P:281).

Parity: the step's residual and KV caches vs the oracle (normwise 2e-2 gate,
R14, plus element-wise bounds) and vs the per-kernel CUDA-graph path of the
same graph. add+RMSNorm / RoPE / SiLU / residual add use the standalone
kernels' per-element arithmetic; the GEMM split-K and the attention merge
orders differ, so the two executors agree within rounding, not bitwise.
Determinism: two runtimes from the same inputs produce identical bits, step
after step (monotonic completion counters, fixed fold / merge orders)."""
import numpy as np
import pytest

import synth
from oracle import layer as OL
from parity import assert_elementwise

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mod(cuda_ok):
    from paper_2604_10180_b200 import decoder as DEC, _kd as K, api
    return DEC, K, api


def relerr(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


def run(DEC, cfg, inp, steps=1, mega=True, fused=False):
    dg = DEC.DecoderGraph(cfg, fuse_silu=fused, fuse_rope=fused)
    rt = DEC.DecoderRuntime(dg, [0] * dg.g.num_kernels, 1, [0], inputs=inp, megakernel=mega)
    for _ in range(steps):
        rt.step()
    rt.sync()
    rt.rt.check()
    return rt


CFGS = {
    "tiny_m4": synth.TINY.with_(n_micro=1),                       # m = 4 rows, one micro-batch
    "tiny_n4": synth.TINY,                                        # 4 micro-batches of 1 row (interleaved schedule)
    "tiny_gqa_ragged": synth.TINY.with_(n_kv_heads=2, n_micro=2, context=77),
}


@pytest.mark.parametrize("name", list(CFGS))
def test_megakernel_step_vs_oracle(mod, name):
    DEC, K, api = mod
    cfg = CFGS[name]
    inp = synth.make_decoder_inputs(cfg)
    rt = run(DEC, cfg, inp)
    assert rt.rt.launch_count(0) == 1
    info = rt.rt.exec_info(0)
    assert info["tasks"] == rt.dg.g.num_kernels * cfg.n_micro and info["grid"] >= 1
    r_ref, kcs, vcs = OL.decoder_step(inp, act="bf16")
    r = rt.residual()
    assert relerr(r, r_ref) < 5e-3
    assert_elementwise(r, r_ref, 2, 1e-2, "residual")
    for l in range(cfg.n_layers):
        # rotated k = x·cos − y·sin of two bf16-rounded GEMM outputs: a 1-ulp
        # rounding flip of x or y (|x| ~ rms) moves k by ~1 ulp at rms scale
        # whatever |k| is, hence the rms-relative term of 2 bf16 ulps (2^-6)
        assert_elementwise(OL.bf16_to_f64(rt.cache("kc", l)), kcs[l], 2, 2e-2, f"k cache {l}")
        assert_elementwise(OL.bf16_to_f64(rt.cache("vc", l)), vcs[l], 2, 1e-2, f"v cache {l}")


RAGGED_LENS = [1, 15, 16, 17, 64, 100, 127, 128]


@pytest.mark.parametrize("n_micro", [1, 2])
def test_megakernel_ragged_lengths(mod, n_micro):
    """Per-row context lengths 1..C: the loader requests every page before the
    appended one ahead of its dependency wait, the appended page after it."""
    DEC, K, api = mod
    cfg = synth.TINY.with_(batch=8, n_micro=n_micro)
    inp = synth.make_decoder_inputs(cfg)
    inp.seq_len[:] = np.array(RAGGED_LENS, np.int32)
    rt = run(DEC, cfg, inp)
    r_ref, kcs, _ = OL.decoder_step(inp, act="bf16")
    assert relerr(rt.residual(), r_ref) < 5e-3
    assert_elementwise(rt.residual(), r_ref, 2, 1e-2, "residual")
    for l in range(cfg.n_layers):
        assert_elementwise(OL.bf16_to_f64(rt.cache("kc", l)), kcs[l], 2, 2e-2, f"k cache {l}")


def test_megakernel_matches_graph_path_over_steps_and_is_deterministic(mod):
    """Three consecutive steps (the epoch-based counters and tickets carry over
    without resets): within rounding of the per-kernel path, and two megakernel
    runtimes agree bitwise."""
    DEC, K, api = mod
    cfg = synth.TINY.with_(n_micro=2)
    inp = synth.make_decoder_inputs(cfg)
    a = run(DEC, cfg, inp, steps=3)
    b = run(DEC, cfg, inp, steps=3)
    g = run(DEC, cfg, inp, steps=3, mega=False)
    assert np.array_equal(a.residual(), b.residual())
    for l in range(cfg.n_layers):
        assert np.array_equal(a.cache("kc", l), b.cache("kc", l))
    assert relerr(a.residual(), g.residual()) < 5e-3
    assert_elementwise(a.residual(), g.residual(), 2, 1e-2, "residual vs graph path")


def test_megakernel_8b_layers_vs_graph_path_and_oracle(mod):
    """Full 8B layer shapes at the bench's batch (B=64, C=4096, N=1): vs the
    per-kernel path element by element; at B=8 also vs the oracle."""
    DEC, K, api = mod
    cfg = synth.LLAMA8B.with_(n_layers=2, batch=8)
    inp = synth.make_decoder_inputs(cfg)
    rt = run(DEC, cfg, inp)
    r_ref, _, _ = OL.decoder_step(inp, act="bf16")
    assert relerr(rt.residual(), r_ref) < 2e-2
    assert_elementwise(rt.residual(), r_ref, 4, 2e-2, "residual (B=8)")
    del rt
    cfg = synth.LLAMA8B.with_(n_layers=2, batch=64)
    inp = synth.make_decoder_inputs(cfg)
    m = run(DEC, cfg, inp, steps=2)
    g = run(DEC, cfg, inp, steps=2, mega=False)
    assert relerr(m.residual(), g.residual()) < 5e-3
    assert_elementwise(m.residual(), g.residual(), 4, 2e-2, "residual (B=64) vs graph path")
    for l in range(cfg.n_layers):
        assert_elementwise(OL.bf16_to_f64(m.cache("kc", l)), OL.bf16_to_f64(g.cache("kc", l)), 2, 2e-2, f"k cache {l}")


@pytest.mark.parametrize("name", ["tiny_m4", "tiny_gqa_ragged"])
def test_megakernel_fused_graph_vs_oracle_and_graph_path(mod, name):
    """The graph with QKV+RoPE/append and gate_up+SiLU declared as single
    kernels (KD_OP_QKV_ROPE, KD_OP_GEMM_SILU): the megakernel applies RoPE and
    SiLU·mul in the GEMM fold (rope_append / silu_mul per-element arithmetic on
    the bf16-rounded sums). vs the oracle, and vs the per-kernel fused path."""
    DEC, K, api = mod
    cfg = CFGS[name]
    inp = synth.make_decoder_inputs(cfg)
    rt = run(DEC, cfg, inp, fused=True)
    assert rt.rt.exec_info(0)["tasks"] == rt.dg.g.num_kernels * cfg.n_micro
    r_ref, kcs, vcs = OL.decoder_step(inp, act="bf16")
    assert relerr(rt.residual(), r_ref) < 5e-3
    assert_elementwise(rt.residual(), r_ref, 2, 1e-2, "residual")
    for l in range(cfg.n_layers):
        assert_elementwise(OL.bf16_to_f64(rt.cache("kc", l)), kcs[l], 2, 2e-2, f"k cache {l}")
        assert_elementwise(OL.bf16_to_f64(rt.cache("vc", l)), vcs[l], 2, 1e-2, f"v cache {l}")
    g = run(DEC, cfg, inp, steps=1, mega=False, fused=True)
    assert_elementwise(rt.residual(), g.residual(), 2, 1e-2, "residual vs per-kernel fused path")


def test_megakernel_rejects_unsupported_schedules(mod):
    """Fused ops and cross-device schedules have no megakernel task: prepare
    fails loudly (KD_ERR_UNSUPPORTED), nothing falls back."""
    DEC, K, api = mod
    cfg = synth.TINY.with_(n_micro=1)
    inp = synth.make_decoder_inputs(cfg)
    dg = DEC.DecoderGraph(cfg, fuse_norm=True)
    with pytest.raises(RuntimeError, match="megakernel"):
        DEC.DecoderRuntime(dg, [0] * dg.g.num_kernels, 1, [0], inputs=inp, megakernel=True)
    dg = DEC.DecoderGraph(cfg)
    with pytest.raises(RuntimeError, match="megakernel"):
        DEC.DecoderRuntime(dg, dg.role_assign(0, 1), 2, [0, 0], inputs=inp, megakernel=True)
