"""kd_debug_timeline (the in-step timeline scripts/step_timeline.py reads):
every GEMM and attention launch captured into a step graph writes per-CTA
%globaltimer stamps to its own region, tagged with its kind, and the stamps
describe a real execution (entry <= exit, launches in stream order), while
the step's result is unchanged by the instrumentation (bitwise)."""
import ctypes as C

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

REG = 512 * 32  # u64 stamps per launch region (include/kd.h)


def test_timeline_stamps_and_bits(cuda_ok):
    import torch
    from paper_2604_10180_b200 import decoder as DEC, _kd as K
    cfg = synth.TINY.with_(n_micro=1)
    inp = synth.make_decoder_inputs(cfg)

    def make():
        dg = DEC.DecoderGraph(cfg, fuse_silu=True, fuse_rope=True, fuse_norm=True)
        return DEC.DecoderRuntime(dg, [0] * dg.g.num_kernels, 1, [0], inputs=inp, use_graph=True)

    ref = make()
    ref.step()
    ref.sync()
    r_ref = ref.residual()

    n_max = 64
    buf = torch.zeros(n_max * REG, dtype=torch.int64, device="cuda")
    K.kd_debug_timeline(C.c_void_p(buf.data_ptr()), C.c_uint64(buf.numel() * 8))
    try:
        rt = make()
        rt.step()  # captures the step graph with the timeline regions baked in
        rt.sync()
        rt.rt.check()
        n = C.c_uint32()
        K.kd_debug_timeline_kinds(None, 0, C.byref(n))
        kinds = (C.c_int32 * n.value)()
        K.kd_debug_timeline_kinds(kinds, n.value, C.byref(n))
        kinds = list(kinds)
    finally:
        K.kd_debug_timeline(None, 0)
    assert np.array_equal(rt.residual().view(np.uint32), r_ref.view(np.uint32))  # instrumentation changes no bit
    assert 300 in kinds, kinds                        # decode attention
    assert any(100 <= k < 200 for k in kinds), kinds  # cluster split-K GEMMs (fused QKV+RoPE / norm)
    assert kinds.count(300) == cfg.n_layers
    T = buf.view(n_max, 512, 32)[: len(kinds)].cpu().numpy()
    prev_entry = 0
    for i, k in enumerate(kinds):
        R = T[i][T[i][:, 0] > 0]
        assert len(R) > 0, f"launch {i} (kind {k}) wrote no stamps"
        end = R[:, [3, 4]].max(axis=1) if k == 300 else R[:, 15]
        assert (end >= R[:, 0]).all(), f"launch {i}: a CTA ends before it starts"
        # stream order: a launch's first CTA never starts before the previous launch's first CTA
        assert R[:, 0].min() >= prev_entry
        prev_entry = R[:, 0].min()
