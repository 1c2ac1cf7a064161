"""Host-side declaration of the decoder kernel graph (no GPU): which kernels a
graph declares for each fusion option, and that the DAG built from their
declared read/write spans still orders every fused kernel after its
producers and before its consumers."""
import pytest

import synth
from paper_2604_10180_b200 import _kd as K
from paper_2604_10180_b200 import decoder as DEC

CFG = synth.TINY.with_(n_layers=3)


def names(dg):
    return [k.name for k in dg.kernels]


def per_layer(dg, layer):
    return [k.name for k in dg.kernels if k.layer == layer]


@pytest.mark.parametrize("opts,layer_ops", [
    ({}, ["norm1", "qkv", "rope", "attn", "o", "norm2", "gu", "silu", "down"]),
    ({"fuse_silu": True}, ["norm1", "qkv", "rope", "attn", "o", "norm2", "gu_silu", "down"]),
    ({"fuse_rope": True}, ["norm1", "qkv_rope", "attn", "o", "norm2", "gu", "silu", "down"]),
    ({"fuse_norm": "o"}, ["norm1", "qkv", "rope", "attn", "o_norm", "gu", "silu", "down"]),
])
def test_layer_kernels_per_fusion(opts, layer_ops):
    dg = DEC.DecoderGraph(CFG, **opts)
    for l in range(CFG.n_layers):
        ops = per_layer(dg, l)
        if l == CFG.n_layers - 1:
            assert ops[-1] == "final_add"
            ops = ops[:-1]
        assert ops == layer_ops


def test_full_norm_fusion_moves_norm1_into_the_previous_down():
    dg = DEC.DecoderGraph(CFG, fuse_silu=True, fuse_rope=True, fuse_norm=True)
    L = CFG.n_layers
    assert per_layer(dg, 0) == ["norm1", "qkv_rope", "attn", "o_norm", "gu_silu", "down_norm"]
    for l in range(1, L - 1):
        assert per_layer(dg, l) == ["qkv_rope", "attn", "o_norm", "gu_silu", "down_norm"]
    assert per_layer(dg, L - 1) == ["qkv_rope", "attn", "o_norm", "gu_silu", "down", "final_add"]
    # the unfused intermediates are never allocated
    assert "o.0" not in dg.buf and "gu.0" not in dg.buf and "qkv.0" not in dg.buf and "d.0" not in dg.buf
    assert f"d.{L - 1}" in dg.buf
    ops = {k.name: k for k in dg.kernels if k.layer == 0}
    assert dg.g.num_kernels == len(dg.kernels)
    assert {k.name for k in dg.kernels if k.layer == 1} >= {"qkv_rope", "o_norm", "down_norm"}
    assert ops["o_norm"].kid < ops["gu_silu"].kid


def test_fused_graph_dag_orders_producers_and_consumers():
    dg = DEC.DecoderGraph(CFG, fuse_silu=True, fuse_rope=True, fuse_norm=True)
    kid = {(k.name, k.layer): k.kid for k in dg.kernels}
    edges = {(e[0], e[1]) for e in dg.g.edges()}
    for l in range(CFG.n_layers - 1):
        # down_norm(l) writes h1.{l+1} and r: the next layer's QKV+RoPE reads h1
        assert (kid[("down_norm", l)], kid[("qkv_rope", l + 1)]) in edges
        assert (kid[("attn", l)], kid[("o_norm", l)]) in edges
        assert (kid[("o_norm", l)], kid[("gu_silu", l)]) in edges
        assert (kid[("gu_silu", l)], kid[("down_norm", l)]) in edges
        # the residual stream: o_norm(l) → down_norm(l) (both read and write r)
        assert (kid[("o_norm", l)], kid[("down_norm", l)]) in edges
    assert (kid[("qkv_rope", 0)], kid[("attn", 0)]) in edges   # q and the KV cache


def test_fp32_graph_ignores_the_bf16_fusions():
    dg = DEC.DecoderGraph(CFG, K.KD_F32, fuse_silu=True, fuse_rope=True, fuse_norm=True)
    assert not (set(names(dg)) & {"gu_silu", "qkv_rope", "o_norm", "down_norm"})
