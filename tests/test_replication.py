"""Delta replication of cross-iteration buffers (PAPER.md
P:465-466 "buffers with cross-iteration RAW dependencies (e.g., KV caches)
are handled via per-GPU replication with asynchronous delta transfers"):
KD_BUF_REPLICATED KV caches let RoPE/append run on another device than
attention. Host side: the plan's schedule and transfers (which charge the
appended slots, not the cache span) are bit-exact vs the oracle."""
import pytest

import synth
from oracle import ddg as OD, placement as OP, schedule as OS


@pytest.fixture(scope="module")
def mods():
    from paper_2604_10180_b200 import decoder as DEC, _kd as K
    from paper_2604_10180_b200.api import Plan
    return DEC, K, Plan


def split_rope_from_attention(DEC, dg):
    """RoPE/append + norms + SiLU on device 0, GEMMs on 1, attention on 2."""
    return [{DEC.T_ATTN: 2}.get(k.template, 0 if k.template in DEC.MEMORY_ROLE else 1) for k in dg.kernels]


def _decl(K, g):
    names = {getattr(K, n): n[len("KD_OP_"):] for n in dir(K) if n.startswith("KD_OP_")}
    out = []
    for op, reads, writes, attrs in g.decl:
        a = {f: getattr(attrs, f) for f, _ in attrs._fields_} if attrs is not None else {}
        out.append((names[op], a, reads, writes))
    return out


@pytest.mark.parametrize("n_micro", [1, 2, 4])
def test_replicated_kv_schedule_and_transfers_bit_exact(mods, n_micro):
    DEC, K, Plan = mods
    cfg = synth.TINY.with_(n_micro=n_micro)
    dg = DEC.DecoderGraph(cfg, replicate_kv=True)
    assign = split_rope_from_attention(DEC, dg)
    m = DEC.b200_machine(3)
    plan = Plan(dg.g, m, assign, n_micro)
    decl = _decl(K, dg.g)
    repl_bufs = {b for b, f in enumerate(dg.g._buf_flags) if f & K.KD_BUF_REPLICATED}
    repl = OS.delta_table(decl, repl_bufs)
    edges = dg.g.edges()
    om = OP.Machine(3, m.hbm_Bps, m.tc_flops, m.link_Bps, m.link_lat_ps, m.launch_ps)
    kern = [(r, w) for _, _, r, w in decl]
    t = [OP.kernel_time_ps(kern[k], dg.g._desc[k][0], om, assign[k]) for k in range(len(kern))]
    assert plan.schedule() == OS.list_schedule(len(kern), t, assign, edges, om, n_micro, repl)
    xf = OS.transfers_of(edges, assign, repl)
    got = {(p, d): b for (i, p, d, b, _, _) in plan.transfers() if i == 0}
    assert got == xf
    # the RoPE → attention transfer carries q and the two appended slots, not the caches
    name = {k.kid: k.name for k in dg.kernels}
    m_, Hq, Hkv, D = cfg.m, cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
    for (p, d), b in got.items():
        if name[p] == "rope" and d == 2:
            assert b == m_ * Hq * D * 2 + 2 * m_ * Hkv * D * 2
    # without the flag the placement violates R6 (PERSISTENT buffer on two devices)
    dg2 = DEC.DecoderGraph(cfg)
    with pytest.raises(Exception):
        Plan(dg2.g, m, [2 if k.name == "attn" else (1 if k.template not in DEC.MEMORY_ROLE else 0)
                        for k in dg2.kernels], n_micro)


def test_replicated_edge_bytes_in_objective(mods):
    """kd_objective charges a replicated-buffer edge its delta (once per
    (src, dst, buffer)), as the oracle's edge_bytes(repl)."""
    DEC, K, Plan = mods
    from paper_2604_10180_b200 import api
    cfg = synth.TINY.with_(n_micro=2)
    dg = DEC.DecoderGraph(cfg, replicate_kv=True)
    assign = split_rope_from_attention(DEC, dg)
    m = DEC.b200_machine(3)
    obj, T, M = api.objective(dg.g, m, assign, 2)
    decl = _decl(K, dg.g)
    repl = OS.delta_table(decl, {b for b, f in enumerate(dg.g._buf_flags) if f & K.KD_BUF_REPLICATED})
    om = OP.Machine(3, m.hbm_Bps, m.tc_flops, m.link_Bps, m.link_lat_ps, m.launch_ps)
    kern = [(r, w) for _, _, r, w in decl]
    t = [[OP.kernel_time_ps(kern[k], dg.g._desc[k][0], om, g) for g in range(3)] for k in range(len(kern))]
    ref = OP.objective(assign, t, OD.edge_bytes(dg.g.edges(), repl), om, 2)
    assert (obj, T, M) == ref
