"""Chunk table of the chunked P2P handoff (reading R10):
the library's kd_plan_chunks is bit-exact against the oracle's independent
restatement (oracle.schedule.chunk_table) on every decoder graph family and
chunk count, and the oracle itself is pinned by hand-worked 8B values and the
closed-form tiling properties. Host only (no GPU)."""
import ctypes as C

import pytest

import synth
from oracle import schedule as OS


@pytest.fixture(scope="module")
def mods():
    from paper_2604_10180_b200 import decoder as DEC, _kd as K
    from paper_2604_10180_b200.api import Plan
    return DEC, K, Plan


def _names(K):
    return {getattr(K, n): n[len("KD_OP_"):] for n in dir(K) if n.startswith("KD_OP_")}


def _oracle_kernels(K, g):
    names = _names(K)
    out = []
    for op, reads, writes, attrs in g.decl:
        a = {f: getattr(attrs, f) for f, _ in attrs._fields_} if attrs is not None else {}
        out.append((names[op], a, [tuple(r) for r in reads], [tuple(w) for w in writes]))
    return out


def _check(DEC, K, Plan, dg, assign, n_dev, n_micro, n_chunks):
    plan = Plan(dg.g, DEC.b200_machine(n_dev), assign, n_micro, n_chunks)
    xs = plan.transfers()
    lib = plan.chunks()
    repl = {b for b, f in enumerate(dg.g._buf_flags) if f & K.KD_BUF_REPLICATED}
    ref = OS.chunk_table(_oracle_kernels(K, dg.g), dg.g.edges(), assign, xs, n_chunks, repl)
    flat = [(t, c, cm, r0, rows, rb, u, b, e) for t, (cm, r0, rows, rb, u, chs) in enumerate(ref)
            for c, (b, e) in enumerate(chs)]
    assert lib == flat
    return xs, ref


CASES = [
    ("tiny", lambda DEC: DEC.DecoderGraph(synth.TINY), "role", 2),
    ("tiny_gqa", lambda DEC: DEC.DecoderGraph(synth.TINY.with_(n_kv_heads=2, n_micro=2, context=77)), "role", 2),
    ("8b", lambda DEC: DEC.DecoderGraph(synth.LLAMA8B.with_(n_layers=2, n_micro=2)), "role", 2),
    ("moe", lambda DEC: DEC.DecoderGraph(synth.TINY.with_(n_experts=4, top_k=2, n_micro=2)), "role", 2),
    ("hybrid", lambda DEC: DEC.DecoderGraph(synth.TINY_HYBRID), "role", 2),
    ("tp2", lambda DEC: DEC.TPDecoderGraph(synth.TINY.with_(n_kv_heads=4, n_micro=2), 2), "own", 4),
    ("sharded3", lambda DEC: DEC.ShardedKVDecoderGraph(synth.TINY.with_(n_micro=2), 2), "own", 3),
    ("role3", lambda DEC: DEC.RoleDecoderGraph(synth.TINY.with_(n_micro=2, batch=4), 3), "own", 4),
    ("role7_8b", lambda DEC: DEC.RoleDecoderGraph(synth.LLAMA8B.with_(n_layers=1, batch=64, n_micro=2), 7), "own", 8),
    ("moe_ep", lambda DEC: DEC.MoEEPDecoderGraph(synth.TINY.with_(n_experts=4, top_k=2, n_micro=2, batch=4), 2, 2),
     "own", 4),
    ("repl_kv", lambda DEC: DEC.DecoderGraph(synth.TINY.with_(n_micro=2), replicate_kv=True), "repl", 3),
]


@pytest.mark.parametrize("name,make,kind,n_dev", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("n_chunks", [1, 2, 3, 4, 8])
def test_chunk_table_bit_exact_vs_oracle(mods, name, make, kind, n_dev, n_chunks):
    DEC, K, Plan = mods
    dg = make(DEC)
    if kind == "role":
        assign = dg.role_assign(0, 1)
    elif kind == "repl":  # RoPE/append apart from attention (delta-replicated KV)
        assign = [{DEC.T_ATTN: 2}.get(k.template, 0 if k.template in DEC.MEMORY_ROLE else 1) for k in dg.kernels]
    else:
        assign = dg.assign()
    _check(DEC, K, Plan, dg, assign, n_dev, dg.cfg.n_micro, n_chunks)


def test_scatter_rows_hand_values(mods):
    """3:1 layout (m = 2 rows per shard): the QKV GEMM's output (a·m = 6 rows)
    travels to shard s as rows [2s, 2s + 2) only; the shards' norm outputs
    (their own 2 rows) travel whole to the GEMM device."""
    DEC, K, Plan = mods
    dg = DEC.RoleDecoderGraph(synth.TINY.with_(n_micro=2, batch=4), 3)
    xs, ref = _check(DEC, K, Plan, dg, dg.assign(), 4, 2, 4)
    name = {k.kid: k.name for k in dg.kernels}
    seen = 0
    for (i, prod, dst, nbytes, *_), (cm, r0, rows, rb, u, chs) in zip(xs, ref):
        if name[prod] == "qkv":
            assert (cm, r0, rows) == (1, 2 * dst, 2) and nbytes == 2 * rb
            seen += 1
        if name[prod].startswith("norm1."):
            assert (r0, rows) == (0, 2)
    assert seen == 3 * 2 * 2  # 3 shards x 2 micro-batches x 2 layers


def test_chunk_table_8b_hand_values(mods):
    """Hand-worked 8B pair (m = 32, N = 2, n_chunks = 4), per cut edge of layer
    1: row bytes and unit from the model shape (H 4096, 32/8 heads × 128, F
    14336) and the consumer's axis:
      h1 → QKV GEMM:   row 8192 B, unit 256 (k-block 128 cols) → 4 × 2048
      qkv → RoPE:      row 12288 B, unit (4+2)·128·2 = 1536 (kv group) → 4 × 3072 (2 groups)
      attn → O GEMM:   row 8192, unit 256 → 4 × 2048 (2 kv heads' 8 q-heads each)
      o → norm2:       row 8192, unit 16 → 4 × 2048
      gu → SiLU:       row 57344, unit 256 (gate+up block) → 4 × 14336
      a → down GEMM:   row 28672, unit 256 → 4 × 7168
    (every transfer: COUNT mode, rows = 32)."""
    DEC, K, Plan = mods
    cfg = synth.LLAMA8B.with_(n_layers=2, n_micro=2)
    dg = DEC.DecoderGraph(cfg)
    assign = dg.role_assign(0, 1)
    xs, ref = _check(DEC, K, Plan, dg, assign, 2, 2, 4)
    name = {k.kid: k.name for k in dg.kernels}
    layer = {k.kid: k.layer for k in dg.kernels}
    hand = {"norm1": (8192, 256, 2048), "qkv": (12288, 1536, 3072), "attn": (8192, 256, 2048),
            "o": (8192, 16, 2048), "gu": (57344, 256, 14336), "silu": (28672, 256, 7168)}
    seen = set()
    for (i, prod, dst, *_), (cm, r0, rows, rb, u, chs) in zip(xs, ref):
        nm = name[prod]
        if layer[prod] != 1 or nm not in hand:
            continue
        rb_h, u_h, q_h = hand[nm]
        assert (cm, r0, rows, rb, u) == (1, 0, 32, rb_h, u_h), nm
        assert chs == [(c * q_h, (c + 1) * q_h) for c in range(4)], nm
        seen.add(nm)
    assert seen == set(hand)


@pytest.mark.parametrize("length,unit,n", [(8192, 256, 4), (12288, 1536, 4), (57344, 256, 3), (100, 16, 8),
                                           (4096, 4096, 4), (28672, 256, 5), (1536, 1536, 8)])
def test_chunks_tile_the_row(length, unit, n):
    """Closed form (R10): ascending, disjoint, tiling [0, length), every
    boundary but the last a multiple of the unit, count = ⌈U/⌈U/n⌉⌉."""
    ch = OS.chunks(length, unit, n)
    assert ch[0][0] == 0 and ch[-1][1] == length
    for (a, b), (c, d) in zip(ch, ch[1:]):
        assert b == c and a < b
    assert all(b % unit == 0 for _, b in ch[:-1])
    U = -(-length // unit)
    assert len(ch) == -(-U // -(-U // n))


def test_cta_mode_for_irregular_producers(mods):
    """MoE dispatch writes [meta | xg] and the grouped GEMM a dynamic row set:
    their transfers are one CTA-released chunk covering the whole output."""
    DEC, K, Plan = mods
    dg = DEC.DecoderGraph(synth.TINY.with_(n_experts=4, top_k=2, n_micro=2))
    plan = Plan(dg.g, DEC.b200_machine(2), dg.role_assign(0, 1), 2, 4)
    ops = {k.kid: k.name for k in dg.kernels}
    xs = plan.transfers()
    by_t = {}
    for t, c, cm, r0, rows, rb, u, b, e in plan.chunks():
        by_t.setdefault(t, []).append((cm, b, e, rb))
    for t, (i, prod, dst, nbytes, *_) in enumerate(xs):
        if ops[prod] in ("dispatch", "gu", "down"):
            assert by_t[t] == [(0, 0, by_t[t][0][3], by_t[t][0][3])]


@pytest.mark.parametrize("name,make,kind,n_dev", [c for c in CASES if c[0] in ("tiny", "role3", "moe_ep", "tp2")],
                         ids=["tiny", "tp2", "role3", "moe_ep"])
def test_workspace_layout_partition(mods, name, make, kind, n_dev):
    """kd_plan_workspace_layout (the poisoning range of tests/test_gpu_race.py):
    ctrl | flags | log | scratch | internal buffers, contiguous and 256-byte
    aligned, ending at kd_plan_workspace_bytes; the flags hold one u64 per
    chunk (+ the residency word) of every incoming transfer."""
    DEC, K, Plan = mods
    dg = make(DEC)
    assign = dg.role_assign(0, 1) if kind == "role" else dg.assign()
    plan = Plan(dg.g, DEC.b200_machine(n_dev), assign, dg.cfg.n_micro, 4)
    chunks = plan.chunks()
    xs = plan.transfers()
    for d in range(n_dev):
        L = plan.workspace_layout(d)
        assert L["ctrl_off"] == 0
        for a, b in (("ctrl", "flags"), ("flags", "log"), ("log", "scratch")):
            assert L[f"{b}_off"] == L[f"{a}_off"] + L[f"{a}_bytes"]
        assert L["act_off"] == L["scratch_off"] + L["scratch_bytes"]
        assert L["act_off"] <= L["total"] == plan.workspace_bytes(d)
        assert all(L[k] % 256 == 0 for k in L if k.endswith("_off"))
        incoming = [t for t, x in enumerate(xs) if x[2] == d]
        need = sum(1 + sum(1 for c in chunks if c[0] == t) for t in incoming)
        assert L["flags_bytes"] >= 8 * need
