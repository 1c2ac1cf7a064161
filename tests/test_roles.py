"""Device-role search (SURVEY §8(a) a1 "search over device roles (a memory-
bound-role GPUs : g GEMM-role GPUs, a+g ∈ {2,4,8}) … N ∈ {1,2,4}"; E6,
P:330-334): kd_place_roles is bit-exact against the oracle's plain
exhaustive enumeration (oracle.placement.place_roles), and the oracle is
pinned by a hand-worked two-kernel example. Host only."""
import random

import pytest

import synth
from oracle import placement as OP


@pytest.fixture(scope="module")
def api():
    from paper_2604_10180_b200 import api as A, _kd as K, decoder as DEC
    return A, K, DEC


def _oracle(A, K, g, m, rows, max_gpus, mask):
    kernels, flops, tmpl, pins = [], [], [], []
    for op, reads, writes, attrs in g.decl:
        kernels.append(([tuple(r) for r in reads], [tuple(w) for w in writes]))
    # the graph's kernel descriptors (flops, templates, pins) as declared
    for kd in g._desc:
        flops.append(kd[0])
        tmpl.append(kd[1])
        pins.append(kd[2])
    weights = {b for b, f in enumerate(g._buf_flags) if f & K.KD_BUF_WEIGHT}
    mm = m.py
    return OP.place_roles(kernels, flops, tmpl, pins, weights, g.edges(), mm["hbm"], mm["tc"], mm["bw"], mm["lat"],
                          mm["launch"], rows, max_gpus, mask)


def _compare(A, K, g, m, rows, max_gpus=8, mask=0b111):
    lib = A.place_roles(g, m, rows, max_gpus, mask)
    ref = _oracle(A, K, g, m, rows, max_gpus, mask)
    assert len(lib) == len(ref)
    for L, R in zip(lib, ref):
        assert (L["gpus"], L["a"], L["gr"], L["n_micro"], L["period_ps"], L["T_mem_ps"], L["T_gemm_ps"], L["M_mem_ps"],
                L["M_gemm_ps"], L["tokens_per_step"], L["role_mask"], L["roles"]) == tuple(R)
    return lib


def test_roles_hand_worked_two_kernel_chain(api):
    """k0 (memory-like): reads 10 000 B of state, writes X (100 B); k1
    (GEMM-like): reads X and a 10 000 B weight, writes Y (100 B). 1 B/ps HBM
    and link, no latency or launch floor, 1 row per micro-batch:
      n=1: mono, N=1, period 10100 + 10200 = 20300;
      n=2: 1:1, N=2, k0 in the GEMM role (mask 1; ties with mask 2 keep the
           first): T_mem = 2·10200, T_gemm = 2·10100, M_mem = 2·100 → 20400;
      n=4: 3:1, N=2, mask 2: T_gemm = 2·(10000 + 3·200) = 21200, T_mem =
           2·10100, M_gemm = 2·3·100 → period 21200, 6 tokens;
      n=8: 7:1, N=2, mask 2: T_gemm = 2·(10000 + 7·200) = 22800, T_mem =
           20200, M_gemm = 1400 → 14 tokens (beats 6:2's 12 / 20200)."""
    A, K, DEC = api
    g = A.Graph()
    st = g.add_buffer(10000, 0)
    x = g.add_buffer(100, K.KD_BUF_PER_MICROBATCH)
    w = g.add_buffer(10000, K.KD_BUF_WEIGHT)
    y = g.add_buffer(100, K.KD_BUF_PER_MICROBATCH | K.KD_BUF_OUTPUT)
    g.add_kernel(K.KD_OP_NONE, [(st, 0, 10000)], [(x, 0, 100)], None, 0, -1, 0)
    g.add_kernel(K.KD_OP_NONE, [(x, 0, 100), (w, 0, 10000)], [(y, 0, 100)], None, 0, -1, 1)
    g.finalize()
    m = A.Machine.uniform(8, 10 ** 12, 10 ** 30, 10 ** 12, 0, 0)
    lib = _compare(A, K, g, m, 1)
    got = [(L["gpus"], L["a"], L["gr"], L["n_micro"], L["period_ps"], L["T_mem_ps"], L["T_gemm_ps"], L["M_mem_ps"],
            L["M_gemm_ps"], L["tokens_per_step"], L["role_mask"]) for L in lib]
    assert got == [(1, 1, 0, 1, 20300, 20300, 0, 0, 0, 1, 0),
                   (2, 1, 1, 2, 20400, 20400, 20200, 200, 0, 2, 1),
                   (4, 3, 1, 2, 21200, 20200, 21200, 0, 600, 6, 2),
                   (8, 7, 1, 2, 22800, 20200, 22800, 0, 1400, 14, 2)]


@pytest.mark.parametrize("cfg_name", ["tiny", "8b", "moe", "hybrid"])
def test_roles_decoder_graphs_bit_exact(api, cfg_name):
    A, K, DEC = api
    cfg = {"tiny": synth.TINY, "8b": synth.LLAMA8B.with_(n_layers=2, batch=32, n_micro=1),
           "moe": synth.TINY.with_(n_experts=4, top_k=2, n_micro=2),
           "hybrid": synth.TINY_HYBRID}[cfg_name]
    dg = DEC.DecoderGraph(cfg)
    _compare(A, K, dg.g, DEC.b200_machine(8), cfg.m)


def test_roles_8b_picks_more_than_two_gpus_where_it_pays(api):
    """SURVEY §8(d) ceilings: at the 8B shape with 32 rows per micro-batch a
    memory-heavy ratio (3:1 at 4 GPUs, 7:1 at 8) with N = 2 gives more tokens
    per GPU than the 1:1 pair, and beats monolithic per GPU at 8 GPUs."""
    A, K, DEC = api
    cfg = synth.LLAMA8B.with_(n_layers=2, batch=32, n_micro=1)
    dg = DEC.DecoderGraph(cfg)
    lib = {L["gpus"]: L for L in A.place_roles(dg.g, DEC.b200_machine(8), cfg.m)}
    per_gpu = {n: L["tokens_per_step"] / (n * L["period_ps"]) for n, L in lib.items()}
    assert lib[4]["a"] == 3 and lib[8]["a"] == 7 and lib[8]["n_micro"] >= 2
    assert per_gpu[8] > per_gpu[2] and per_gpu[8] > per_gpu[1]
    names = [k.name for k in dg.kernels]
    roles8 = lib[8]["roles"]
    assert all(roles8[i] == 1 for i, n in enumerate(names) if n in ("qkv", "o", "gu", "down"))
    assert all(roles8[i] == 0 for i, n in enumerate(names) if n in ("attn", "rope"))


@pytest.mark.parametrize("seed", range(12))
def test_roles_random_graphs_bit_exact(api, seed):
    A, K, DEC = api
    rnd = random.Random(seed)
    nb = rnd.randint(2, 6)
    g = A.Graph()
    sz = [rnd.randint(64, 4096) for _ in range(nb)]
    flags = [K.KD_BUF_WEIGHT if rnd.random() < 0.3 else 0 for _ in range(nb)]
    ids = [g.add_buffer(s, f) for s, f in zip(sz, flags)]
    nk = rnd.randint(2, 9)
    for k in range(nk):
        def span():
            i = rnd.randrange(nb)
            a = rnd.randrange(sz[i])
            return (ids[i], a, rnd.randint(1, sz[i] - a))
        reads = [span() for _ in range(rnd.randint(1, 3))]
        writes = [s for s in (span() for _ in range(rnd.randint(1, 2))) if not flags[ids.index(s[0])]]
        if not writes:  # writes never target a weight buffer
            writes = [(ids[flags.index(0)], 0, 8)] if 0 in flags else [span()]
        tm = rnd.choice([-1, -1, 0, 1, 2])
        pin = rnd.choice([-1, -1, -1, 0, 1]) if tm == -1 else -1
        g.add_kernel(K.KD_OP_NONE, reads, writes, None, rnd.randint(0, 10 ** 7), pin, tm)
    g.finalize()
    m = A.Machine.uniform(8, 6 * 10 ** 12, 10 ** 15, 8 * 10 ** 11, rnd.randint(0, 5000), rnd.randint(0, 3000))
    _compare(A, K, g, m, rnd.randint(1, 64), rnd.choice([1, 2, 4, 8]), rnd.choice([1, 2, 3, 5, 7]))
