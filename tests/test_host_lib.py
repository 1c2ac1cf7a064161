"""CPU tests of the C-ABI library (no GPU needed): it loads, exports every
symbol include/kd.h declares, and its host half (DAG, cost, placement,
schedule, chunks) is bit-exact against the independent oracle."""
import os
import random
import re

import pytest

from oracle import ddg as OD, placement as OP, schedule as OS

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def kd():
    import paper_2604_10180_b200 as pkg
    from paper_2604_10180_b200 import _kd, api
    return pkg, _kd, api


def test_library_loads_and_exports_header_symbols(kd):
    _, K, _ = kd
    hdr = open(os.path.join(ROOT, "include", "kd.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    declared = set(re.findall(r"\b(kd_[a-z0-9_]+)\s*\(", hdr))
    assert len(declared) >= 40
    missing = [s for s in sorted(declared) if not hasattr(K.lib, s)]
    assert not missing, missing
    assert set(K.EXPORTED) == declared, set(K.EXPORTED) ^ declared
    assert K.lib.kd_version() >= 1


def test_error_paths(kd):
    _, K, api = kd
    g = api.Graph()
    b = g.add_buffer(64, K.KD_BUF_WEIGHT)
    with pytest.raises(K.KdError) as e:
        g.add_kernel(K.KD_OP_NONE, [(b, 60, 8)], [])
    assert e.value.status == K.KD_ERR_RANGE
    with pytest.raises(K.KdError) as e:
        g.add_kernel(K.KD_OP_NONE, [(b, 0, 0)], [])
    assert e.value.status == K.KD_ERR_INVALID_ARG
    with pytest.raises(K.KdError) as e:
        g.add_kernel(K.KD_OP_NONE, [], [(b, 0, 8)])       # writes a weight
    assert e.value.status == K.KD_ERR_INVALID_ARG
    with pytest.raises(K.KdError) as e:
        g.edges()
    assert e.value.status == K.KD_ERR_STATE
    g.finalize()
    with pytest.raises(K.KdError) as e:
        g.add_buffer(8)
    assert e.value.status == K.KD_ERR_STATE


def test_fused_norm_op_host_checks(kd):
    """KD_OP_GEMM_RMSNORM host side: scratch sizing (barrier words + per-CTA
    partial sums), dtype validation before any device work, the graph accepts
    the op id and its 4-read / 2-write declaration."""
    _, K, api = kd
    a = K.kd_attr_gemm_rmsnorm(64, 4096, 4096, K.KD_BF16, 1e-5, 0)
    assert api.op_scratch_bytes(K.KD_OP_GEMM_RMSNORM, a) == 64 * 1024 + 64 * 160 * 4
    bad = K.kd_attr_gemm_rmsnorm(64, 4096, 4096, K.KD_F32, 1e-5, 0)
    import ctypes as C
    assert K.kd_op_gemm_rmsnorm(C.byref(bad), None, None, None, None, None, None, None) == K.KD_ERR_UNSUPPORTED
    g = api.Graph()
    X, W, r, gam, h = (g.add_buffer(n, f) for n, f in ((64, 0), (64, K.KD_BUF_WEIGHT), (64, 0),
                                                       (16, K.KD_BUF_WEIGHT), (32, 0)))
    g.add_kernel(K.KD_OP_GEMM_RMSNORM, [(X, 0, 64), (W, 0, 64), (r, 0, 64), (gam, 0, 16)], [(h, 0, 32), (r, 0, 64)], a)
    with pytest.raises(K.KdError):
        g.add_kernel(K.KD_OP_PREFILL_ATTENTION + 1, [], [(h, 0, 8)])  # (the highest op id + 1)
    g.finalize()


def rand_trace(rng, K_, nbuf=4, maxlen=48):
    ks = []
    for _ in range(K_):
        def spans(n):
            out = []
            for _ in range(n):
                b = rng.randrange(nbuf)
                o = rng.randrange(maxlen - 1)
                out.append((b, o, rng.randrange(1, maxlen - o + 1)))
            return out
        ks.append((spans(rng.randrange(0, 3)), spans(rng.randrange(0, 3))))
    return ks


def lib_graph(api, ks, nbuf=4, maxlen=48, flops=None, templates=None, pins=None):
    g = api.Graph()
    for _ in range(nbuf):
        g.add_buffer(maxlen)
    for k, (r, w) in enumerate(ks):
        g.add_kernel(0, r, w, flops=(flops[k] if flops else 0), template=(templates[k] if templates else -1),
                     pin=(pins[k] if pins else -1))
    g.finalize()
    return g


@pytest.mark.parametrize("seed", range(60))
def test_ddg_bit_exact_vs_oracle(kd, seed):
    _, _, api = kd
    rng = random.Random(1000 + seed)
    ks = rand_trace(rng, rng.randrange(1, 40))
    g = lib_graph(api, ks)
    assert g.edges() == OD.build_ddg(ks)


def rand_machine(rng, n, homog=False):
    if homog:
        return OP.Machine(n, [rng.randrange(1, 50)] * n, [rng.randrange(1, 50)] * n,
                          [[7] * n for _ in range(n)], [[rng.randrange(0, 10 ** 12)] * n for _ in range(n)],
                          rng.randrange(0, 10 ** 11))
    return OP.Machine(n, [rng.randrange(1, 50) for _ in range(n)], [rng.randrange(1, 50) for _ in range(n)],
                      [[rng.randrange(1, 20) for _ in range(n)] for _ in range(n)],
                      [[rng.randrange(0, 10 ** 12) for _ in range(n)] for _ in range(n)], rng.randrange(0, 10 ** 11))


def to_lib_machine(api, m):
    return api.Machine(m.hbm_Bps, m.tc_flops, m.link_Bps, m.link_lat_ps, m.launch_ps)


@pytest.mark.parametrize("seed", range(40))
def test_cost_objective_place_bit_exact(kd, seed):
    _, K, api = kd
    rng = random.Random(2000 + seed)
    K_ = rng.randrange(2, 9)
    n = rng.randrange(1, 4)
    ks = rand_trace(rng, K_, nbuf=3, maxlen=40)
    flops = [rng.randrange(0, 100) for _ in range(K_)]
    templates = [rng.choice([-1, 0, 1, 2]) for _ in range(K_)]
    pins = [rng.choice([-1, -1, -1, rng.randrange(n)]) for _ in range(K_)]
    om = rand_machine(rng, n, homog=(seed % 3 == 0))
    lm = to_lib_machine(api, om)
    edges = OD.build_ddg(ks)
    g = lib_graph(api, ks, 3, 40, flops, templates, pins)
    t = api.cost(g, lm)
    assert t == [[OP.kernel_time_ps(ks[k], flops[k], om, d) for d in range(n)] for k in range(K_)]
    for N in (1, 2, 4):
        assign = [rng.randrange(n) for _ in range(K_)]
        o, T, M = api.objective(g, lm, assign, N)
        oo, oT, oM = OP.objective(assign, t, OD.edge_bytes(edges), om, N)
        assert (o, T, M) == (oo, oT, oM)
        try:
            ref = OP.place_exhaustive(ks, flops, templates, pins, edges, om, N)
        except ValueError:
            with pytest.raises(K.KdError) as e:
                api.place(g, lm, N)
            assert e.value.status == K.KD_ERR_PIN_CONFLICT
            continue
        a, obj, _ = api.place(g, lm, N)
        assert (a, obj) == (ref[0], ref[1])


@pytest.mark.parametrize("seed", range(30))
def test_schedule_bit_exact(kd, seed):
    _, _, api = kd
    rng = random.Random(3000 + seed)
    K_ = rng.randrange(1, 12)
    n = rng.randrange(1, 4)
    N = rng.randrange(1, 5)
    ks = rand_trace(rng, K_, nbuf=3, maxlen=40)
    flops = [rng.randrange(0, 100) for _ in range(K_)]
    om = rand_machine(rng, n)
    lm = to_lib_machine(api, om)
    g = lib_graph(api, ks, 3, 40, flops)
    edges = OD.build_ddg(ks)
    assign = [rng.randrange(n) for _ in range(K_)]
    plan = api.Plan(g, lm, assign, N)
    t = [OP.kernel_time_ps(ks[k], flops[k], om, assign[k]) for k in range(K_)]
    ref = OS.list_schedule(K_, t, assign, edges, om, N)
    assert plan.schedule() == ref
    assert plan.makespan == max(e[4] for e in ref)
    xf = OS.transfers_of(edges, assign)
    got = {(p, d): b for (i, p, d, b, _, _) in plan.transfers() if i == 0}
    assert got == xf


def test_chunks_bit_exact(kd):
    _, _, api = kd
    for length in (1, 63, 64, 65, 4096, 10000, 1 << 20):
        for unit in (1, 16, 64, 128):
            for n in (1, 2, 3, 4, 7):
                assert api.chunks(length, unit, n) == OS.chunks(length, unit, n)
