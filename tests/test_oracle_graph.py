"""Pins for oracle/ddg.py, oracle/placement.py, oracle/schedule.py against the
worked examples in tests/golden/spec_examples.json, brute force and invariants
(SURVEY §8(c) pins: DAG, placement, schedule, chunks). CPU only."""
import json
import os
import random

import pytest

from oracle import ddg, placement as PL, schedule as SC

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
PS = 10 ** 12


def rand_trace(rng, K, nbuf=4, maxlen=48):
    ks = []
    for _ in range(K):
        def spans(n):
            out = []
            for _ in range(n):
                b = rng.randrange(nbuf)
                o = rng.randrange(maxlen - 1)
                out.append((b, o, rng.randrange(1, maxlen - o + 1)))
            return out
        ks.append((spans(rng.randrange(0, 3)), spans(rng.randrange(0, 3))))
    return ks


# ------------------------------------------------------------------ DDG
def test_spec_ddg_examples():
    for key in ("ddg_single_edge", "ddg_most_recent_writer"):
        ex = GOLD[key]
        ks = [([tuple(s) for s in r], [tuple(s) for s in w]) for r, w in ex["kernels"]]
        assert [list(e) for e in ddg.build_ddg(ks)] == ex["edges"], ex["cite"]


@pytest.mark.parametrize("seed", range(40))
def test_registry_equals_per_byte_bruteforce(seed):
    rng = random.Random(seed)
    ks = rand_trace(rng, rng.randrange(1, 30))
    assert ddg.build_ddg(ks) == ddg.brute_force_ddg(ks)


def test_ddg_invariants_and_in_place():
    rng = random.Random(123)
    for _ in range(20):
        ks = rand_trace(rng, 25)
        e1 = ddg.build_ddg(ks)
        assert e1 == ddg.build_ddg(ks)                 # idempotent
        assert all(s < d for s, d, *_ in e1)           # forward, acyclic, no self edges
    # in-place kernel (reads and writes the same bytes): edge from the previous writer only
    ks = [([], [(0, 0, 8)]), ([(0, 0, 8)], [(0, 0, 8)]), ([(0, 0, 8)], [])]
    assert ddg.build_ddg(ks) == [(0, 1, 0, 0, 8), (1, 2, 0, 0, 8)]
    # WAR / WAW produce no edges; unwritten (weight) bytes produce no edges
    ks = [([(1, 0, 4)], []), ([], [(1, 0, 4)]), ([], [(1, 0, 4)])]
    assert ddg.build_ddg(ks) == []


# ------------------------------------------------------------------ placement
def _machine(n, bw=1, lat=0, hbm=10 ** 12, tc=10 ** 15, launch=0):
    return PL.Machine(n, [hbm] * n, [tc] * n, [[bw] * n for _ in range(n)],
                      [[lat] * n for _ in range(n)], launch)


def _objective_from_table(t, dij, m, N):
    K = len(t)
    best = None
    import itertools
    for a in itertools.product(range(m.n_dev), repeat=K):
        o, _, _ = PL.objective(list(a), t, dij, m, N)
        if best is None or o < best[1]:
            best = (list(a), o)
    return best


def test_spec_placement_examples():
    ex = GOLD["place_independent"]
    t = [[x * PS for x in row] for row in ex["t_s"]]
    a, o = _objective_from_table(t, {}, _machine(2), 2)
    assert a == ex["assign"] and o == 2 * ex["objective_s"] * PS   # per step = N x per micro-batch
    ex = GOLD["place_colocate"]
    m = _machine(2, bw=PS, lat=int(ex["edge_cost_s"] * PS) - PS)  # 1 byte edge: l + 1 s = 5 s
    a, o = _objective_from_table([[x * PS for x in r] for r in ex["t_s"]], {(0, 1): 1}, m, 2)
    assert a in ex["assign_options"] and o == 2 * ex["objective_s"] * PS


def test_linearization_counts_and_identity():
    ex = GOLD["milp_counts"]
    K, G, E = ex["K"], ex["G"], ex["E"]
    assert K * G == ex["x_vars"] and E * G * (G - 1) == ex["y_vars"]
    # y^{u,g}_{ij} = x_{i,u} x_{j,g}: exactly one (u,g) pair is "on" per edge; it is cut iff u != g
    import itertools
    for a in itertools.product(range(G), repeat=K):
        for (i, j) in [(0, 1), (1, 2)]:
            ys = [(u, g) for u in range(G) for g in range(G) if u != g and a[i] == u and a[j] == g]
            assert len(ys) == (1 if a[i] != a[j] else 0)


def _rand_problem(rng, K, n):
    ks = rand_trace(rng, K, nbuf=3, maxlen=40)
    flops = [rng.randrange(0, 100) for _ in range(K)]
    edges = ddg.build_ddg(ks)
    m = PL.Machine(n, [rng.randrange(1, 50) for _ in range(n)], [rng.randrange(1, 50) for _ in range(n)],
                   [[rng.randrange(1, 20) for _ in range(n)] for _ in range(n)],
                   [[rng.randrange(0, 10 ** 12) for _ in range(n)] for _ in range(n)], rng.randrange(0, 10 ** 11))
    return ks, flops, edges, m


@pytest.mark.parametrize("seed", range(12))
def test_template_enumeration_equals_all_assignments_without_templates(seed):
    rng = random.Random(seed)
    K, n = rng.randrange(2, 8), rng.randrange(1, 4)
    ks, flops, edges, m = _rand_problem(rng, K, n)
    for N in (1, 2):
        a1 = PL.place_exhaustive(ks, flops, [-1] * K, [-1] * K, edges, m, N)
        a2 = PL.place_all_assignments(ks, flops, edges, m, N)
        assert a1 == a2


def test_objective_audit_and_single_gpu():
    rng = random.Random(5)
    ks, flops, edges, m = _rand_problem(rng, 6, 1)
    t = [[PL.kernel_time_ps(k, f, m, 0)] for k, f in zip(ks, flops)]
    a, o = PL.place_exhaustive(ks, flops, [-1] * 6, [-1] * 6, edges, m, 1)
    assert a == [0] * 6 and o == sum(x[0] for x in t)          # S:277 degenerate case


def test_bandwidth_monotone_and_slow_link_degeneracy():
    rng = random.Random(9)
    for _ in range(6):
        ks, flops, edges, m = _rand_problem(rng, 6, 2)
        prev = None
        for scale in (1, 4, 64, 10 ** 6):
            m2 = PL.Machine(2, m.hbm_Bps, m.tc_flops, [[b * scale for b in r] for r in m.link_Bps], m.link_lat_ps, m.launch_ps)
            _, o = PL.place_exhaustive(ks, flops, [-1] * 6, [-1] * 6, edges, m2, 2)
            assert prev is None or o <= prev
            prev = o
        # comm cost -> infinity: the latency objective uses one GPU when any edge exists
        m3 = PL.Machine(2, [7, 7], [7, 7], [[1, 1], [1, 1]], [[10 ** 30] * 2] * 2, 0)
        a, _ = PL.place_exhaustive(ks, flops, [-1] * 6, [-1] * 6, edges, m3, 1)
        if edges:
            assert len(set(a[s] for s, *_ in edges) | set(a[d] for _, d, *_ in edges)) == 1


def test_templates_and_pins_respected():
    rng = random.Random(3)
    ks, flops, edges, m = _rand_problem(rng, 8, 3)
    tmpl = [0, 1, 2, 3, 0, 1, 2, 3]
    pins = [-1, -1, 2, -1, -1, -1, -1, -1]
    a, _ = PL.place_exhaustive(ks, flops, tmpl, pins, edges, m, 2)
    assert a[2] == a[6] == 2 and a[0] == a[4] and a[1] == a[5] and a[3] == a[7]
    with pytest.raises(ValueError):
        PL.place_exhaustive(ks, flops, tmpl, [0, -1, -1, -1, 1, -1, -1, -1], edges, m, 2)


# ------------------------------------------------------------------ schedule
def test_spec_schedule_chain_latency():
    ex = GOLD["sched_chain"]
    # two kernels, k0 -> k1 via a 1-byte edge whose transfer takes 0.5 s
    m = PL.Machine(2, [1] * 2, [1] * 2, [[PS] * 2] * 2, [[int(ex["transfer_s"] * PS) - 1] * 2] * 2, 0)
    edges = [(0, 1, 0, 0, 1)]
    ent = SC.list_schedule(2, [int(x * PS) for x in ex["t_s"]], [0, 1], edges, m, 1)
    assert max(e[4] for e in ent) == int(ex["latency_s"] * PS)
    # all on one GPU: sum of t
    ent = SC.list_schedule(2, [PS, PS], [0, 0], edges, m, 1)
    assert max(e[4] for e in ent) == 2 * PS


def _check_schedule(K, t, assign, edges, m, N, ent):
    start = {(i, k): s for d, i, k, s, e in ent}
    endt = {(i, k): e for d, i, k, s, e in ent}
    assert len(ent) == K * N
    xfer = SC.transfers_of(edges, assign)
    for s, d, *_ in edges:                               # causality
        for i in range(N):
            lag = 0
            if assign[s] != assign[d]:
                u, g = assign[s], assign[d]
                lag = m.link_lat_ps[u][g] + PL.ceil_div(xfer[(s, g)] * PS, m.link_Bps[u][g])
            assert start[(i, d)] >= endt[(i, s)] + lag
    for dev in range(m.n_dev):                           # one kernel at a time
        mine = sorted((s, e) for d, i, k, s, e in ent if d == dev)
        for (s0, e0), (s1, e1) in zip(mine, mine[1:]):
            assert s1 >= e0
    seen = set()                                         # global order is topological
    for d, i, k, s, e in ent:
        for src, dst, *_ in edges:
            if dst == k:
                assert (i, src) in seen
        seen.add((i, k))


@pytest.mark.parametrize("seed", range(10))
def test_schedule_causality_and_work_conservation(seed):
    rng = random.Random(seed)
    K, n, N = rng.randrange(2, 10), rng.randrange(1, 4), rng.randrange(1, 5)
    ks, flops, edges, m = _rand_problem(rng, K, n)
    assign = [rng.randrange(n) for _ in range(K)]
    t = [PL.kernel_time_ps(ks[k], flops[k], m, assign[k]) + 1 for k in range(K)]
    ent = SC.list_schedule(K, t, assign, edges, m, N)
    _check_schedule(K, t, assign, edges, m, N, ent)
    # work conservation: with no edges nothing ever waits
    ent = SC.list_schedule(K, t, assign, [], m, N)
    for dev in range(n):
        ends = sorted(e for d, i, k, s, e in ent if d == dev)
        if ends:
            assert ends[-1] == N * sum(t[k] for k in range(K) if assign[k] == dev)


def test_bottleneck_law_pipelined_chain():
    # balanced two-stage alternating chain, transfers cheaper than compute:
    # steady state per micro-batch -> max_g W_g
    K = 6
    assign = [0, 1, 0, 1, 0, 1]
    t = [10 * PS] * K
    edges = [(k, k + 1, 0, 0, 1) for k in range(K - 1)]
    m = PL.Machine(2, [1] * 2, [1] * 2, [[PS] * 2] * 2, [[2 * PS - 1] * 2] * 2, 0)
    N = 64
    ent = SC.list_schedule(K, t, assign, edges, m, N)
    mk = max(e[4] for e in ent)
    W = max(sum(t[k] for k in range(K) if assign[k] == g) for g in range(2))
    assert mk <= 1.05 * N * W
    # no pipelining (N=1) is the serial sum
    ent1 = SC.list_schedule(K, t, assign, edges, m, 1)
    assert max(e[4] for e in ent1) == sum(t) + (K - 1) * 2 * PS


def test_chunks_closed_form():
    for length in (1, 63, 64, 65, 4096, 10000):
        for unit in (1, 16, 64):
            for n in (1, 2, 3, 4, 7):
                cs = SC.chunks(length, unit, n)
                assert cs[0][0] == 0 and cs[-1][1] == length
                assert all(a < b for a, b in cs)
                assert all(b0 == a1 for (_, b0), (a1, _) in zip(cs, cs[1:]))
                assert all(a % unit == 0 for a, _ in cs)
                U = -(-length // unit)
                q = -(-U // n)
                # count = ceil(U / ceil(U / n)) (<= min(n, U); SURVEY's "= min(n, U)" is
                # not what its own formula yields, e.g. U=4, n=3 -> 2 chunks; R10)
                assert len(cs) == -(-U // q) <= min(n, U)
                assert all(b - a == q * unit for a, b in cs[:-1])
