"""Oracle — cost model, placement objective and exhaustive placement search
(test infrastructure only).

PAPER.md §3.2 "Policy Planner", equations numbered as in SURVEY:
  E1  Σ_g x_{k,g} = 1 — assign is a total map
  E2  T_g = Σ_k t_{k,g} x_{k,g}
  E3  M_g = Σ_{(i,j)∈E} Σ_{u≠g} c^{u,g}_{ij} y^{u,g}_{ij},
      y^{u,g}_{ij} = x_{i,u} x_{j,g}
  E4  c^{u,g}_{ij} = ℓ_{u,g} + d_ij / bw_{u,g}
  E5  W_g = max(T_g, M_g)
  E6  min max_g W_g  throughput policy
  E7  min Σ t x + Σ c y      latency policy

Readings: R7 integer picoseconds, ceil divisions, ties to the
lexicographically smallest assign; R8 with N micro-batches T_g and M_g are per
step = N × per-micro-batch sums; N = 1 has nothing to overlap inside a step so
its objective is the serial E7 sum; A10 the profiled t_{k,g} is replaced by a
roofline: t = max(⌈bytes·10¹²/HBM⌉, ⌈flops·10¹²/TC⌉) + launch floor, bytes =
the kernel's declared read+write span bytes (union per buffer); A15 repeated
layers share one placement (kernels with the same template id are
co-assigned); A4 pinned kernels keep their device.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

from .ddg import _union, edge_bytes

PS = 10 ** 12


@dataclass
class Machine:
    n_dev: int
    hbm_Bps: List[int]          # per device, bytes/s
    tc_flops: List[int]         # per device, flop/s
    link_Bps: List[List[int]]   # [u][g] bytes/s (diagonal unused)
    link_lat_ps: List[List[int]]
    launch_ps: int


def ceil_div(a: int, b: int) -> int:
    return -(-a // b)


def span_bytes(spans) -> int:
    return sum(e - s for ivs in _union(spans).values() for s, e in ivs)


def kernel_bytes(kernel) -> int:
    reads, writes = kernel[0], kernel[1]
    return span_bytes(reads) + span_bytes(writes)


def kernel_time_ps(kernel, flops: int, m: Machine, dev: int) -> int:
    """Roofline t_{k,g} in integer ps (A10, R7)."""
    b = kernel_bytes(kernel)
    return max(ceil_div(b * PS, m.hbm_Bps[dev]), ceil_div(flops * PS, m.tc_flops[dev])) + m.launch_ps


def edge_cost_ps(d_ij: int, m: Machine, u: int, g: int) -> int:
    """E4 in integer ps."""
    return m.link_lat_ps[u][g] + ceil_div(d_ij * PS, m.link_Bps[u][g])


def objective(assign: Sequence[int], t: Sequence[Sequence[int]],
              dij: Dict[Tuple[int, int], int], m: Machine, n_micro: int):
    """E2–E7 for a complete assignment. t[k][g] per-micro-batch kernel times;
    dij per-micro-batch edge bytes. Returns (objective, T[g], M[g])."""
    T = [0] * m.n_dev
    M = [0] * m.n_dev
    for k, g in enumerate(assign):
        T[g] += t[k][g]
    for (i, j), d in dij.items():
        u, g = assign[i], assign[j]
        if u != g:                       # y^{u,g}_{ij} = x_{i,u} x_{j,g} = 1
            M[g] += edge_cost_ps(d, m, u, g)
    T = [n_micro * x for x in T]
    M = [n_micro * x for x in M]
    if n_micro == 1:
        obj = sum(T) + sum(M)           # E7 (R8)
    else:
        obj = max(max(a, b) for a, b in zip(T, M))   # E5/E6
    return obj, T, M


def template_classes(templates: Sequence[int], pins: Sequence[int]):
    """Free classes in first-occurrence order and the fixed device of pinned
    classes. templates[k] = -1 means kernel k is its own class."""
    cls_of = []
    key_to_cls: Dict[Tuple, int] = {}
    for k, tid in enumerate(templates):
        key = ("t", tid) if tid >= 0 else ("k", k)
        if key not in key_to_cls:
            key_to_cls[key] = len(key_to_cls)
        cls_of.append(key_to_cls[key])
    ncls = len(key_to_cls)
    fixed: List[Optional[int]] = [None] * ncls
    for k, p in enumerate(pins):
        if p >= 0:
            c = cls_of[k]
            if fixed[c] is not None and fixed[c] != p:
                raise ValueError("pin conflict")
            fixed[c] = p
    return cls_of, fixed


def place_exhaustive(kernels, flops, templates, pins, edges, m: Machine, n_micro: int):
    """Plain exhaustive enumeration (C3): every device choice for every free
    class, in lexicographic order; the first strict minimum wins, which is the
    lexicographically smallest assign among optima (R7).
    Returns (assign, objective)."""
    K = len(kernels)
    t = [[kernel_time_ps(kernels[k], flops[k], m, g) for g in range(m.n_dev)] for k in range(K)]
    dij = edge_bytes(edges)
    cls_of, fixed = template_classes(templates, pins)
    free = [c for c in range(len(fixed)) if fixed[c] is None]
    best = None
    for choice in itertools.product(range(m.n_dev), repeat=len(free)):
        dev_of_cls = list(fixed)
        for c, g in zip(free, choice):
            dev_of_cls[c] = g
        assign = [dev_of_cls[cls_of[k]] for k in range(K)]
        obj, _, _ = objective(assign, t, dij, m, n_micro)
        if best is None or obj < best[1]:
            best = (assign, obj)
    return best


def place_all_assignments(kernels, flops, edges, m: Machine, n_micro: int):
    """Even plainer: all n^K assignments with no template/pin structure
    ("exhaustive enumeration … ≤12 kernels, ≤3 GPUs")."""
    K = len(kernels)
    t = [[kernel_time_ps(kernels[k], flops[k], m, g) for g in range(m.n_dev)] for k in range(K)]
    dij = edge_bytes(edges)
    best = None
    for assign in itertools.product(range(m.n_dev), repeat=K):
        obj, _, _ = objective(list(assign), t, dij, m, n_micro)
        if best is None or obj < best[1]:
            best = (list(assign), obj)
    return best


# ---------------------------------------------------------------- device-role search
def place_roles(kernels, flops, templates, pins, weight_bufs, edges, hbm: int, tc: int, link_Bps: int,
                link_lat_ps: int, launch_ps: int, rows: int, max_gpus: int, micro_mask: int):
    """Exhaustive device-role search: for every GPU count n in {1, 2, 4, 8}
    (n <= max_gpus), every split n = a memory-role + gr GEMM-role GPUs, every
    allowed N = 2^j (micro_mask bit j) and every memory/GEMM role of each
    free template class, evaluate the E6 step period of that layout and keep
    the most tokens per GPU-second (a·N·rows/(n·period)); ties keep the first
    in (a, N, mask) order. A memory-role kernel runs on each of the `a` GPUs
    over its own `rows` rows: t = max(⌈(W+A)·10¹²/hbm⌉, ⌈F·10¹²/tc⌉) + launch;
    a GEMM-role kernel runs once per micro-batch over a·rows rows with its
    weights split over the gr GPUs: t = max(⌈(⌈W/gr⌉ + a·A)·10¹²/hbm⌉,
    ⌈⌈a·F/gr⌉·10¹²/tc⌉) + launch (W = weight-span bytes, A = other bytes).
    A cut edge of d bytes costs, per micro-batch, a·(ℓ + ⌈d·10¹²/bw⌉) at the
    GEMM side (each GEMM GPU gathers every shard) or gr·(ℓ + ⌈⌈d/gr⌉·10¹²/bw⌉)
    at the memory side. Period = max(T_mem, T_gemm, M_mem, M_gemm)·… for
    N >= 2, their sum for N = 1 (R8). n = 1 is monolithic (a = 1, no GEMM
    role). pins: -1 free, 0 memory, 1 GEMM. Returns, per n, (n, a, gr, N,
    period, T_mem, T_gemm, M_mem, M_gemm, tokens, mask, roles[K])."""
    K = len(kernels)
    order: Dict[Tuple[int, int], int] = {}
    cls = []
    for k in range(K):
        key = (0, templates[k]) if templates[k] >= 0 else (1, k)
        if key not in order:
            order[key] = len(order)
        cls.append(order[key])
    C = len(order)
    fixed = [-1] * C
    for k in range(K):
        if pins[k] >= 0:
            fixed[cls[k]] = pins[k]
    free = [c for c in range(C) if fixed[c] < 0]
    W, A = [], []
    for reads, writes in kernels:
        W.append(span_bytes([s for s in list(reads) + list(writes) if s[0] in weight_bufs]))
        A.append(span_bytes([s for s in reads if s[0] not in weight_bufs]) +
                 span_bytes([s for s in writes if s[0] not in weight_bufs]))
    d = edge_bytes(edges)

    def t(b, f):
        return max(ceil_div(b * PS, hbm), ceil_div(f * PS, tc)) + launch_ps

    out = []
    for n in (1, 2, 4, 8):
        if n > max_gpus:
            continue
        best = None
        for a in ([1] if n == 1 else range(1, n)):
            gr = n - a
            for j in range(3):
                if not micro_mask >> j & 1:
                    continue
                N = 1 << j
                for mask in range(1 if n == 1 else 1 << len(free)):
                    role = [0] * C
                    if n > 1:
                        for c in range(C):
                            role[c] = 1 if fixed[c] == 1 else 0
                        for b, c in enumerate(free):
                            role[c] = mask >> b & 1
                    Tm = sum(t(W[k] + A[k], flops[k]) for k in range(K) if role[cls[k]] == 0)
                    Tg = sum(t(ceil_div(W[k], gr) + a * A[k], ceil_div(a * flops[k], gr))
                             for k in range(K) if role[cls[k]] == 1)
                    Mm = Mg = 0
                    for (i, jj), nbytes in d.items():
                        ri, rj = role[cls[i]], role[cls[jj]]
                        if ri == rj:
                            continue
                        if rj == 1:
                            Mg += a * (link_lat_ps + ceil_div(nbytes * PS, link_Bps))
                        else:
                            Mm += gr * (link_lat_ps + ceil_div(ceil_div(nbytes, gr) * PS, link_Bps))
                    Tm, Tg, Mm, Mg = N * Tm, N * Tg, N * Mm, N * Mg
                    period = Tm + Tg + Mm + Mg if N == 1 else max(Tm, Tg, Mm, Mg)
                    tok = a * N * rows
                    if best is None or tok * best[4] > best[9] * period:
                        best = (n, a, gr, N, period, Tm, Tg, Mm, Mg, tok, mask, [role[cls[k]] for k in range(K)])
        out.append(best)
    return out
