"""Oracle — RAW data-dependency graph (test infrastructure only).

Follows PAPER.md §3.1 "Data dependency analysis": "the analyzer
maintains a global buffer registry that tracks the last writer of each buffer.
When a kernel reads a buffer, the analyzer queries the registry to identify the
most recent writer. If the writer differs from the current kernel, a
dependency edge is added from the writer to the reader. By iterating over
kernels in execution order …  only … Read-After-Write (RAW) dependencies."
Library-kernel read/write sets are declared.

Readings: R1 byte-span granularity; R2 all reads of a kernel are
resolved before its own writes apply, never self-edges; R3 one record per
(src, dst, buf, maximal contiguous span) and d_ij = Σ record lengths;
R4 no WAR/WAW edges; R5 never-written bytes (weights, inputs) have no writer.

A kernel is given as (reads, writes), each a list of (buf, offset, length).
An edge record is (src, dst, buf, offset, length).
"""
from __future__ import annotations

from typing import Dict, List, Sequence, Tuple

Span = Tuple[int, int, int]          # (buf, offset, length)
Edge = Tuple[int, int, int, int, int]  # (src, dst, buf, offset, length)


def _union(spans: Sequence[Span]) -> Dict[int, List[Tuple[int, int]]]:
    """Per buffer, the sorted disjoint union [start, end) of the spans."""
    per: Dict[int, List[Tuple[int, int]]] = {}
    for buf, off, ln in spans:
        per.setdefault(buf, []).append((off, off + ln))
    out = {}
    for buf, iv in per.items():
        iv.sort()
        merged = [list(iv[0])]
        for s, e in iv[1:]:
            if s <= merged[-1][1]:
                merged[-1][1] = max(merged[-1][1], e)
            else:
                merged.append([s, e])
        out[buf] = [(s, e) for s, e in merged]
    return out


class Registry:
    """Last writer of every byte range of every buffer, as a sorted list of
    disjoint (start, end, writer) intervals per buffer (the "global buffer
    registry" of P:276 at byte granularity, R1)."""

    def __init__(self):
        self.iv: Dict[int, List[Tuple[int, int, int]]] = {}

    def lookup(self, buf: int, s: int, e: int) -> List[Tuple[int, int, int]]:
        """Sub-intervals of [s,e) that have a writer, with that writer."""
        res = []
        for a, b, w in self.iv.get(buf, []):
            lo, hi = max(a, s), min(b, e)
            if lo < hi:
                res.append((lo, hi, w))
        return res

    def write(self, buf: int, s: int, e: int, writer: int):
        old = self.iv.get(buf, [])
        new = []
        for a, b, w in old:
            if b <= s or a >= e:
                new.append((a, b, w))
            else:
                if a < s:
                    new.append((a, s, w))
                if b > e:
                    new.append((e, b, w))
        new.append((s, e, writer))
        new.sort()
        self.iv[buf] = new


def build_ddg(kernels: Sequence[Tuple[Sequence[Span], Sequence[Span]]]) -> List[Edge]:
    """Registry algorithm (C2). Kernels are in program (execution) order."""
    reg = Registry()
    edges: List[Edge] = []
    for k, (reads, writes) in enumerate(kernels):
        for buf, ivs in sorted(_union(reads).items()):
            for s, e in ivs:
                hits = [h for h in reg.lookup(buf, s, e) if h[2] != k]
                # merge adjacent pieces with the same writer -> maximal spans
                hits.sort()
                run = None
                for lo, hi, w in hits:
                    if run and run[2] == w and run[1] == lo:
                        run = (run[0], hi, w)
                    else:
                        if run:
                            edges.append((run[2], k, buf, run[0], run[1] - run[0]))
                        run = (lo, hi, w)
                if run:
                    edges.append((run[2], k, buf, run[0], run[1] - run[0]))
        for buf, ivs in _union(writes).items():
            for s, e in ivs:
                reg.write(buf, s, e, k)
    edges.sort(key=lambda x: (x[1], x[0], x[2], x[3]))
    return edges


def brute_force_ddg(kernels) -> List[Edge]:
    """Independent per-byte enumeration (C2 pin): for every kernel j and every
    byte b it reads, the writer is the largest i < j whose write set contains
    b (no m in (i, j) writes b); consecutive bytes with the same writer form
    one record."""
    def bytes_of(spans):
        s = set()
        for buf, off, ln in spans:
            for x in range(off, off + ln):
                s.add((buf, x))
        return s

    wsets = [bytes_of(w) for _, w in kernels]
    edges = []
    for j, (reads, _) in enumerate(kernels):
        rb = sorted(bytes_of(reads))
        writer_of = {}
        for (buf, x) in rb:
            for i in range(j - 1, -1, -1):
                if (buf, x) in wsets[i]:
                    writer_of[(buf, x)] = i
                    break
        run = None
        for (buf, x) in rb:
            w = writer_of.get((buf, x))
            if run and w is not None and run[0] == w and run[1] == buf and run[3] == x:
                run = (w, buf, run[2], x + 1)
            else:
                if run:
                    edges.append((run[0], j, run[1], run[2], run[3] - run[2]))
                run = (w, buf, x, x + 1) if w is not None else None
        if run:
            edges.append((run[0], j, run[1], run[2], run[3] - run[2]))
    edges.sort(key=lambda x: (x[1], x[0], x[2], x[3]))
    return edges


def edge_bytes(edges: Sequence[Edge], repl=None) -> Dict[Tuple[int, int], int]:
    """d_ij = Σ record lengths over records (i, j) (Table 2, R3).
    repl: {(src, buf): delta bytes} for REPLICATED buffers (P:465-466 delta
    replication): their records charge the producer's delta once per
    (src, dst, buf) instead of the span."""
    d: Dict[Tuple[int, int], int] = {}
    seen = set()
    for s, t, buf, _, ln in edges:
        if repl is not None and (s, buf) in repl:
            add = repl[(s, buf)] if (s, t, buf) not in seen else 0
            seen.add((s, t, buf))
            d[(s, t)] = d.get((s, t), 0) + add
            continue
        d[(s, t)] = d.get((s, t), 0) + ln
    return d
