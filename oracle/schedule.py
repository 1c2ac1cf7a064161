"""Oracle — discrete-event list schedule of a disaggregated step and the chunk
partition (test infrastructure only).

Semantics follow PAPER.md §3.3: a worker "posts the corresponding recv
kernels before launching k. After k completes … posts the corresponding send
kernels" on separate communication streams; multiple requests
(here: micro-batches) run concurrently and earlier ones get priority so their
communication phases stagger. The executable reading is SPEC's
simulator with readings R10/R11:

* a device runs one kernel at a time; when it is idle it starts, among the
  entries (micro-batch i, kernel k) placed on it whose inputs are available,
  the one with the smallest key (i, k) (work conserving, R11);
* a cut edge's data (the union of the spans the producer's consumers on one
  remote device read, per micro-batch) is one transfer on the ordered channel
  (u → g); a channel carries one transfer at a time in issue order; a transfer
  issued at the producer's end takes c = ℓ + ⌈bytes·10¹²/bw⌉ ps (E4);
* integer picoseconds throughout (R7).
"""
from __future__ import annotations

from typing import Dict, List, Sequence, Tuple

from .ddg import _union
from .placement import PS, Machine, ceil_div


def transfers_of(edges, assign) -> Dict[Tuple[int, int], int]:
    """(producer k, remote device g) -> bytes: union of the edge-record spans
    from k to kernels placed on g ≠ assign[k] (R3 dedup)."""
    spans: Dict[Tuple[int, int], list] = {}
    for s, d, buf, off, ln in edges:
        g = assign[d]
        if g != assign[s]:
            spans.setdefault((s, g), []).append((buf, off, ln))
    return {key: sum(e - a for ivs in _union(v).values() for a, e in ivs)
            for key, v in spans.items()}


def list_schedule(K: int, t_dev: Sequence[int], assign: Sequence[int], edges,
                  m: Machine, n_micro: int):
    """Simulate one step. t_dev[k] = t_{k,assign[k]} (ps, per micro-batch).
    Returns a list of entries (dev, i, k, start, end) sorted by
    (start, dev, i, k) — a global topological order whose restriction to each
    device is that device's execution order."""
    preds: Dict[int, List[int]] = {k: [] for k in range(K)}
    for s, d, *_ in edges:
        if s not in preds[d]:
            preds[d].append(s)
    xfer = transfers_of(edges, assign)
    out_x: Dict[int, List[Tuple[int, int]]] = {}
    for (k, g), b in sorted(xfer.items()):
        out_x.setdefault(k, []).append((g, b))

    end: Dict[Tuple[int, int], int] = {}
    arrival: Dict[Tuple[int, int, int], int] = {}   # (i, producer, dev) -> time
    chan_free: Dict[Tuple[int, int], int] = {}
    started = set()
    running: Dict[int, Tuple[int, int, int]] = {}    # dev -> (end, i, k)
    entries = []
    todo = {(i, k) for i in range(n_micro) for k in range(K)}
    tau = 0

    def available(i, k, now):
        g = assign[k]
        for p in preds[k]:
            if (i, p) not in end or end[(i, p)] > now:
                return False
            if assign[p] != g and arrival[(i, p, g)] > now:
                return False
        return True

    while todo or running:
        # 1) completions at or before tau, in (end, i, k) order, issue sends
        fin = sorted((e, i, k, d) for d, (e, i, k) in running.items() if e <= tau)
        for e, i, k, d in fin:
            del running[d]
            for g, b in out_x.get(k, []):
                u = assign[k]
                st = max(e, chan_free.get((u, g), 0))
                arr = st + m.link_lat_ps[u][g] + ceil_div(b * PS, m.link_Bps[u][g])
                chan_free[(u, g)] = arr
                arrival[(i, k, g)] = arr
        # 2) idle devices start their smallest available (i, k)
        for d in range(m.n_dev):
            if d in running:
                continue
            ready = sorted((i, k) for (i, k) in todo if assign[k] == d and available(i, k, tau))
            if ready:
                i, k = ready[0]
                todo.discard((i, k))
                e = tau + t_dev[k]
                end[(i, k)] = e
                running[d] = (e, i, k)
                entries.append((d, i, k, tau, e))
        # 3) advance time to the next event
        cand = [e for (e, _, _) in running.values() if e > tau]
        cand += [a for a in arrival.values() if a > tau]
        if not cand:
            if todo:
                raise RuntimeError("schedule deadlock")
            break
        tau = min(cand)
    entries.sort(key=lambda x: (x[3], x[0], x[1], x[2]))
    return entries


def chunks(length: int, unit: int, n: int) -> List[Tuple[int, int]]:
    """Chunk partition of a span of `length` bytes along an axis of `unit`
    bytes into n chunks (C4, R10; the paper has no chunking):
    q = ⌈⌈length/unit⌉/n⌉·unit ; chunk c = [c·q, min((c+1)·q, length));
    empty chunks dropped."""
    q = ceil_div(ceil_div(length, unit), n) * unit
    out = []
    for c in range(n):
        a, b = c * q, min((c + 1) * q, length)
        if a < b:
            out.append((a, b))
    return out
