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


def transfers_of(edges, assign, repl=None) -> Dict[Tuple[int, int], int]:
    """(producer k, remote device g) -> bytes: union of the edge-record spans
    from k to kernels placed on g ≠ assign[k] (R3 dedup); records on a
    REPLICATED buffer (repl = {(src, buf): delta bytes}) add the producer's
    delta once per buffer instead."""
    spans: Dict[Tuple[int, int], list] = {}
    deltas: Dict[Tuple[int, int], set] = {}
    for s, d, buf, off, ln in edges:
        g = assign[d]
        if g == assign[s]:
            continue
        if repl is not None and (s, buf) in repl:
            deltas.setdefault((s, g), set()).add(buf)
            spans.setdefault((s, g), [])
        else:
            spans.setdefault((s, g), []).append((buf, off, ln))
    return {key: sum(e - a for ivs in _union(v).values() for a, e in ivs) +
            sum(repl[(key[0], b)] for b in deltas.get(key, ()))
            for key, v in spans.items()}


def delta_table(kernels, replicated_bufs):
    """{(kernel, buf): bytes it writes per step into a REPLICATED buffer}: the
    appended K or V slot for RoPE/append (rows·Hkv·D·elem, capped at the
    span), else the declared span (R24-R26 reading of P:465-466).
    kernels[k] = (op_name, attrs_dict, reads, writes)."""
    out = {}
    for k, (op, a, _r, writes) in enumerate(kernels):
        for wi, (buf, _off, ln) in enumerate(writes):
            if buf not in replicated_bufs:
                continue
            d = ln
            if op in ("ROPE_APPEND", "QKV_ROPE") and wi in (1, 2):
                esz = 4 if a.get("dtype", 0) == 1 else 2
                d = min(ln, a["rows"] * a["n_kv_heads"] * a["head_dim"] * esz)
            out[(k, buf)] = out.get((k, buf), 0) + d
    return out


def list_schedule(K: int, t_dev: Sequence[int], assign: Sequence[int], edges,
                  m: Machine, n_micro: int, repl=None):
    """Simulate one step. t_dev[k] = t_{k,assign[k]} (ps, per micro-batch).
    Returns a list of entries (dev, i, k, start, end) sorted by
    (start, dev, i, k) — a global topological order whose restriction to each
    device is that device's execution order."""
    preds: Dict[int, List[int]] = {k: [] for k in range(K)}
    for s, d, *_ in edges:
        if s not in preds[d]:
            preds[d].append(s)
    xfer = transfers_of(edges, assign, repl)
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


# ---------------------------------------------------------------- chunk table (a2 / a13, R10)
# Which producers stream per chunk ("COUNT" release: their primary output is a
# dense bf16 [rows][cols] block written exactly once) and which consumers read
# a remote input chunk by chunk, with the unit of their streamable axis
# ("GEMM consumer → K chunks in 64-col multiples; attention
# consumer of QKV → kv-group chunks; SiLU·mul consumer → 64-col blocks …;
# RMSNorm consumer → column chunks"). Restated here from DESIGN.md's reading
# R10, independently of the library. `op` is the kd.h op NAME, `a` the op's
# attribute fields as a dict; BF16 = 0.

def count_geometry(op, a):
    """(rows, row_bytes) of a COUNT producer's primary output, else None."""
    bf = a.get("dtype", 0) == 0
    if op == "ADD_RMSNORM" and bf:
        return a["rows"], 2 * a["hidden"]
    if op in ("GEMM", "GEMM_SILU") and bf:
        return a["M"], 2 * (a["N"] // 2 if op == "GEMM_SILU" else a["N"])
    if op == "GEMM_RMSNORM" and bf:
        return a["M"], 2 * a["N"]
    if op == "ROPE_APPEND" and bf:
        return a["rows"], 2 * a["n_heads"] * a["head_dim"]
    if op == "ATTENTION" and bf and not (a["flags"] & 1):
        return a["rows"], 2 * a["n_heads"] * a["head_dim"]
    if op == "ATTN_MERGE":
        return a["rows"], 2 * a["n_heads"] * a["head_dim"]
    if op == "SILU_MUL" and bf:
        return a["rows"], 2 * a["ffn"]
    return None


def consumer_unit(op, a, ri, row_bytes):
    """Chunk unit in bytes consumer `op` needs on read ri, 0 if not chunk-aware."""
    if a.get("dtype", 0) != 0:
        return 0
    kblock = lambda m: (2 if (m + 15) // 16 * 16 <= 128 else 1) * 64 * 2
    if op in ("GEMM", "GEMM_SILU", "GEMM_RMSNORM"):
        return kblock(a["M"]) if ri == 0 and 2 * a["K"] == row_bytes else 0
    if op == "QKV_ROPE":
        return kblock(a["rows"]) if ri == 0 and 2 * a["hidden"] == row_bytes else 0
    if op in ("ADD_RMSNORM", "RESIDUAL_ADD"):
        return 16 if 1 <= ri <= a["n_delta"] and 2 * a["hidden"] == row_bytes else 0
    if op == "SILU_MUL":
        return 256 if ri == 0 and 4 * a["ffn"] == row_bytes else 0
    if op == "ROPE_APPEND":
        if ri != 0 or 2 * (a["n_heads"] + 2 * a["n_kv_heads"]) * a["head_dim"] != row_bytes:
            return 0
        return 2 * (a["n_heads"] // a["n_kv_heads"] + 2) * a["head_dim"]
    return 0


def chunk_table(kernels, edges, assign, transfers, n_chunks, replicated=frozenset()):
    """Chunk table of a plan: for every transfer (micro, producer, dst, ...) in
    plan order, (count_mode, rows, row_bytes, unit, [(begin, end), ...]).
    kernels[k] = (op_name, attrs_dict, reads[(buf, off, len)], writes[...]).
    The unit of a producer is the lcm of the units of its remote chunk-aware
    consumers — reads of whole rows of its primary output, every byte of which
    it wrote — capped at the row; chunks follow `chunks` (R10). A GEMM output
    scattered to a device carries only the rows read there (R24); producers
    that mirror replicated buffers release per CTA (R28)."""
    from math import gcd
    srcs: Dict[Tuple[int, int], set] = {}
    for s, d, buf, _off, _ln in edges:
        srcs.setdefault((d, buf), set()).add(s)
    unit_of: Dict[int, int] = {}
    for k, (op, a, reads, _w) in enumerate(kernels):
        for ri, (buf, off, ln) in enumerate(reads):
            ps = srcs.get((k, buf))
            if not ps or len(ps) != 1:
                continue
            src = next(iter(ps))
            if assign[src] == assign[k]:
                continue
            pop, pa, _pr, pw = kernels[src]
            geo = count_geometry(pop, pa)
            if geo is None or not pw:
                continue
            rows, rb = geo
            wb, wo, wl = pw[0]
            if buf != wb or off < wo or off + ln > wo + wl or rows * rb != wl or (off - wo) % rb or ln % rb:
                continue
            u = consumer_unit(op, a, ri, rb)
            if u:
                cur = unit_of.get(src, 0)
                unit_of[src] = u if cur == 0 else cur // gcd(cur, u) * u
    out = []
    for (_i, prod, dst, *_rest) in transfers:
        pop, pa, _pr, pw = kernels[prod]
        ln = pw[0][2] if pw else 0
        geo = count_geometry(pop, pa)
        mirrors = any(w[0] in replicated for w in pw)
        if geo is not None and not mirrors and geo[0] * geo[1] == ln and geo[1] > 0:
            rows, rb = geo
            u = unit_of.get(prod, rb)
            u = rb if u > rb else u
            row0, nrows = 0, rows
            if pop in ("GEMM", "GEMM_SILU", "GEMM_RMSNORM"):
                # scatter: only the rows the destination device reads (one
                # contiguous range of the read spans, widened to whole rows)
                w0b, w0o = pw[0][0], pw[0][1]
                got = _union([(b, o, l) for s_, d_, b, o, l in edges
                              if s_ == prod and assign[d_] == dst and b == w0b]).get(w0b, [])
                if got:
                    lo, hi = got[0][0], got[-1][1]
                    if sum(e - a for a, e in got) == hi - lo:
                        row0 = (lo - w0o) // rb
                        nrows = -(-(hi - w0o) // rb) - row0
            out.append((1, row0, nrows, rb, u, chunks(rb, u, n_chunks)))
        else:
            L = max(ln, 1)
            out.append((0, 0, 1, L, L, [(0, L)]))
    return out
