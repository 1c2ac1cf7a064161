"""Oracle — the online monitor's queueing-aware policy switch (test
infrastructure only; nothing on the product path imports it).

PAPER.md §3.4 "Online Monitor": "At each window boundary, the
monitor computes the average request latency L̄_req and the pure execution
latency L̄_exec, which aggregates computation and communication time while
excluding queueing delay. The ratio L̄_req / L̄_exec serves as an indicator of
queueing pressure. A low ratio ... favors the latency-oriented policy, whereas
a high ratio ... triggering a switch to the throughput-oriented policy."
Defaults W = 300 ms, β = 1.5.

Readings (R21): a request belongs to the window in which it
finishes; "high" means ratio > β (ratio == β keeps/chooses latency); a window
without finished requests keeps the current policy. Written out plainly with
exact fractions, windows evaluated one by one in time order.
"""
from __future__ import annotations

from fractions import Fraction
from typing import List, Sequence, Tuple

LATENCY, THROUGHPUT = 2, 1  # KD_OBJ_LATENCY, KD_OBJ_THROUGHPUT


def policy_trace(requests: Sequence[Tuple[int, int, int]], window_ns: int, beta: Fraction,
                 initial: int = LATENCY, horizon_ns: int = None) -> Tuple[List[int], int]:
    """requests: (t_end_ns, req_latency_ns, exec_latency_ns). Returns the
    policy after each window boundary up to `horizon_ns` (default: the window
    after the last request) and the number of switches."""
    if not requests and horizon_ns is None:
        return [], 0
    last = max(t for t, _, _ in requests) if requests else 0
    n_windows = (horizon_ns // window_ns) if horizon_ns is not None else last // window_ns + 1
    policy, switches, out = initial, 0, []
    for w in range(n_windows):
        members = [(r, e) for t, r, e in requests if t // window_ns == w]
        if members:
            mean_req = Fraction(sum(r for r, _ in members), len(members))
            mean_exec = Fraction(sum(e for _, e in members), len(members))
            new = THROUGHPUT if mean_req > beta * mean_exec else LATENCY
            if new != policy:
                switches += 1
            policy = new
        out.append(policy)
    return out, switches
