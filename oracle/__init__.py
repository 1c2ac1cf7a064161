"""ORACLE — test infrastructure only.

A plain, slow, obviously-correct CPU implementation of what the hot path of
kernel disaggregation (arXiv 2604.10180) computes. It shares NO code with the
CUDA path (`paper_2604_10180_b200/`), and neither imports the other. Only
`tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import it. The product path never routes through
here; if the CUDA extension is missing the product fails loudly.

Modules (each function cites the passage it follows; P:n = PAPER.md line n,
S:n = SPEC.md line n, R# = the readings listed in SURVEY.md §8(c) and DESIGN.md):
  layer     — decoder-layer math in fp64 (C1; R12 storage rounding)
  prefill   — the prefill phase of the same layer: RoPE at every prompt
              position + paged-cache fill, causal attention (f4)
  ddg       — RAW data-dependency graph by last-writer registry + per-byte
              brute force (C2)
  placement — cost model, objective E1–E7 in integer picoseconds, plain
              exhaustive enumeration (C3)
  schedule  — discrete-event list schedule + chunk partition (P:380, P:401-402,
              C4, R10, R11)
  monitor   — online monitor's windowed queueing-ratio policy switch
              (R21)

Parity pins live in tests/test_oracle_*.py. Functions without an independent
pin say "parity unpinned" in their docstring (none at present).
"""
from . import layer, prefill, ddg, placement, schedule, monitor  # noqa: F401
