"""B200-native kernel disaggregation (arXiv 2604.10180) — the pipelined
cross-GPU decoder-layer hot path as a C-ABI library (include/kd.h, libkd.so)
with a thin Python binding. Importing requires the built library; there is
no CPU fallback.
"""
from . import _kd  # noqa: F401  (raises ImportError if libkd.so is missing)
from ._kd import KdError, check  # noqa: F401
from .api import (Graph, Machine, Plan, Runtime, chunks, cost, objective, place)  # noqa: F401
