"""B200-native kernel disaggregation (arXiv 2604.10180) — the pipelined
cross-GPU decoder-layer hot path as a C-ABI library (include/kd.h, libkd.so)
with a thin Python binding.

`paper_2604_10180_b200.build` compiles the library and needs nothing else;
every other module loads libkd.so on import and raises ImportError if it is
missing — there is no CPU fallback.
"""
_LAZY = {"Graph", "Machine", "Plan", "Runtime", "chunks", "cost", "objective", "place", "KdError", "check"}


def __getattr__(name):
    if name in _LAZY:
        from . import api, _kd
        return getattr(api, name) if hasattr(api, name) else getattr(_kd, name)
    raise AttributeError(name)
