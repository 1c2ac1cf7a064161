"""Build libkd.so (host planner + sm_100a kernels + runtime) in-tree with nvcc.

`python -m paper_2604_10180_b200.build` or `build()`; incremental by mtime.
Every .cu is compiled with -gencode arch=compute_100a,code=sm_100a -lineinfo.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# KD_BUILD_TAG / KD_EXTRA_NVCC: A/B variants (libkd_<tag>.so, loaded with KD_LIB)
_TAG = os.environ.get("KD_BUILD_TAG", "")
BUILD = os.path.join(PKG, "_build" + (f"_{_TAG}" if _TAG else ""))
LIB = os.path.join(PKG, f"libkd_{_TAG}.so" if _TAG else "libkd.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-I", os.path.join(ROOT, "include"), "-I", CSRC,
          "-Xcompiler", "-fPIC,-Wall,-Wno-unused-function", "--expt-relaxed-constexpr"] + \
    os.environ.get("KD_EXTRA_NVCC", "").split()


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "host", "*.cpp")) + glob.glob(os.path.join(CSRC, "kernels", "*.cu")))


def _headers():
    return (glob.glob(os.path.join(CSRC, "**", "*.hpp"), recursive=True)
            + glob.glob(os.path.join(CSRC, "**", "*.cuh"), recursive=True)
            + [os.path.join(ROOT, "include", "kd.h")])


def _compile(src, verbose=False):
    obj = os.path.join(BUILD, os.path.relpath(src, CSRC).replace(os.sep, "_") + ".o")
    dep = max([os.path.getmtime(src)] + [os.path.getmtime(h) for h in _headers()])
    if os.path.exists(obj) and os.path.getmtime(obj) >= dep:
        return obj
    if src.endswith(".cu"):
        cmd = [NVCC] + ARCH + COMMON + ["-Xptxas", "-v" if verbose else "-O3", "-c", src, "-o", obj]
    else:
        cmd = [NVCC, "-x", "c++"] + COMMON + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart_static", "-ldl", "-lrt", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
