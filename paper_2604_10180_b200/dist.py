"""Multi-process plumbing for one process per GPU (torchrun): every rank
builds the same graph and plan (deterministic), runs only its own logical
device, and maps its peers' workspaces through CUDA IPC so that producer
kernels can store cut-edge outputs and release flags directly in the
consumer GPU's HBM over NVLink. torch.distributed is used
for the handle exchange and barriers only — no collective on the data path.
"""
from __future__ import annotations

import ctypes as C
import hashlib
import struct
from typing import Dict, List, Sequence

from . import _kd as K


def plan_digest(plan) -> str:
    """sha256 over the plan's schedule, transfers and workspace sizes; all
    ranks must agree before any peer pointer is used."""
    h = hashlib.sha256()
    for e in plan.schedule():
        h.update(struct.pack("<IIIqq", *e))
    for t in plan.transfers():
        h.update(struct.pack("<IIIQqq", *t))
    n_dev = plan.m.n_dev
    for d in range(n_dev):
        h.update(struct.pack("<Q", plan.workspace_bytes(d)))
    return h.hexdigest()


def all_gather_bytes(dist, payload: bytes, group=None) -> List[bytes]:
    """all_gather of one small byte string per rank of `group` (gloo or nccl)."""
    out: List = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, payload, group=group)
    return out


def check_same_plan(dist, plan, group=None):
    digests = all_gather_bytes(dist, plan_digest(plan).encode(), group)
    if len(set(digests)) != 1:
        raise RuntimeError(f"ranks derived different plans: {digests}")


def export_workspace(ptr: int) -> bytes:
    """64-byte IPC handle of the allocation holding ptr + its offset."""
    handle = (C.c_uint8 * 64)()
    off = C.c_uint64()
    K.check(K.kd_ipc_get_handle(C.c_void_p(ptr), handle, C.byref(off)), "kd_ipc_get_handle")
    return bytes(handle) + struct.pack("<Q", off.value)


def import_workspace(blob: bytes) -> int:
    handle = (C.c_uint8 * 64).from_buffer_copy(blob[:64])
    (off,) = struct.unpack("<Q", blob[64:72])
    p = C.c_void_p()
    K.check(K.kd_ipc_open(handle, off, C.byref(p)), "kd_ipc_open")
    return p.value


def exchange_workspaces(dist, my_dev: int, blob: bytes, group=None) -> Dict[int, bytes]:
    """Every rank of `group` contributes (logical device, exported blob);
    returns the peers' blobs keyed by logical device."""
    got = all_gather_bytes(dist, struct.pack("<I", my_dev) + blob, group)
    out = {}
    for g in got:
        (d,) = struct.unpack("<I", g[:4])
        if d != my_dev:
            out[d] = g[4:]
    if len(out) != dist.get_world_size(group) - 1:
        raise RuntimeError("duplicate logical devices across ranks")
    return out
