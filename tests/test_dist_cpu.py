"""Multi-process host logic on CPU (gloo, world_size 2): every rank derives
the identical plan (the flag protocol depends on it) and the workspace-handle
exchange maps each rank's logical device to its peer's blob."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        from paper_2604_10180_b200 import decoder as DEC, dist as kdist
        from paper_2604_10180_b200.api import Plan, place
        cfg = synth.LLAMA8B.with_(n_layers=4, n_micro=2)
        dg = DEC.DecoderGraph(cfg)
        m = DEC.b200_machine(world)
        a, obj, _ = place(dg.g, m, cfg.n_micro)
        plan = Plan(dg.g, m, a, cfg.n_micro)
        kdist.check_same_plan(dist, plan)                       # raises if ranks disagree
        fake = bytes([rank]) * 64 + (1000 + rank).to_bytes(8, "little")
        peers = kdist.exchange_workspaces(dist, rank, fake)
        q.put((rank, kdist.plan_digest(plan), {d: (b[0], int.from_bytes(b[64:72], "little")) for d, b in peers.items()}))
    finally:
        dist.destroy_process_group()


def test_two_rank_plan_agreement_and_handle_exchange():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    res.sort()
    assert res[0][1] == res[1][1]
    assert res[0][2] == {1: (1, 1001)}
    assert res[1][2] == {0: (0, 1000)}
