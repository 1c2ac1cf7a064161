"""One process per logical device (the torchrun layout), on the single GPU of
the test box: two processes share cuda:0, each runs only its role's kernels,
and producer kernels store cut-edge outputs + release flags directly in the
other process's workspace, mapped through CUDA IPC. The result must be
bitwise equal to the monolithic step."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _graph(DEC, kind, cfg):
    if kind == "sharded":  # f2: 2 KV shards (devices 0, 1) + GEMMs (device 2), LSE partials streamed to the merge
        dg = DEC.ShardedKVDecoderGraph(cfg, 2)
        return dg, dg.assign(), 3
    dg = DEC.DecoderGraph(cfg)
    return dg, dg.role_assign(0, 1), 2


def _cfg(kind):
    import synth
    if kind == "pair8b":  # full 8B layer widths, the bench's m = 32 tiling, short context
        return synth.LLAMA8B.with_(n_layers=2, batch=64, n_micro=2, context=512)
    return synth.TINY


def _rank(rank, world, port, q, steps, kind="pair"):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import synth
        from paper_2604_10180_b200 import decoder as DEC
        cfg = _cfg(kind)
        inp = synth.make_decoder_inputs(cfg)
        dg, assign, n_dev = _graph(DEC, kind, cfg)
        rt = DEC.DecoderRuntime(dg, assign, n_dev, [0], inputs=inp, local_devs=[rank], dist=dist)
        for _ in range(steps):
            rt.step()
        rt.sync()
        rt.rt.check()
        dist.barrier()
        q.put((rank, rt.residual() if rank == 0 else None, len(rt.plan.transfers())))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,world", [("pair", 2), ("sharded", 3), ("pair8b", 2)])
def test_processes_ipc_bitwise_equals_monolithic(cuda_ok, kind, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    steps = 2
    procs = [ctx.Process(target=_rank, args=(r, world, port, q, steps, kind)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict((r, (x, n)) for r, x, n in [q.get(timeout=600) for _ in range(world)])
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    import synth
    from paper_2604_10180_b200 import decoder as DEC
    cfg = _cfg(kind)
    inp = synth.make_decoder_inputs(cfg)
    dg, _, _ = _graph(DEC, kind, cfg)
    mono = DEC.DecoderRuntime(dg, [0] * dg.g.num_kernels, 1, [0], inputs=inp)
    for _ in range(steps):
        mono.step()
    mono.sync()
    assert res[0][1] > 0
    assert np.array_equal(res[0][0], mono.residual())
