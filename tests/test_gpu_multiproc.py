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


def _rank(rank, world, port, q, steps):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import synth
        from paper_2604_10180_b200 import decoder as DEC
        cfg = synth.TINY
        inp = synth.make_decoder_inputs(cfg)
        dg = DEC.DecoderGraph(cfg)
        rt = DEC.DecoderRuntime(dg, dg.role_assign(0, 1), 2, [0], inputs=inp, local_devs=[rank], dist=dist)
        for _ in range(steps):
            rt.step()
        rt.sync()
        rt.rt.check()
        dist.barrier()
        q.put((rank, rt.residual() if rank == 0 else None, len(rt.plan.transfers())))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_two_processes_ipc_bitwise_equals_monolithic(cuda_ok):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    steps = 2
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q, steps)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (x, n)) for r, x, n in [q.get(timeout=600) for _ in range(2)])
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    import synth
    from paper_2604_10180_b200 import decoder as DEC
    cfg = synth.TINY
    inp = synth.make_decoder_inputs(cfg)
    dg = DEC.DecoderGraph(cfg)
    mono = DEC.DecoderRuntime(dg, [0] * dg.g.num_kernels, 1, [0], inputs=inp)
    for _ in range(steps):
        mono.step()
    mono.sync()
    assert res[0][1] > 0
    assert np.array_equal(res[0][0], mono.residual())
