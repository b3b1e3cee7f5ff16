"""The library's own multi-rank path on >= 2 GPUs (skipped on a 1-GPU box): world_size 2, one row
strip per rank, NCCL communicator from a uid broadcast over a gloo process group
(ncclCommInitRank), the NCCL halo group captured in the iteration graph (and, separately, launched
directly), the overlapped exchange, and the GLOBAL_ON_ROOT gathers of the moments and the state
(grouped NCCL receives on rank 0).  Everything must equal the 1-rank chain bit for bit
(Alg. 1; north_star: bitwise independent of world_size)."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                                 reason="needs >= 2 GPUs")]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem():
    from gpu_common import make_problem
    kw, _ = make_problem(130, 96, kernel="gauss9", cnn=(8, 32), z=True)
    return kw


def _worker(rank, world, port, flags, q):
    import torch.distributed as dist
    from paper_2511_00870_b200 import SCOPE_GLOBAL_ON_ROOT, Sampler, pnpula_get_unique_id
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(rank)
        obj = [pnpula_get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        kw = _problem()
        s = Sampler(**kw, tiles=(world, 1), rank=rank, world_size=world, device=rank, nccl_uid=obj[0],
                    flags=flags)
        try:
            s.run(14, 4, 77)
            mean, var, n = s.moments(scope=SCOPE_GLOBAL_ON_ROOT)
            x, z, t = s.state(scope=SCOPE_GLOBAL_ON_ROOT)
        finally:
            s.close()
        if rank == 0:
            q.put(dict(x=x, z=z, mean=mean, var=var, t=t, n=n))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("flags", [0, 0x4])   # graph replays (NCCL captured) / direct launches
def test_two_ranks_equal_one_rank(flags):
    import torch.multiprocessing as mp
    from gpu_common import gpu_run
    ref = gpu_run(_problem(), 14, 4, 77)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, flags, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert got["t"] == 14 and got["n"] == 10
    for k in ("x", "z", "mean", "var"):
        np.testing.assert_array_equal(got[k], ref[k], err_msg=k)
