"""Multi-process (world_size 2, gloo, CPU) check of the SPMD halo-exchange plan that the
library's NCCL path executes: every rank owns n_tiles/world consecutive tiles, posts the
library's messages (pnpula_plan_halo, canonical (src, dst) order) as point-to-point
sends/receives, and must end with every ghost frame equal to the global image (zero
outside it) -- Alg. 1 line 5, ghost regions P:494-498."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2511_00870_b200 as pk


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _tile_rect(ny, nx, ty, tx, t):
    a, b = pk.pnpula_partition(ny, ty, t // tx)
    c, d = pk.pnpula_partition(nx, tx, t % tx)
    return a, c, b - a, d - c


def _worker(rank, world, port, case, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ny, nx, ty, tx, h = case
        nt = ty * tx
        per = nt // world
        mine = range(rank * per, (rank + 1) * per)
        owner = lambda t: t // per
        img = (np.arange(ny * nx, dtype=np.float32).reshape(ny, nx) + 1.0)
        pads = {}
        for t in mine:
            i0, j0, th, tw = _tile_rect(ny, nx, ty, tx, t)
            pad = np.zeros((th + 2 * h, tw + 2 * h), np.float32)
            pad[h:h + th, h:h + tw] = img[i0:i0 + th, j0:j0 + tw]
            pads[t] = pad
        msgs = pk.pnpula_plan_halo(ny, nx, ty, tx, h)
        reqs, recvs = [], []
        for k, (s, d, (ri, rj, rh, rw)) in enumerate(msgs):
            if s in pads and d in pads:               # same rank: local copy
                si0, sj0, _, _ = _tile_rect(ny, nx, ty, tx, s)
                di0, dj0, _, _ = _tile_rect(ny, nx, ty, tx, d)
                band = pads[s][ri - si0 + h:ri - si0 + h + rh, rj - sj0 + h:rj - sj0 + h + rw]
                pads[d][ri - di0 + h:ri - di0 + h + rh, rj - dj0 + h:rj - dj0 + h + rw] = band
            elif s in pads:
                si0, sj0, _, _ = _tile_rect(ny, nx, ty, tx, s)
                band = torch.from_numpy(np.ascontiguousarray(
                    pads[s][ri - si0 + h:ri - si0 + h + rh, rj - sj0 + h:rj - sj0 + h + rw]))
                reqs.append(dist.isend(band, dst=owner(d), tag=k))
            elif d in pads:
                buf = torch.zeros((rh, rw))
                reqs.append(dist.irecv(buf, src=owner(s), tag=k))
                recvs.append((d, (ri, rj, rh, rw), buf))
        for r in reqs:
            r.wait()
        for d, (ri, rj, rh, rw), buf in recvs:
            di0, dj0, _, _ = _tile_rect(ny, nx, ty, tx, d)
            pads[d][ri - di0 + h:ri - di0 + h + rh, rj - dj0 + h:rj - dj0 + h + rw] = buf.numpy()
        gp = np.zeros((ny + 2 * h, nx + 2 * h), np.float32)
        gp[h:h + ny, h:h + nx] = img
        ok = True
        for t, pad in pads.items():
            i0, j0, th, tw = _tile_rect(ny, nx, ty, tx, t)
            ok &= bool(np.array_equal(pad, gp[i0:i0 + th + 2 * h, j0:j0 + tw + 2 * h]))
        out[rank] = int(ok)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [(37, 29, 2, 2, 4), (64, 50, 2, 1, 8), (41, 70, 2, 4, 5), (90, 33, 6, 1, 9)])
def test_two_rank_halo_exchange_plan(case):
    world = 2
    ctx = mp.get_context("spawn")
    out = ctx.Array("i", [0] * world)
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert list(out) == [1] * world
