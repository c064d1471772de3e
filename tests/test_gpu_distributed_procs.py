"""Two processes (both on cuda:0, torch.distributed over gloo) run
tt_svd_distributed as ranks 0 and 1 of a P = 4 partitioned tensor (two slabs
each), exchanging the per-rank R factors through the C-ABI callback (staged
through host memory for gloo).  Every rank must end with the same TT, bitwise
equal to the in-process four-slab run, whose parity with the reference
test_gpu_tt_svd.py pins.  A functional test of the multi-process code path
(the bench runs it over NCCL, one GPU per rank); no timing is taken here.
"""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def rank_main(rank, world, port, gdims, seed, r_max, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist
    from helpers import split_slabs
    from oracle.oracle import random_tensor
    import paper_2102_00104_b200 as tt
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    P = gdims[0]
    glob = random_tensor(seed, gdims)
    slabs, ldims, ld = split_slabs(glob, gdims, P)
    rows = int(np.prod(ldims)) // ldims[-1]
    per = P // world
    mine = [torch.from_numpy(np.ascontiguousarray(s.T)).cuda().t()[:rows] for s in slabs[rank * per:(rank + 1) * per]]

    def exchange(send, recv):  # rank-ordered all-gather, staged through the host for gloo
        h = send.detach().cpu()
        parts = [torch.empty_like(h) for _ in range(world)]
        dist.all_gather(parts, h)
        recv.copy_(torch.cat(parts).to(recv.device))

    T = tt.tt_svd_distributed(mine, ldims, (r_max, 0.0), P_total=P, part0=rank * per, exchange=exchange)
    q.put((rank, T.ranks(), [c.data.copy() for c in T.cores]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("extra,r_max", [(9, 4), (7, 6)])
def test_two_processes_match_in_process(extra, r_max):
    import torch
    import torch.multiprocessing as mp
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from helpers import split_slabs
    from oracle.oracle import random_tensor
    import paper_2102_00104_b200 as tt
    world, P = 2, 4
    gdims = [P] + [2] * extra
    seed = 4242
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=rank_main, args=(rk, world, port, gdims, seed, r_max, q)) for rk in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rk, ranks, cores = q.get(timeout=300)
        res[rk] = (ranks, cores)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    glob = random_tensor(seed, gdims)
    slabs, ldims, ld = split_slabs(glob, gdims, P)
    rows = int(np.prod(ldims)) // ldims[-1]
    dev = [torch.from_numpy(np.ascontiguousarray(s.T)).cuda().t()[:rows] for s in slabs]
    ref = tt.tt_svd_distributed(dev, ldims, (r_max, 0.0))
    for rk in range(world):
        ranks, cores = res[rk]
        assert ranks == ref.ranks()
        for a, b in zip(cores, ref.cores):
            assert np.array_equal(a, b.data)
