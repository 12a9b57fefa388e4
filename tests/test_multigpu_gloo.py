"""The N>1 path's host logic on CPU with world_size 2 over gloo: shard
planning (contiguous, disjoint, complete cover of the packed layouts), per-rank
slices assembled in rank order equal the oracle's full result, the collision
count all-reduce, and max-over-ranks timing.  The per-shard compute here is the
oracle (CPU); the GPU kernels' shard parity is tests/test_gpu_parity.py."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch
    import torch.distributed as dist

    import oracle
    from paper_1308_1419_b200 import multi

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, rho = 700, 16
        plan = multi.shard_plan(n, rho, world)
        me = plan[rank]
        pts = oracle.gen_points(n, 3, 42)
        r0 = min(n, me.block_rows[0] * rho)
        r1 = min(n, me.block_rows[1] * rho)
        part = oracle.edm_rows(pts, r0, r1)
        assert part.size == me.size
        # gather slices in rank order (rank 0 assembles)
        sizes = [None] * world
        dist.all_gather_object(sizes, part.size)
        slices = [None] * world
        dist.all_gather_object(slices, part.tobytes())
        full = b"".join(slices)
        # collision hits of this shard's rows, all-reduced
        sph = oracle.gen_points(n, 4, 7)
        _, h = oracle.collide_rows_u8(sph, 0.0625, r0, r1)
        total = multi.reduce_hits(torch.tensor([h], dtype=torch.int64))
        # max over ranks
        t = multi.max_over_ranks(float(rank + 1))
        if rank == 0:
            q.put((full, sizes, total, t, [s.elems for s in plan], [s.pairs for s in plan]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_path_gloo(world, orc, tg):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    full, sizes, total, t, elems, pairs = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = 700
    want = orc.edm_reference(orc.gen_points(n, 3, 42))
    assert full == want.tobytes()
    assert sum(sizes) == orc.tri_count(n)
    _, hits = orc.collide_reference(orc.gen_points(n, 4, 7), 0.0625)
    assert total == hits
    assert t == float(world)
    assert elems[0][0] == 0 and elems[-1][1] == orc.tri_count(n)
    assert all(a[1] == b[0] for a, b in zip(elems, elems[1:]))
    assert pairs[0][0] == 0 and pairs[-1][1] == orc.tri_count(n, False)
