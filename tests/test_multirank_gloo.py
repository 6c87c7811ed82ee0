"""CPU, world_size 2 over gloo: the RHS-sharded multi-GPU path's host logic (sharding, gather,
max-over-ranks timing). The per-rank solve here is the numpy oracle (test infrastructure);
on GPUs each rank calls the C-ABI against its own resident factors."""
import math
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2003_02585_b200.multi import shard_rhs


def test_shard_rhs_partitions():
    for total in (0, 1, 5, 16, 33):
        for world in (1, 2, 3, 8):
            blocks = [shard_rhs(total, r, world) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == total
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_rhs(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist
    from oracle import hs_oracle as O
    from paper_2003_02585_b200.multi import max_over_ranks, solve_sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        setup = O.ProblemSetup(O.Box(2), [32, 32, 1], [2, 2, 1], O.Medium("constant", kappa=6 * math.pi),
                               O.PmlSpec(width=6))
        s = O.DdmSolver(setup)
        f = O.gaussian_source(s.ggrid, O.Box(2), O.seeded_centers(3, 5, O.Box(2)), 2.0 / 32)
        B = s.scale_source(f).T.copy()
        U = solve_sharded(lambda b: np.stack([s.ddm_solve(x.copy(), 1)[0] for x in b]), B, rank, world)
        t = max_over_ranks(float(rank + 1))
        if rank == 0:
            ref = np.stack([s.ddm_solve(x.copy(), 1)[0] for x in B])
            out.put((float(np.max(np.abs(U - ref))), t))
    finally:
        dist.destroy_process_group()


def test_rhs_sharded_solve_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    err, tmax = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert err == 0.0  # sharding is exact: same per-RHS computation, gathered in order
    assert tmax == 2.0
