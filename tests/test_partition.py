"""Subdomain-partitioned multi-rank path.

CPU (gloo, world_size 2): the host logic — default ownership (balanced per rank, deterministic),
the traffic model (traces cross ranks only between owners of neighbouring subdomains), and the
host-staged exchange helper (one message per peer, offsets and counts as the library lists them).

GPU (-m gpu): two ranks share the one B200 of the test box, each with its own handle holding only
its subdomains' factors; the exchange is host-staged over gloo, so neither rank's kernels wait on
the other's. u must equal the single-process solve bit for bit (each global node is accumulated
by one home rank in the reference's order, and summing it with zeros is exact), counters exactly,
sweep norms to roundoff."""
import ast
import math
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2003_02585_b200.multi import partition_owners, partition_traffic

COUNTERS = ["traces_generated", "traces_routed", "traces_discarded", "local_solves", "skipped_zero_solves"]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("dim,counts,world", [(2, [4, 4], 2), (2, [8, 8], 8), (2, [4, 4], 8), (3, [4, 4, 4], 8),
                                              (3, [2, 2, 2], 2), (2, [3, 2], 4)])
def test_default_owners_balanced(dim, counts, world):
    o = partition_owners(dim, counts, world)
    nsub = int(np.prod(counts[:dim]))
    assert len(o) == nsub and min(o) >= 0 and max(o) < world
    assert partition_owners(dim, counts, world) == o  # deterministic
    per = np.bincount(o, minlength=world)
    assert per.max() - per.min() <= 1
    ms, makespan, cross, traces = partition_traffic(dim, counts, 1, world, o)
    ms1, makespan1, cross1, traces1 = partition_traffic(dim, counts, 1, 1, [0] * nsub)
    assert ms == ms1 and cross1 == 0 and traces1.sum() == traces.sum()
    # every step's busiest rank: at least the even share, at most the single-rank schedule
    assert math.ceil(nsub * 2 ** dim / world) <= makespan <= makespan1


def test_traffic_only_between_neighbour_owners():
    dim, counts, world = 2, [4, 4], 4
    o = partition_owners(dim, counts, world)
    _, _, _, tr = partition_traffic(dim, counts, 1, world, o)
    nb = np.zeros((world, world), bool)
    for j in range(4):
        for i in range(4):
            for di, dj in ((1, 0), (-1, 0), (0, 1), (0, -1)):
                if 0 <= i + di < 4 and 0 <= j + dj < 4:
                    nb[o[i + 4 * j], o[i + di + 4 * (j + dj)]] = True
    assert np.all(tr[~nb] == 0)
    single = partition_traffic(dim, counts, 1, 1, [0] * 16)[3]
    # routed traces per application: 2D rounds=1 routes 10 of the 16 (sweep, direction) pairs
    assert tr.sum() == single.sum()


def _gloo_exchange_worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2003_02585_b200.multi import exchange_host
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        other = 1 - rank
        # rank 0 sends 5 doubles and receives 3; rank 1 the mirror (message lengths differ)
        ns, nr = (5, 3) if rank == 0 else (3, 5)
        send = np.arange(ns, dtype=np.float64) + 100 * rank
        recv = np.full(nr + 2, -1.0)
        exchange_host(send, recv, [other], [0], [ns], [2], [nr])
        q.put((rank, recv.tolist()))
    finally:
        dist.destroy_process_group()


def test_exchange_host_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_exchange_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got[0] == [-1.0, -1.0, 100.0, 101.0, 102.0]
    assert got[1] == [-1.0, -1.0, 0.0, 1.0, 2.0, 3.0, 4.0]


# --------------------------------------------------------------------------------------------
# GPU: two ranks on one device, host-staged exchange

def _setup(hs, z):
    dim = int(z["dim"])
    med = ast.literal_eval(str(z["medium"]))
    if med["media.kind"] == "constant":
        m = hs.Medium("constant", kappa=med["media.kappa"])
    else:
        m = hs.Medium("two_layered", kappa_down=med["media.kappa_down"], kappa_up=med["media.kappa_up"],
                      axis=med["media.axis"], eta=med["media.eta_L"], eps=med["media.epsilon"])
    return hs.ProblemSetup(dim, [int(z["n"])] * dim, list(z["parts"]), m, pml_width=int(z["pad"]))


def _gpu_worker(rank, world, port, name, owner, q):
    import torch
    import torch.distributed as dist
    import paper_2003_02585_b200 as hs
    from paper_2003_02585_b200.multi import PartitionedDdmSolver
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        z = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", name + ".npz"))
        s = PartitionedDdmSolver(_setup(hs, z), device=0, owner=owner)
        reps = []
        U = s.ddm_solve(z["b"], int(z["rounds"]), reps, True)
        info = s.partition_info()
        q.put((rank, U, [[getattr(r, k) for k in COUNTERS] for r in reps],
               [list(r.sweep_contrib_norm) for r in reps], [list(r.round_residuals) for r in reps], info))
    except Exception as e:  # surface the failure in the parent
        q.put((rank, repr(e), None, None, None, None))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("name,owner", [("ddm_2d_2x2", None), ("ddm_2d_2x2", [0, 1, 1, 0]), ("ddm_2d_3x2_r2", None),
                                        ("ddm_2d_layered", None), ("ddm_3d_2x2x2", None)])
def test_partitioned_equals_single_process(golden, name, owner):
    import paper_2003_02585_b200 as hs
    z = golden(name)
    single = hs.DdmSolver(_setup(hs, z))
    reps1 = []
    U1 = single.ddm_solve(z["b"], int(z["rounds"]), reps1, True)
    del single
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, name, owner, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r[0], r[1:]) for r in (q.get(timeout=600) for _ in range(2)))
    for p in procs:
        p.join(timeout=120)
    for r in (0, 1):
        U, cnt, nrm, res_r, info = res[r]
        assert not isinstance(U, str), U
        assert np.array_equal(U, U1), f"rank {r}: max |diff| {np.max(np.abs(U - U1)):.3e}"
        assert cnt == [[getattr(x, k) for k in COUNTERS] for x in reps1]
        for a, b in zip(nrm, reps1):
            np.testing.assert_allclose(a, b.sweep_contrib_norm, rtol=1e-12)
        for a, b in zip(res_r, reps1):
            assert a == b.round_residuals
        assert info[1] == 2 and info[2] >= 1 and info[3] > 0
    assert np.array_equal(U1, z["u"]) or float(np.linalg.norm(U1 - z["u"]) / np.linalg.norm(z["u"])) <= 1e-9
    for p in procs:
        assert p.exitcode == 0


def _gpu_worker_case(rank, world, port, case, q):
    import torch
    import torch.distributed as dist
    import paper_2003_02585_b200 as hs
    from paper_2003_02585_b200.multi import PartitionedDdmSolver
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        setup, b, kind = _case(hs, case)
        s = PartitionedDdmSolver(setup, device=0)
        if kind != "gmres":
            b = s.scale_source(b)
        if kind == "gmres":
            g = s.gmres(b, 1e-8, 30, 1)
            q.put((rank, g.x, g.iterations, g.history))
        else:
            reps = []
            U = s.ddm_solve(b, 1, reps, True)
            q.put((rank, U, [[getattr(r, k) for k in COUNTERS] for r in reps], None))
    except Exception as e:
        q.put((rank, repr(e), None, None))
        raise
    finally:
        dist.destroy_process_group()


def _case(hs, case):
    from paper_2003_02585_b200 import sources
    if case == "gmres":  # tests/golden/gmres_2d: GMRES preconditioned by partitioned sweeps
        z = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "gmres_2d.npz"))
        med = ast.literal_eval(str(z["medium"]))
        setup = hs.ProblemSetup(2, [int(z["n"])] * 2, list(z["parts"]),
                                hs.Medium("constant", kappa=med["media.kappa"]), pml_width=int(z["pad"]))
        return setup, z["b"], "gmres"
    # BASELINE config 1 geometry (256^2, 4x4, PML 20, omega = 2 pi 16), two seeded sources
    setup = hs.ProblemSetup(2, [256, 256], [4, 4], hs.Medium("constant", kappa=2 * math.pi * 16), pml_width=20)
    lo, hi = [-20, -20], [276, 276]  # the padded global grid
    f = sources.gaussian_sources(2, lo, hi, [1 / 256] * 2, [0.0, 0.0], sources.seeded_centers(7, 2, 2), 2.0 / 256)
    return setup, f, "ddm"


@pytest.mark.gpu
@pytest.mark.parametrize("case,world", [("c1", 4), ("gmres", 2)])
def test_partitioned_cases(case, world):
    import paper_2003_02585_b200 as hs
    setup, b, kind = _case(hs, case)
    single = hs.DdmSolver(setup)
    if kind == "gmres":
        g1 = single.gmres(b, 1e-8, 30, 1)
    else:
        b = single.scale_source(b)
        reps1 = []
        U1 = single.ddm_solve(b, 1, reps1, True)
    del single
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker_case, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict((r[0], r[1:]) for r in (q.get(timeout=600) for _ in range(world)))
    for p in procs:
        p.join(timeout=120)
    for r in range(world):
        x, a, h = res[r]
        assert not isinstance(x, str), x
        if kind == "gmres":
            assert np.array_equal(x, g1.x) and a == g1.iterations and h == g1.history
        else:
            assert np.array_equal(x, U1)
            assert a == [[getattr(x1, k) for k in COUNTERS] for x1 in reps1]
    for p in procs:
        assert p.exitcode == 0
