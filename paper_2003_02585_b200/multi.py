"""Multi-GPU plumbing: one process per GPU.

Two ways to spread the DDM hot path over ranks:

* **RHS sharding** (`shard_rhs`, `solve_sharded`). Right-hand sides are independent units (each
  one is a full set of diagonal sweeps against the same resident subdomain factors), so every
  rank solves its own block of RHS against its own device-resident factorization: no collective
  touches the data path. This is what `bench.py --gpus N` measures (weak scaling).
* **Subdomain partitioning** (`PartitionedDdmSolver`). Each rank factorizes and
  solves only the subdomains it owns, so one problem's factors are spread over the GPUs (C5's
  106 GB of packed factors). After each macro-step of the sweep schedule the library hands this
  module one message per neighbouring rank (traces deposited for that rank's subdomains and
  solution values on its home nodes); they travel as NCCL send/recv pairs ordered on the
  library's stream (no host synchronisation), or, for gloo groups, staged through host memory.
"""
from __future__ import annotations

import ctypes
import os
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

from . import _lib as L
from .api import DdmSolver, ProblemSetup, _raise


def shard_rhs(n_total: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous block of RHS indices owned by `rank` (sizes differ by at most one)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(n_total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def solve_sharded(solve: Callable[[np.ndarray], np.ndarray], B: np.ndarray, rank: int, world: int,
                  gather: bool = True, group=None):
    """Solves this rank's shard of B (R_total, N) with `solve` ((r, N) -> (r, N)); with gather,
    returns the full (R_total, N) solution on every rank (torch.distributed all_gather_object),
    else only the local shard."""
    lo, hi = shard_rhs(B.shape[0], rank, world)
    local = solve(B[lo:hi]) if hi > lo else np.zeros((0, B.shape[1]), dtype=B.dtype)
    if not gather or world == 1:
        return local
    import torch.distributed as dist
    parts = [None] * world
    dist.all_gather_object(parts, (lo, local), group=group)
    out = np.zeros_like(B)
    for plo, arr in parts:
        out[plo:plo + arr.shape[0]] = arr
    return out


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (device timing is reported as the max over ranks)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------------------------
# subdomain partitioning

def partition_owners(dim: int, counts: Sequence[int], world: int) -> List[int]:
    """The library's balanced default ownership (hs_partition_owners), flattened id order."""
    c = (ctypes.c_int * 3)(*(list(counts) + [1, 1, 1])[:3])
    nsub = int(np.prod(list(counts)[:dim]))
    o = (ctypes.c_int * nsub)()
    rc = L.lib().hs_partition_owners(int(dim), c, int(world), o)
    if rc:
        _raise(rc)
    return list(o)


def partition_traffic(dim: int, counts: Sequence[int], rounds: int, world: int, owner: Sequence[int]):
    """(macro_steps, makespan_tasks, cross_faces, traces[world][world]) of an ownership."""
    c = (ctypes.c_int * 3)(*(list(counts) + [1, 1, 1])[:3])
    o = (ctypes.c_int * len(owner))(*owner)
    ms, mk, cf = ctypes.c_int(), ctypes.c_int64(), ctypes.c_int64()
    tr = (ctypes.c_int64 * (world * world))()
    rc = L.lib().hs_partition_traffic(int(dim), c, int(rounds), int(world), o, ctypes.byref(ms), ctypes.byref(mk),
                                      ctypes.byref(cf), tr)
    if rc:
        _raise(rc)
    return ms.value, mk.value, cf.value, np.array(list(tr), dtype=np.int64).reshape(world, world)


class _DevArray:
    """A raw device pointer as a torch-importable array (__cuda_array_interface__, no copy)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f8", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def exchange_host(send: np.ndarray, recv: np.ndarray, peers, soff, scnt, roff, rcnt, group=None):
    """One exchange round over host buffers (gloo): message i goes to / comes from peers[i]."""
    import torch
    import torch.distributed as dist
    st = torch.from_numpy(send)
    rt = torch.from_numpy(recv)
    reqs = []
    for i, p in enumerate(peers):
        if scnt[i]:
            reqs.append(dist.isend(st[soff[i]:soff[i] + scnt[i]], int(p), group=group))
        if rcnt[i]:
            reqs.append(dist.irecv(rt[roff[i]:roff[i] + rcnt[i]], int(p), group=group))
    for r in reqs:
        r.wait()


def _same_nccl_as_torch():
    """Point the library's dlopen at the libnccl PyTorch links (the nvidia-nccl wheel) unless the
    caller chose one (HS_NCCL_LIB): a process holds one object per soname, so loading the system
    libnccl.so.2 first would leave a later `import torch` bound to a different, older build."""
    if os.environ.get("HS_NCCL_LIB"):
        return
    try:
        import importlib.util
        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        return
    for d in (spec.submodule_search_locations or []) if spec else []:
        cand = os.path.join(d, "lib", "libnccl.so.2")
        if os.path.exists(cand):
            os.environ["HS_NCCL_LIB"] = cand
            return


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId from the library's own NCCL binding (hs_nccl_unique_id)."""
    _same_nccl_as_torch()
    buf = (ctypes.c_ubyte * 128)()
    rc = L.lib().hs_nccl_unique_id(buf)
    if rc:
        _raise(rc)
    return bytes(buf)


def nccl_version() -> int:
    _same_nccl_as_torch()
    v = ctypes.c_int()
    rc = L.lib().hs_nccl_version(ctypes.byref(v))
    if rc:
        _raise(rc)
    return v.value


class NcclDdmSolver(DdmSolver):
    """DdmSolver partitioned over `world` ranks (one GPU each) with the library's native NCCL
    transport (hs_ddm_create_nccl): the exchange and reductions are issued by the library on its
    solver stream, no Python on the data path, applications CUDA-graph captured. `uid` is the
    128-byte id from nccl_unique_id() on one rank, distributed to all by the caller."""

    def __init__(self, setup: ProblemSetup, device: int, rank: int, world: int, uid: bytes,
                 owner: Optional[Sequence[int]] = None):
        self._rank, self._world = int(rank), int(world)
        self._uid = (ctypes.c_ubyte * 128)(*uid)
        self._owner = None if owner is None else (ctypes.c_int * len(owner))(*owner)
        super().__init__(setup, device)

    def _create(self, p, device, h, sub, piv):
        _same_nccl_as_torch()
        return L.lib().hs_ddm_create_nccl(ctypes.byref(p), device, self._rank, self._world, self._owner, self._uid,
                                          ctypes.byref(h), ctypes.byref(sub), ctypes.byref(piv))

    def partition_info(self):
        """(rank, world, owned subdomains, doubles sent per application, messages per application)."""
        r, w, o = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        sd, ms = ctypes.c_int64(), ctypes.c_int64()
        rc = L.lib().hs_ddm_partition_info(self._h, ctypes.byref(r), ctypes.byref(w), ctypes.byref(o),
                                           ctypes.byref(sd), ctypes.byref(ms))
        if rc:
            _raise(rc)
        return r.value, w.value, o.value, sd.value, ms.value


def make_partitioned(setup: ProblemSetup, device: int = 0, group=None, owner: Optional[Sequence[int]] = None,
                     transport: str = "auto"):
    """The partitioned solver for a torch.distributed group: the native NCCL transport for NCCL
    groups (transport "auto" / "nccl"; the id travels once through the group at construction),
    the caller-callback transport otherwise ("callback"; gloo groups stage through host memory)."""
    import torch.distributed as dist
    native = transport == "nccl" or (transport == "auto" and dist.get_backend(group) == "nccl")
    if not native:
        return PartitionedDdmSolver(setup, device, group, owner)
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    box = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    return NcclDdmSolver(setup, device, rank, world, box[0], owner)


class PartitionedDdmSolver(DdmSolver):
    """DdmSolver whose subdomains are spread over the ranks of a torch.distributed group
    (hs_ddm_create_partitioned) with a caller-supplied transport: this class's callbacks move the
    library's messages through torch.distributed (gloo groups stage through host memory). NCCL
    groups should use make_partitioned / NcclDdmSolver, whose transport is native. Every rank
    constructs it with the same setup and calls ddm_solve / ddm_solve_device collectively with the
    same b; every rank receives the full u."""

    def __init__(self, setup: ProblemSetup, device: int = 0, group=None, owner: Optional[Sequence[int]] = None):
        import torch
        import torch.distributed as dist
        self._group = group
        self._rank = dist.get_rank(group)
        self._world = dist.get_world_size(group)
        self._nccl = dist.get_backend(group) == "nccl"
        self._device = torch.device("cuda", device)
        self._owner = None if owner is None else (ctypes.c_int * len(owner))(*owner)
        self._error = None
        self._xcb = L.EXCHANGE_FN(self._exchange)
        self._arcb = L.ALLREDUCE_FN(self._allreduce)
        super().__init__(setup, device)

    def _create(self, p, device, h, sub, piv):
        return L.lib().hs_ddm_create_partitioned(ctypes.byref(p), device, self._rank, self._world, self._owner,
                                                 self._xcb, self._arcb, None, ctypes.byref(h), ctypes.byref(sub),
                                                 ctypes.byref(piv))

    def _peer(self, p):  # group rank -> global rank (torch.distributed p2p takes global ranks)
        import torch.distributed as dist
        return dist.get_global_rank(self._group, p) if self._group is not None else p

    def _exchange(self, user, npeers, peers, soff, scnt, roff, rcnt, send_ptr, recv_ptr, stream):
        try:
            import torch
            import torch.distributed as dist
            pe = [self._peer(peers[i]) for i in range(npeers)]
            so = [soff[i] for i in range(npeers)]
            sc = [scnt[i] for i in range(npeers)]
            ro = [roff[i] for i in range(npeers)]
            rc = [rcnt[i] for i in range(npeers)]
            ns, nr = max(o + c for o, c in zip(so, sc)), max(o + c for o, c in zip(ro, rc))
            ext = torch.cuda.ExternalStream(stream, device=self._device)
            send = torch.as_tensor(_DevArray(send_ptr, max(ns, 1)), device=self._device)
            recv = torch.as_tensor(_DevArray(recv_ptr, max(nr, 1)), device=self._device)
            if self._nccl:  # device-to-device over NVLink, ordered on the library's stream
                with torch.cuda.stream(ext):
                    ops = []
                    for i, p in enumerate(pe):
                        if sc[i]:
                            ops.append(dist.P2POp(dist.isend, send[so[i]:so[i] + sc[i]], p, self._group))
                        if rc[i]:
                            ops.append(dist.P2POp(dist.irecv, recv[ro[i]:ro[i] + rc[i]], p, self._group))
                    for w in dist.batch_isend_irecv(ops):
                        w.wait()
            else:  # host-staged (gloo)
                ext.synchronize()
                hs = send[:ns].cpu().numpy() if ns else np.zeros(0)
                hr = np.zeros(nr)
                exchange_host(hs, hr, pe, so, sc, ro, rc, self._group)
                if nr:
                    with torch.cuda.stream(ext):
                        recv[:nr].copy_(torch.from_numpy(hr))
                    ext.synchronize()
            return 0
        except Exception as e:  # reported by the C-ABI as HS_ERR_CUDA; kept for re-raise
            self._error = e
            return 1

    def _allreduce(self, user, ptr, count, stream):
        try:
            import torch
            import torch.distributed as dist
            ext = torch.cuda.ExternalStream(stream, device=self._device)
            t = torch.as_tensor(_DevArray(ptr, count), device=self._device)
            if self._nccl:
                with torch.cuda.stream(ext):
                    dist.all_reduce(t, group=self._group)
            else:
                ext.synchronize()
                h = t.cpu()
                dist.all_reduce(h, group=self._group)
                with torch.cuda.stream(ext):
                    t.copy_(h)
                ext.synchronize()
            return 0
        except Exception as e:
            self._error = e
            return 1

    def partition_info(self):
        """(rank, world, owned subdomains, doubles sent per application, messages per application)."""
        r, w, o = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        sd, ms = ctypes.c_int64(), ctypes.c_int64()
        rc = L.lib().hs_ddm_partition_info(self._h, ctypes.byref(r), ctypes.byref(w), ctypes.byref(o),
                                           ctypes.byref(sd), ctypes.byref(ms))
        if rc:
            _raise(rc)
        return r.value, w.value, o.value, sd.value, ms.value
