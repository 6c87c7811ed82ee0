"""Multi-GPU plumbing: one process per GPU, RHS sharded across ranks.

Right-hand sides are independent units of the DDM hot path (each one is a full set of diagonal
sweeps against the same resident subdomain factors), so the B200 design scales by giving every
rank its own contiguous block of RHS and its own device-resident factorization: no collective
touches the data path. Collectives appear only for (a) the max-over-ranks timing and (b) an
optional gather of the solutions to one rank. See DESIGN.md "Multi-GPU".
"""
from __future__ import annotations

from typing import Callable, Tuple

import numpy as np


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
