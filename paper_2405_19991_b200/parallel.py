"""Slab decomposition of the periodic cell for multi-GPU runs.

The grid is cut along axis 0 (x, the slowest C-order axis) into contiguous
slabs, one per rank.  Every stencil on the path (operator and smoother,
macro loads, tensor/sensitivity, filter, restriction, prolongation) reaches one
plane in x, so a slab plus one ghost plane on each side is enough; the ghost
planes are refreshed with point-to-point sends to the two neighbours (NCCL over
NVLink on B200 nodes, gloo on CPU for tests).  The only global couplings are
scalars (PCG dot products, tensor sums, OC candidate means, governor means),
which are all-reduced.  Coarse levels whose slabs would get thinner than
``min_planes`` are agglomerated: every rank gathers the level and runs the rest
of the V-cycle redundantly, keeping its own slab of the correction.

Round 1 ships the plan, the exchange and the agglomeration primitives with
world-size-2 gloo tests (tests/test_parallel_gloo.py); ``bench.py`` under
torchrun runs replicas.  The device solver consumes this plan next.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class SlabLevel:
    dims: tuple          # global level dims
    distributed: bool    # slab-partitioned (True) or agglomerated on every rank (False)
    x0: int              # first owned plane (global index; 0 when agglomerated)
    x1: int              # one past the last owned plane (nx when agglomerated)

    @property
    def nx_local(self) -> int:
        return self.x1 - self.x0


def level_dims(dims, coarse_target: int = 64):
    """The reference level chain (solver.py:217-231)."""
    chain = [tuple(int(n) for n in dims)]
    while int(np.prod(chain[-1])) > coarse_target and all(n % 2 == 0 for n in chain[-1] if n > 1):
        chain.append(tuple(n // 2 if n > 1 else 1 for n in chain[-1]))
    return chain


class SlabPlan:
    """Which x planes each rank owns on every multigrid level."""

    def __init__(self, dims, world: int, rank: int, min_planes: int = 2, coarse_target: int = 64):
        if world < 1 or not (0 <= rank < world):
            raise ValueError(f"bad rank {rank} of {world}")
        self.world, self.rank = world, rank
        self.levels: list[SlabLevel] = []
        distributed = world > 1
        for d in level_dims(dims, coarse_target):
            nx = d[0]
            if distributed and (nx % world or nx // world < min_planes):
                distributed = False        # agglomerate from here down
            if distributed:
                w = nx // world
                self.levels.append(SlabLevel(d, True, rank * w, (rank + 1) * w))
            else:
                self.levels.append(SlabLevel(d, False, 0, nx))
        if world > 1 and not self.levels[0].distributed:
            raise ValueError(f"dims {tuple(dims)} cannot be split into {world} slabs of >= {min_planes} planes")

    @property
    def agglomeration_level(self) -> int:
        """First level that every rank holds in full (len(levels) if none)."""
        for i, lev in enumerate(self.levels):
            if not lev.distributed:
                return i
        return len(self.levels)

    def left(self) -> int:
        return (self.rank - 1) % self.world

    def right(self) -> int:
        return (self.rank + 1) % self.world


def with_ghosts(local, nghost: int = 1):
    """Allocate a copy of a slab (x leading) with ghost planes on both sides."""
    t = local
    shape = list(t.shape)
    shape[0] += 2 * nghost
    out = t.new_zeros(shape)
    out[nghost:nghost + t.shape[0]] = t
    return out


def halo_exchange(padded, plan: SlabPlan, group=None):
    """Refresh the two ghost planes of a padded slab (axis 0) from the periodic neighbours.

    padded[0] <- left neighbour's last owned plane; padded[-1] <- right neighbour's first.
    Uses point-to-point isend/irecv (NCCL for CUDA tensors, gloo for CPU tensors)."""
    import torch.distributed as dist
    if plan.world == 1:
        padded[0] = padded[-2]
        padded[-1] = padded[1]
        return padded
    first = padded[1].contiguous()
    last = padded[-2].contiguous()
    recv_left = padded.new_empty(first.shape)
    recv_right = padded.new_empty(first.shape)
    ops = [dist.P2POp(dist.isend, last, plan.right(), group),
           dist.P2POp(dist.isend, first, plan.left(), group),
           dist.P2POp(dist.irecv, recv_left, plan.left(), group),
           dist.P2POp(dist.irecv, recv_right, plan.right(), group)]
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    padded[0] = recv_left
    padded[-1] = recv_right
    return padded


def allreduce_sum(t, group=None):
    """Sum small scalar vectors over ranks (PCG dots, tensor sums, OC means)."""
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def gather_level(local, plan: SlabPlan, group=None):
    """Agglomerate a distributed level: every rank receives the full field (x leading)."""
    import torch
    import torch.distributed as dist
    if plan.world == 1:
        return local
    parts = [torch.empty_like(local) for _ in range(plan.world)]
    dist.all_gather(parts, local.contiguous(), group=group)
    return torch.cat(parts, dim=0)


def owned_part(full, plan: SlabPlan, level: int = 0):
    lev = plan.levels[level]
    return full[lev.x0:lev.x1]
