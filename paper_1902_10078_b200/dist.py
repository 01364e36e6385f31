"""Batch partitioner and the config-3 scalar all-reduce.

Matrices are independent, so a batch shards over ranks as contiguous slices
of whole matrices with no data-path collective.  The only exchange is the
learning step's two scalars -- the summed log-likelihood and the summed
d tau2 -- reduced with one all-reduce (NCCL over NVLink on GPUs, gloo in the
CPU tests).  The per-matrix gradients L_bar stay on the rank that owns the
matrix.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_bounds(batch: int, world: int, rank: int) -> tuple[int, int]:
    """[start, stop) of the matrices rank `rank` owns: contiguous, sizes
    differing by at most one (the first batch % world ranks take one more)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(batch, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def reduce_totals(per_matrix: list[torch.Tensor], group=None) -> torch.Tensor:
    """Sum each per-matrix vector locally, then all-reduce the sums across
    ranks in one collective (a 2 x fp64 all-reduce for config 3)."""
    local = torch.stack([v.sum() for v in per_matrix]).to(torch.float64)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(local, op=dist.ReduceOp.SUM, group=group)
    return local


def marginal_likelihood_grad_sharded(L, y, tau2: float, group=None, check: bool = True, out=None):
    """Config-3 step on this rank's shard (the matrices shard_bounds gave it):
    local fused sweeps, then the global (sum loss, sum tau2_bar) -- the one
    16-byte all-reduce of the step.  ``out`` = preallocated (loss, l_bar,
    tau2_bar, status) as for api.marginal_likelihood_grad (bench.py reuses
    them across steps).  Returns (totals[2], loss[B_local], l_bar, tau2_bar[B_local])."""
    from .api import marginal_likelihood_grad

    loss, l_bar, t_bar = marginal_likelihood_grad(L, y, tau2, check=check, out=out)
    return reduce_totals([loss, t_bar], group), loss, l_bar, t_bar
