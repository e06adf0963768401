"""Data-parallel plumbing of the TMC hot path.

Datapoints are independent problems (each carries its own K proposal samples per latent),
so rank r of W owns a contiguous slice of the global batch and every per-datapoint output stays
local.  The one exchange is a SUM all-reduce of the objective J = sum_b logp[b] (and, in a training
step, of shared-parameter gradients), issued on the caller's process group: NCCL over NVLink on
the GPU box, gloo in the CPU tests.  No kernel code lives here.
"""
from __future__ import annotations

from typing import List, Optional


def shard_ids(B: int, rank: int, world: int) -> List[int]:
    """Global datapoint ids owned by `rank` (contiguous, equal sizes; B must divide evenly)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank/world {rank}/{world}")
    if B % world:
        raise ValueError(f"B={B} is not divisible by world={world}")
    per = B // world
    return list(range(rank * per, (rank + 1) * per))


def reduce_objective(local_sum, group=None):
    """In-place SUM all-reduce of a float64 tensor holding this rank's partial objective(s)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(local_sum, op=dist.ReduceOp.SUM, group=group)
    return local_sum


def gather_per_datapoint(local, group=None):
    """All-gather equal-sized per-datapoint tensors into global batch order (rank-major)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return local
    parts = [torch.empty_like(local) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, local.contiguous(), group=group)
    return torch.cat(parts, dim=0)


def data_parallel_estimate(graph, inputs, ws, logp, grads, obj, dlogp=None, group=None, stream=None):
    """One data-parallel step of the hot path on this rank's shard: the TMC
    forward and reverse pass of the local datapoints (libtmc; no communication), then the objective
    obj[0] = sum_b logp[b] (fp64) SUM all-reduced over the group.  graph.B = the local batch."""
    import torch
    import paper_1806_08593_b200 as tmc
    tmc.tmc_estimate(graph, inputs, logp, dlogp, grads, ws, stream)
    torch.sum(logp, dim=0, keepdim=True, out=obj[:1])
    return reduce_objective(obj, group)


def max_over_ranks(values, group=None):
    """In-place MAX all-reduce (device timings: the job time is the slowest rank's)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(values, op=dist.ReduceOp.MAX, group=group)
    return values


# ---------------------------------------------------------------- shared-root star
# a global latent theta (K_theta samples) shared by N data points.  The data points are
# sharded over ranks; each rank's graph is the root plus its own children.  The root's incoming
# messages are additive in the log domain, so ONE all-reduce of a [B][K_theta + 1] fp64 vector per
# step joins the shards (include/tmc.h, tmc_forward_children / tmc_forward_root).
def shard_children(N: int, rank: int, world: int) -> List[int]:
    """Global ids (0-based) of the data points rank `rank` holds: contiguous blocks, the first
    N % world ranks one larger; a rank may hold none when N < world."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank/world {rank}/{world}")
    base, extra = divmod(N, world)
    start = rank * base + min(rank, extra)
    return list(range(start, start + base + (1 if rank < extra else 0)))


def exchange_root_messages(root_msg, group=None):
    """The one data-path collective of the shared-root star: in-place SUM all-reduce of the
    shard's root messages (fp64 residual sums and offset sums add across shards)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(root_msg, op=dist.ReduceOp.SUM, group=group)
    return root_msg


def shared_root_estimate(graph, inputs, ws, logp, root_msg, grads=None, dlogp=None, group=None, stream=None):
    """One sharded TMC evaluation of a shared-root star: children forward -> all-reduce of the
    root messages -> root elimination (logp, identical on every rank) -> reverse pass of this
    rank's latents under the global root marginal.  graph.direction must be TMC_DIR_UP."""
    import paper_1806_08593_b200 as tmc
    tmc.tmc_forward_children(graph, inputs, root_msg, ws, stream)
    exchange_root_messages(root_msg, group)
    tmc.tmc_forward_root(graph, inputs, root_msg, logp, ws, stream)
    if grads is not None:
        tmc.tmc_backward(graph, inputs, ws, dlogp, grads, stream=stream)
    return logp
