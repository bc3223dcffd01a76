"""Multi-GPU plumbing of the path: which (frame, sensor) work items a rank renders, and the one collective the path
has — the sum of the per-Gaussian SceneParamGrads over ranks.

The path shards over independent frames with the scene replicated; there is no intra-render split.
One process per GPU; `torch.distributed` is plumbing only (NCCL over NVLink on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

from typing import List, Sequence


def assign_frames(n_frames: int, world: int, rank: int, costs: Sequence[float] | None = None) -> List[int]:
    """Whole frames to ranks. Without costs: round-robin (frame f -> rank f % world), which keeps one compose per
    frame per GPU. With per-frame costs (e.g. the previous iteration's intersection counts): longest-processing-time
    greedy, deterministic on every rank (ties by frame index)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("need 0 <= rank < world")
    if costs is None:
        return [f for f in range(n_frames) if f % world == rank]
    if len(costs) != n_frames:
        raise ValueError("one cost per frame")
    load = [0.0] * world
    mine: List[int] = []
    for f in sorted(range(n_frames), key=lambda k: (-float(costs[k]), k)):
        r = min(range(world), key=lambda k: (load[k], k))
        load[r] += float(costs[f])
        if r == rank:
            mine.append(f)
    return sorted(mine)


def init_comm(ctx, group=None):
    """Create the library's own NCCL communicator over the ranks of `group` (torch.distributed is only the out-of-band
    channel for the 128-byte id, exactly what MPI_Bcast is in a C++ trainer). Returns the world size (1: nothing to do)."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return 1
    from . import api
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    box = [api.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    ctx.comm_init(box[0], rank, world)
    return world


def allreduce_grads(grads, group=None, ctx=None):
    """In-place SUM of the contiguous 27*N-float SceneParamGrads buffer over all ranks (one collective per step).
    With a ctx that owns a communicator (init_comm) the collective is the library's splatb200_allreduce_grads: ncclAllReduce
    on the ctx stream, ordered after the view streams, ActorGrad slots included. Otherwise `grads` (the torch tensor bound
    with splatb200_grads_bind_device) is reduced by torch.distributed — the CPU / gloo tests and callers that keep
    their own process group."""
    import torch.distributed as dist
    if ctx is not None and ctx.comm_world > 1:
        ctx.allreduce_grads()
        return grads
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        if ctx is not None:
            ctx.join()
        dist.all_reduce(grads, op=dist.ReduceOp.SUM, group=group)
    return grads


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Timing rule: a multi-GPU number is the MAX over ranks."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def shard_range(total: int, world: int, rank: int, align: int = 4):
    """[lo, hi) of a flat buffer of `total` floats owned by `rank`: equal shards (the last one may be shorter), aligned to
    `align` elements so that 128-bit accesses stay aligned."""
    per = -(-total // world)
    per = -(-per // align) * align
    lo = min(total, rank * per)
    return lo, min(total, lo + per)


def sharded_optimizer_step(ctx, grads, params_flat, cfg, step, group=None):
    """the optimizer step fused with the gradient collective. Instead of all-reducing the 27*N-float
    SceneParamGrads buffer and stepping everywhere, every rank (1) reduce-scatters it — each rank ends up with the SUM of
    its own shard —, (2) agrees on the groups to skip (a non-finite gradient anywhere skips the group everywhere: one
    6-int all-reduce), (3) runs Adam on its shard only (moments are only ever touched there: optimizer state and work
    divide by the world size), (4) all-gathers the updated parameters. Same bytes on the wire as the all-reduce.
    `grads`: the torch tensor bound with ctx.bind_grads_device; `params_flat`: ONE torch tensor holding the scene in the
    gradient buffer's layout [mean 3N | scale_log 3N | quat 4N | opacity N | color 3N | feature d_f N], whose slices are
    bound with ctx.bind_scene_device. Returns the skipped groups."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank(group) if world > 1 else 0
    if ctx.comm_world > 1:     # the library's own communicator: the whole step is one C-ABI call
        return ctx.sharded_optimizer_step(cfg, step)
    # torch collectives run on torch's current stream, the library's kernels on the ctx stream (and the view streams):
    # order the collectives after the backward kernels, and the library's reads after the collectives
    ctx.join()
    if grads.is_cuda:
        ctx.sync()
    total = grads.numel()
    lo, hi = shard_range(total, world, rank)
    per = shard_range(total, world, 0)[1]
    gloo = world > 1 and dist.get_backend(group) == "gloo"   # CPU tests: gloo has no reduce-scatter -> all-reduce, keep the shard
    if gloo:
        dist.all_reduce(grads, op=dist.ReduceOp.SUM, group=group)
    elif world > 1:
        if per * world != total:       # reduce_scatter_tensor wants equal shards: pad through a staging copy
            padded = torch.zeros(per * world, dtype=grads.dtype, device=grads.device)
            padded[:total] = grads
            out = torch.empty(per, dtype=grads.dtype, device=grads.device)
            dist.reduce_scatter_tensor(out, padded, op=dist.ReduceOp.SUM, group=group)
            grads[lo:hi] = out[:hi - lo]
        else:
            dist.reduce_scatter_tensor(grads[lo:hi], grads, op=dist.ReduceOp.SUM, group=group)
    if grads.is_cuda:
        torch.cuda.current_stream(grads.device).synchronize()
    flags = torch.tensor(ctx.grads_nonfinite_range(lo, hi), dtype=torch.int32, device=grads.device)
    if world > 1:
        dist.all_reduce(flags, op=dist.ReduceOp.MAX, group=group)
    skip = [int(x) for x in flags.tolist()]
    ctx.optimizer_step_range(cfg, step, lo, hi, skip_groups=skip)
    if params_flat is not None and params_flat.is_cuda:
        ctx.sync()      # the all-gather below (torch's stream) reads what k_adam wrote on the ctx stream
    if gloo:
        send = torch.zeros(per, dtype=params_flat.dtype)
        send[:hi - lo] = params_flat[lo:hi]
        parts = [torch.empty(per, dtype=params_flat.dtype) for _ in range(world)]
        dist.all_gather(parts, send, group=group)
        params_flat.copy_(torch.cat(parts)[:total])
    elif world > 1:
        if per * world != total:
            send = torch.zeros(per, dtype=params_flat.dtype, device=params_flat.device)
            send[:hi - lo] = params_flat[lo:hi]
            recv = torch.empty(per * world, dtype=params_flat.dtype, device=params_flat.device)
            dist.all_gather_into_tensor(recv, send, group=group)
            params_flat.copy_(recv[:total])
        else:
            dist.all_gather_into_tensor(params_flat, params_flat[lo:hi].clone(), group=group)
    return [k for k in range(6) if skip[k]]
