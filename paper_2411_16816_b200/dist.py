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


def allreduce_grads(grads, group=None):
    """In-place SUM of the contiguous 27*N-float SceneParamGrads buffer over all ranks (one collective per step).
    `grads` is a torch tensor: on the GPU it is the buffer bound with splatb200_grads_bind_device, so NCCL reduces the
    kernels' output in place."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
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
