"""Multi-GPU plumbing for the frame-parallel render.

Frames (distinct (camera, t) pairs) are independent given a replicated scene
and replicated key-frame masks, so the data path has no collective: frame f
goes to rank f mod N.  torch.distributed (NCCL on GPUs, gloo in the CPU tests)
is used only for setup and reporting:

* ``broadcast_scene``  scene arrays from rank 0 to every rank;
* ``share_keyframe_masks``  key-frame k is built by rank k mod N, then one
  all-reduce (sum of disjoint rows; no bitwise reduction is needed);
* ``gather_frames``  optional collection of rendered frames on rank 0;
* ``max_over_ranks``  the job time is the slowest rank's device time.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def world():
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def shard_frames(frames: list, rank: int, world_size: int) -> list:
    """Round-robin partition of the sequence: frame f -> rank f mod N."""
    return [x for i, x in enumerate(frames) if i % world_size == rank]


def broadcast_scene(tensors: dict, src: int = 0) -> dict:
    """In-place broadcast of every scene tensor from `src` (dict order is the
    protocol: all ranks must pass the same keys with the same shapes)."""
    _, n = world()
    if n > 1:
        for k in sorted(tensors):
            dist.broadcast(tensors[k], src=src)
    return tensors


def share_keyframe_masks(n_keyframes: int, words: int, build, device) -> torch.Tensor:
    """masks[k] = build(k) computed on rank k mod N, replicated everywhere.

    `build(k, out)` fills the int32 row `out` (ceil(N/32) words).  Rows are
    disjoint across ranks, so a SUM all-reduce reproduces every row exactly."""
    rank, n = world()
    masks = torch.zeros((n_keyframes, words), dtype=torch.int32, device=device)
    for k in range(n_keyframes):
        if k % n == rank:
            build(k, masks[k])
    if n > 1:
        # int32 sum of one non-zero row and zeros is exact for every bit pattern
        dist.all_reduce(masks, op=dist.ReduceOp.SUM)
    return masks


def max_over_ranks(value: float, device) -> float:
    _, n = world()
    if n == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device) -> float:
    _, n = world()
    if n == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def gather_frames(frames: torch.Tensor, dst: int = 0):
    """Collect equally-shaped per-rank frame batches (K,3,H,W) on `dst`.
    Returns the list of per-rank batches on dst, None elsewhere."""
    rank, n = world()
    if n == 1:
        return [frames]
    out = [torch.empty_like(frames) for _ in range(n)] if rank == dst else None
    dist.gather(frames, gather_list=out, dst=dst)
    return out
