"""Keyframe-sharded densification of a sequence: one process per GPU, NCCL only for the cloud.

The reference is single-process; this module is the multi-GPU design on
top of the same stages.  The reference's stage C filters the centre of every full
consistency window and feeds it to the fusion FIFO, so for D depth results d_0..d_{D-1}

    filtered centres  c = half .. D-1-half            (half = window // 2)
    fused frame c     = valid pixels of filtered c, minus duplicates of the filtered frames
                        c+1 .. c+buffer-1 that exist

Every fused frame therefore depends on the depth results [c-half, c+buffer-1+half] only, and the
per-keyframe PatchMatch seeds are per keyframe, so contiguous blocks of centres can
be produced by different ranks with a halo of depth maps recomputed on each side and no
data-path collective.  The only exchange is the final cloud: rank-ordered, exact-size
send/recv to one rank (an all-gather-v), which keeps the reference's "oldest keyframe first"
output order (T/test_pipeline.py:320-321).

The warp-initialisation chain is sequential by nature; a shard restarts it at the
first depth result of its halo.  With ``warp=False`` shards reproduce the single-stream result
bit for bit; with ``warp=True`` only the initialisation of the restarted frames differs.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .pipeline import (
    ConsistencyConfig,
    DepthStage,
    DeviceDepthResult,
    DeviceFusedCloud,
    FusedCloud,
    FusionBuffer,
    FusionConfig,
    consistency_filter_device,
)


@dataclass(frozen=True)
class ShardPlan:
    """Work of one rank over a sequence of ``n_results`` depth results."""

    rank: int
    world: int
    centres: range   # filtered / fused frames this rank emits (indices into the depth results)
    filtered: range  # frames it must filter (its centres + the newer frames fusion compares with)
    depth: range     # depth results it must compute (filtered frames + consistency halo)


def plan_shards(n_results: int, world: int, window: int = 5, buffer: int = 4) -> list:
    """Contiguous, balanced blocks of fused frames with their halos (empty ranges when the
    sequence is shorter than one consistency window)."""
    if world < 1:
        raise ValueError(f"world size must be >= 1, got {world}")
    half = window // 2
    first, last = half, n_results - (window - 1 - half)  # centres are [first, last)
    n = max(0, last - first)
    plans = []
    for r in range(world):
        a = first + (n * r) // world
        b = first + (n * (r + 1)) // world
        if a >= b:
            plans.append(ShardPlan(r, world, range(a, a), range(a, a), range(a, a)))
            continue
        f_hi = min(b + buffer - 1, last)
        plans.append(ShardPlan(r, world, range(a, b), range(a, f_hi),
                               range(a - half, f_hi + (window - 1 - half))))
    return plans


def densify_shard(groups, plan: ShardPlan, stage: DepthStage, consistency: ConsistencyConfig,
                  fusion: FusionConfig) -> list:
    """Run one rank's share.  ``groups[i]`` is the stereo group (or PreparedGroup factory
    result) of depth result i of the whole sequence; returns the DeviceFusedCloud batches of
    ``plan.centres`` in order."""
    if len(plan.centres) == 0:
        return []
    half = consistency.window // 2
    depth = {}
    for i in plan.depth:
        g = groups[i]() if callable(groups[i]) else groups[i]
        depth[i] = stage.process_device(g)
    filtered = {}
    for c in plan.filtered:
        win = [(depth[j].pano, depth[j].pose) for j in range(c - half, c - half + consistency.window) if j != c]
        pano = consistency_filter_device(depth[c].pano, depth[c].pose, win, consistency)
        filtered[c] = DeviceDepthResult(depth[c].id, pano, depth[c].pose, depth[c].image)
    out = []
    for c in plan.centres:
        fb = FusionBuffer(stage.camera, FusionConfig(buffer=fusion.buffer, reproj_px=fusion.reproj_px,
                                                     rel_depth_tol=fusion.rel_depth_tol), device=stage.device)
        # the FIFO state when frame c is the oldest: c plus the newer filtered frames that exist
        newer = [filtered[j] for j in range(c + 1, c + fusion.buffer) if j in filtered]
        fb._frames.extend([filtered[c], *newer])
        out.append(fb._fuse_oldest())
    return out


def _as_tensors(batches, device):
    if batches:
        pts = torch.cat([b.points for b in batches]).to(device)
        col = torch.cat([b.colors for b in batches]).to(device)
        ids = torch.cat([torch.full((len(b),), b.source_id, dtype=torch.int64, device=b.points.device)
                         for b in batches]).to(device)
    else:
        pts = torch.zeros((0, 3), dtype=torch.float64, device=device)
        col = torch.zeros((0, 3), dtype=torch.uint8, device=device)
        ids = torch.zeros((0,), dtype=torch.int64, device=device)
    return pts.contiguous(), col.contiguous(), ids.contiguous()


def gather_cloud(batches, dst: int = 0, group=None, device=None):
    """All-gather-v of the fused cloud to rank ``dst`` in rank order.

    ``batches``: this rank's DeviceFusedCloud list (tensors on the device the process group
    communicates from: CUDA for NCCL, CPU for gloo).  Returns a FusedCloud on ``dst`` and None
    elsewhere.  Without an initialised process group it is a local concatenation."""
    import torch.distributed as dist

    if device is None:
        device = batches[0].points.device if batches else torch.device("cpu")
    pts, col, ids = _as_tensors(batches, device)
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return FusedCloud(pts.cpu().numpy(), col.cpu().numpy(), ids.cpu().numpy())
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    counts = [torch.zeros(1, dtype=torch.int64, device=device) for _ in range(world)]
    dist.all_gather(counts, torch.tensor([pts.shape[0]], dtype=torch.int64, device=device), group=group)
    counts = [int(c.item()) for c in counts]
    if rank != dst:
        if counts[rank]:
            for t in (pts, col, ids):
                dist.send(t, dst, group=group)
        return None
    parts = []
    for r in range(world):
        if r == dst:
            parts.append((pts, col, ids))
            continue
        n = counts[r]
        bufs = (torch.empty((n, 3), dtype=torch.float64, device=device),
                torch.empty((n, 3), dtype=torch.uint8, device=device),
                torch.empty((n,), dtype=torch.int64, device=device))
        if n:
            for t in bufs:
                dist.recv(t, r, group=group)
        parts.append(bufs)
    return FusedCloud(torch.cat([p[0] for p in parts]).cpu().numpy(), torch.cat([p[1] for p in parts]).cpu().numpy(),
                      torch.cat([p[2] for p in parts]).cpu().numpy())


def densify_sequence(groups, stage_factory, consistency: ConsistencyConfig, fusion: FusionConfig,
                     rank: int = 0, world: int = 1, dst: int = 0, group=None):
    """Sharded equivalent of the reference's depth + consistency + fusion stages over a whole
    sequence (P:402-486 without ingest / view filter).  ``stage_factory()`` builds this rank's
    DepthStage.  Returns (FusedCloud on ``dst`` else None, ShardPlan)."""
    plan = plan_shards(len(groups), world, consistency.window, fusion.buffer)[rank]
    stage = stage_factory()
    batches = densify_shard(groups, plan, stage, consistency, fusion)
    return gather_cloud(batches, dst=dst, group=group, device=stage.device), plan
