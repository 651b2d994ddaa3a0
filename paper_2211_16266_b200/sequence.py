"""Keyframe-sharded densification of a sequence: one process per GPU, NCCL for halos and cloud.

The reference is single-process; this module is the multi-GPU design on
top of the same stages.  The reference's stage C filters the centre of every full
consistency window and feeds it to the fusion FIFO, so for D depth results d_0..d_{D-1}

    filtered centres  c = half .. D-1-half            (half = window // 2)
    fused frame c     = valid pixels of filtered c, minus duplicates of the filtered frames
                        c+1 .. c+buffer-1 that exist

The per-keyframe PatchMatch seeds are per keyframe, so the depth results are cut into
contiguous blocks, one per rank, and **every depth map is computed exactly once**.  What the
carried state of the reference's stream needs across a block boundary travels over NVLink as
point-to-point transfers between neighbouring ranks (``exchange_frames``):

  1. raw halo      depth + mask of the ``half`` depth results either side of the block: the
                   consistency window of the block's first / last centres;
  2. filtered halo depth + filtered mask of the first ``buffer - 1`` centres of the next block: the
                   newer frames the fusion FIFO compares the block's last centres with;
  3. the cloud     rank-ordered, exact-size send/recv to one rank (an all-gather-v), which keeps the
                   reference's "oldest keyframe first" output order (T/test_pipeline.py:320-321).

9.2 MB per 1920x960 frame and at most 2 half + buffer - 1 = 7 frames in, 7 out per rank, against
~45 ms of PatchMatch per depth map: the exchange is never on the critical path.

The warp-initialisation chain is sequential by nature; a shard restarts it at the
first depth result of its block (``prime`` extra depth results before the block can be run to
warm the chain up; they are not used for anything else).  With ``warp=False`` shards reproduce
the single-stream result bit for bit; with ``warp=True`` only the initialisation of each
block's first frames differs.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from .pipeline import (
    ConsistencyConfig,
    DepthStage,
    DeviceDepthPanorama,
    DeviceDepthResult,
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
    depth: range           # depth results this rank computes (the blocks partition 0 .. n_results-1)
    centres: range         # frames it filters and fuses (indices into the depth results)
    raw_halo: tuple        # depth results of other ranks its consistency windows read
    filtered_halo: tuple   # filtered frames of other ranks its fusion FIFO reads


def plan_shards(n_results: int, world: int, window: int = 5, buffer: int = 4) -> list:
    """Contiguous, balanced blocks of fused frames; every depth result belongs to exactly one
    rank (the block of its centre, the sequence ends going to the first / last block with
    centres).  Ranks without a centre (sequence shorter than ``world`` windows) stay idle."""
    if world < 1:
        raise ValueError(f"world size must be >= 1, got {world}")
    half = window // 2
    first, last = half, n_results - (window - 1 - half)  # centres are [first, last)
    n = max(0, last - first)
    blocks = [(first + (n * r) // world, first + (n * (r + 1)) // world) for r in range(world)]
    busy = [r for r, (a, b) in enumerate(blocks) if a < b]
    plans = []
    for r, (a, b) in enumerate(blocks):
        if a >= b:
            plans.append(ShardPlan(r, world, range(a, a), range(a, a), (), ()))
            continue
        lo = 0 if r == busy[0] else a
        hi = n_results if r == busy[-1] else b
        raw = sorted({j for c in range(a, b) for j in range(c - half, c - half + window)} - set(range(lo, hi)))
        filt = sorted({j for c in range(a, b) for j in range(c + 1, c + buffer) if j < last} - set(range(a, b)))
        plans.append(ShardPlan(r, world, range(lo, hi), range(a, b), tuple(raw), tuple(filt)))
    return plans


def _owner(plans, index: int, what: str) -> int:
    for p in plans:
        if index in getattr(p, what):
            return p.rank
    raise ValueError(f"no rank owns {what} frame {index}")


class ShardRun:
    """One rank's share, in the three phases the exchanges separate.  ``groups[i]`` is the stereo
    group (or a callable returning a StereoGroup / PreparedGroup) of depth result i of the whole
    sequence; ``refs[i] = (keyframe id, pose)`` of its reference (taken from the groups when they are
    not callables)."""

    def __init__(self, groups, plan: ShardPlan, stage: DepthStage, consistency: ConsistencyConfig,
                 fusion: FusionConfig, refs=None, prime: int = 0):
        self.groups, self.plan, self.stage = groups, plan, stage
        self.consistency, self.fusion = consistency, fusion
        self.refs = refs if refs is not None else [(g.reference.id, g.reference.pose) for g in groups]
        self.prime = prime
        self.raw = {}        # depth result index -> DeviceDepthResult (own block + received halo)
        self.filtered = {}   # centre index -> DeviceDepthResult (own centres + received halo)
        self.computed = 0    # depth maps this rank ran PatchMatch for

    def _group(self, i):
        g = self.groups[i]
        return g() if callable(g) else g

    def compute_depth(self) -> None:
        if len(self.plan.depth) == 0:
            return
        for i in range(max(0, self.plan.depth.start - self.prime), self.plan.depth.start):
            self.stage.process_device(self._group(i))  # warms the warp chain up, result unused
            self.computed += 1
        for i in self.plan.depth:
            self.raw[i] = self.stage.process_device(self._group(i))
            self.computed += 1

    def frame_tensors(self, what: str, index: int):
        """(depth f32 (H,W), valid u8 (H,W)) of a frame this rank holds, as sent to a neighbour."""
        res = (self.raw if what == "raw" else self.filtered)[index]
        return res.pano.depth, res.pano.valid

    def empty_frame(self, device):
        h, w = self.stage.camera.shape
        return (torch.empty((h, w), dtype=torch.float32, device=device),
                torch.empty((h, w), dtype=torch.uint8, device=device))

    def accept_frame(self, what: str, index: int, depth: torch.Tensor, valid: torch.Tensor) -> None:
        """A halo frame received from its owner (no image: halo frames are only compared with)."""
        dev = self.stage.device
        kid, pose = self.refs[index]
        pano = DeviceDepthPanorama(self.stage.camera, depth.to(dev), valid.to(dev))
        (self.raw if what == "raw" else self.filtered)[index] = DeviceDepthResult(kid, pano, pose, None)

    def filter_centres(self) -> None:
        half = self.consistency.window // 2
        for c in self.plan.centres:
            win = [(self.raw[j].pano, self.raw[j].pose) for j in range(c - half, c - half + self.consistency.window)
                   if j != c]
            pano = consistency_filter_device(self.raw[c].pano, self.raw[c].pose, win, self.consistency)
            self.filtered[c] = DeviceDepthResult(self.raw[c].id, pano, self.raw[c].pose, self.raw[c].image)

    def fuse_centres(self) -> list:
        """DeviceFusedCloud batches of ``plan.centres`` in order."""
        out = []
        fb = FusionBuffer(self.stage.camera, self.fusion, device=self.stage.device)
        for c in self.plan.centres:
            # the FIFO state when frame c is the oldest: c plus the newer filtered frames that exist
            newer = [self.filtered[j] for j in range(c + 1, c + self.fusion.buffer) if j in self.filtered]
            fb._frames.clear()
            fb._frames.extend([self.filtered[c], *newer])
            out.append(fb._fuse_oldest())
        return out


def exchange_frames(run: ShardRun, plans, what: str, group=None, comm_device=None) -> int:
    """Point-to-point halo exchange: every rank sends the frames of ``what`` ("raw" / "filtered")
    it owns to the ranks whose plan lists them in ``<what>_halo`` and receives its own halo, as one
    batch of isend / irecv (NCCL groups them into one launch; ``ncclSend`` / ``ncclRecv`` between
    NVLink peers).  Both sides walk the same (receiver, frame, tensor) order, which is what pairs
    the operations.  ``comm_device``: where the process group communicates from (the stage's GPU
    for NCCL; "cpu" for gloo, the frames are then staged through host memory).  Returns the
    number of bytes this rank received."""
    import torch.distributed as dist

    me = run.plan.rank
    own = "depth" if what == "raw" else "centres"
    dev = torch.device(comm_device) if comm_device is not None else run.stage.device
    ops, incoming, keep = [], [], []
    for p in plans:  # receiver
        for f in getattr(p, what + "_halo"):
            src = _owner(plans, f, own)
            if p.rank == me:
                bufs = run.empty_frame(dev)
                incoming.append((f, bufs))
                ops += [dist.P2POp(dist.irecv, t, src, group) for t in bufs]
            elif src == me:
                tensors = [t.to(dev).contiguous() for t in run.frame_tensors(what, f)]
                keep.append(tensors)
                ops += [dist.P2POp(dist.isend, t, p.rank, group) for t in tensors]
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    got = 0
    for f, (depth, valid) in incoming:
        run.accept_frame(what, f, depth, valid)
        got += depth.numel() * depth.element_size() + valid.numel() * valid.element_size()
    return got


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
                     rank: int = 0, world: int = 1, dst: int = 0, group=None, refs=None, prime: int = 0,
                     comm_device=None, stats: dict | None = None):
    """Sharded equivalent of the reference's depth + consistency + fusion stages over a whole
    sequence (P:402-486 without ingest / view filter): this rank's block of depth maps, the two
    halo exchanges, its fused frames, and the cloud gather.  ``stage_factory()`` builds this
    rank's DepthStage.  Returns (FusedCloud on ``dst`` else None, ShardPlan); ``stats`` (optional
    dict) receives the depth maps computed and the halo bytes received."""
    plans = plan_shards(len(groups), world, consistency.window, fusion.buffer)
    stage = stage_factory()
    run = ShardRun(groups, plans[rank], stage, consistency, fusion, refs=refs, prime=prime)
    run.compute_depth()
    halo_bytes = 0
    if world > 1:
        halo_bytes += exchange_frames(run, plans, "raw", group=group, comm_device=comm_device)
    run.filter_centres()
    if world > 1:
        halo_bytes += exchange_frames(run, plans, "filtered", group=group, comm_device=comm_device)
    batches = run.fuse_centres()
    if stats is not None:
        stats.update(depth_maps_computed=run.computed, halo_bytes_received=halo_bytes,
                     fused_frames=len(batches), points=sum(len(b) for b in batches))
    dev = torch.device(comm_device) if comm_device is not None else stage.device
    return gather_cloud(batches, dst=dst, group=group, device=dev), plans[rank]


def simulate_shards(groups, world: int, stage_factory, consistency: ConsistencyConfig, fusion: FusionConfig,
                    refs=None, prime: int = 0):
    """All ``world`` shards run one after the other in this process, the exchanges done by handing
    tensors across (tests and single-GPU checks of the sharding arithmetic).  Returns
    (FusedCloud, [ShardRun])."""
    plans = plan_shards(len(groups), world, consistency.window, fusion.buffer)
    runs = [ShardRun(groups, p, stage_factory(), consistency, fusion, refs=refs, prime=prime) for p in plans]
    for run in runs:
        run.compute_depth()
    for what, own in (("raw", "depth"), ("filtered", "centres")):
        if what == "filtered":
            for run in runs:
                run.filter_centres()
        for run in runs:
            for f in getattr(run.plan, what + "_halo"):
                depth, valid = runs[_owner(plans, f, own)].frame_tensors(what, f)
                run.accept_frame(what, f, depth.clone(), valid.clone())
    batches = [b for run in runs for b in run.fuse_centres()]
    return gather_cloud(batches), runs
