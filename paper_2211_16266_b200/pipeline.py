"""Per-keyframe driver, geometric-consistency filter and fusion — host side.

Mirrors the hot-path half of the reference's ``densify360.pipeline`` (P = pipeline.py there):
``DepthStage``, ``consistency_filter``, ``FusionBuffer``
with their config / result types.  Depth maps stay in HBM between the stages
(``DeviceDepthResult``); the numpy-facing classes convert at the boundary only.
The ingest / threading orchestration of P:351-540 is out of scope.
"""
from __future__ import annotations

import time
from collections import deque
from dataclasses import dataclass

import ctypes as C
import numpy as np
import torch

from . import _lib
from .engine import (
    DepthPanorama,
    DeviceCamera,
    DeviceKeyframe,
    DeviceDepthPanorama,
    DevicePlaneMap,
    PatchMatchWorkspace,
    PatchSpec,
    PreparedGroup,
    _device,
    _ptr,
    _stream,
    _up,
    median_outlier_filter_device,
    pole_mask_device,
    random_init_device,
    run_patchmatch_device,
    warp_plane_map_device,
)
from .errors import ConfigError
from .geometry import EquirectCamera, RigidPose
from .keyframes import StereoGroup

POLE_LAT_LIMIT_DEG = 85.0


@dataclass(frozen=True)
class ConsistencyConfig:
    window: int = 5
    min_support: int = 2
    rel_depth_tol: float = 0.01

    def __post_init__(self) -> None:
        if self.window < 2:
            raise ConfigError(f"consistency.window must be >= 2, got {self.window}")
        if not (1 <= self.min_support < self.window):
            raise ConfigError("consistency.min_support must satisfy 1 <= min_support < window, "
                              f"got min_support={self.min_support}, window={self.window}")
        if self.rel_depth_tol <= 0:
            raise ConfigError(f"consistency.rel_depth_tol must be > 0, got {self.rel_depth_tol}")


@dataclass(frozen=True)
class FusionConfig:
    buffer: int = 4
    reproj_px: float = 1.0
    rel_depth_tol: float = 0.01

    def __post_init__(self) -> None:
        if self.buffer < 1:
            raise ConfigError(f"fusion.buffer must be >= 1, got {self.buffer}")
        if self.reproj_px <= 0:
            raise ConfigError(f"fusion.reproj_px must be > 0, got {self.reproj_px}")
        if self.rel_depth_tol <= 0:
            raise ConfigError(f"fusion.rel_depth_tol must be > 0, got {self.rel_depth_tol}")


@dataclass
class FusedCloud:
    """World points (N,3) f64, colours (N,3) u8, source keyframe ids (N,) i64."""

    points: np.ndarray
    colors: np.ndarray
    source_ids: np.ndarray

    @classmethod
    def empty(cls) -> "FusedCloud":
        return cls(np.zeros((0, 3), np.float64), np.zeros((0, 3), np.uint8), np.zeros((0,), np.int64))

    @classmethod
    def concat(cls, batches) -> "FusedCloud":
        batches = list(batches)
        if not batches:
            return cls.empty()
        return cls(np.concatenate([b.points for b in batches]), np.concatenate([b.colors for b in batches]),
                   np.concatenate([b.source_ids for b in batches]))

    def __len__(self) -> int:
        return self.points.shape[0]


@dataclass
class DepthResult:
    """Host view of one densified keyframe."""

    id: int
    pano: DepthPanorama
    pose: RigidPose
    image: np.ndarray
    seconds: float


class DeviceDepthResult:
    """Densified keyframe resident on the GPU: depth f32, valid u8, RGB u8."""

    def __init__(self, id: int, pano: DeviceDepthPanorama, pose: RigidPose, image: torch.Tensor, seconds: float = 0.0):
        self.id, self.pano, self.pose, self.image, self.seconds = id, pano, pose, image, seconds

    @classmethod
    def from_host(cls, r: DepthResult, device=None) -> "DeviceDepthResult":
        dev = _device(device)
        img = np.asarray(r.image)
        if img.ndim == 2:
            img = np.repeat(img[..., None], 3, axis=2)
        return cls(r.id, DeviceDepthPanorama.from_host(r.pano, dev), r.pose, _up(img, np.uint8, dev), r.seconds)

    def to_host(self) -> DepthResult:
        return DepthResult(self.id, self.pano.to_host(), self.pose, self.image.cpu().numpy(), self.seconds)


def project_points(camera: EquirectCamera, pose: RigidPose, points: np.ndarray):
    """World points -> continuous (u, v) and range in ``pose`` (host helper)."""
    local = (np.asarray(points, np.float64) - pose.translation) @ pose.rotation
    rng = np.linalg.norm(local, axis=1)
    lon = np.arctan2(local[:, 0], local[:, 2])
    lon = np.where(lon >= np.pi, lon - 2.0 * np.pi, lon)
    u = (lon + np.pi) * (camera.width / (2.0 * np.pi)) - 0.5
    v = np.arccos(np.clip(-local[:, 1] / np.maximum(rng, 1e-300), -1.0, 1.0)) * (camera.height / np.pi) - 0.5
    return u, v, rng


# ---------------------------------------------------------------------------------------
# DepthStage
# ---------------------------------------------------------------------------------------

class DepthStage:
    """Sequential densification worker with plane-map warping between jobs.

    Extra knobs over the reference: ``top_k`` / ``precision`` (kernel policy), ``init_rng``
    ("pcg64" reproduces the reference's random hypotheses, "philox" draws on the device)."""

    def __init__(self, camera: EquirectCamera, spec: PatchSpec, depth_range, iterations: int, seed: int,
                 warp: bool = True, workers: int | None = None, median_window: int = 5,
                 median_rel_threshold: float = 0.2, top_k: int | None = None, precision: str | None = None,
                 init_rng: str = "pcg64", device=None, count_evals: bool = False):
        self.camera, self.spec = camera, spec
        self.depth_range = tuple(depth_range)
        self.iterations, self.seed, self.warp, self.workers = iterations, seed, warp, workers
        self.median_window, self.median_rel_threshold = median_window, median_rel_threshold
        self.top_k, self.precision, self.init_rng = top_k, precision, init_rng
        self.device = _device(device)
        self._prev: tuple | None = None
        self.count_evals = count_evals
        self._ws = PatchMatchWorkspace(camera, self.device)

    @property
    def workspace(self) -> PatchMatchWorkspace:
        return self._ws

    def process_device(self, group: StereoGroup | PreparedGroup) -> DeviceDepthResult:
        prep = group if isinstance(group, PreparedGroup) else PreparedGroup(
            group, self.spec, top_k=self.top_k, precision=self.precision, device=self.device)
        ref = prep.group.reference
        with torch.cuda.device(self.device):
            if self.warp and self._prev is not None:
                prev_map, prev_pose = self._prev
                init = warp_plane_map_device(prev_map, prev_pose, ref.pose, self.camera, winner=self._ws.winner)
            else:
                init = DevicePlaneMap.empty(self.camera, self.depth_range, self.device)
            init = random_init_device(init, self.depth_range, self.seed + ref.id, self.init_rng)
            plane_map, pano = run_patchmatch_device(prep, init, self.iterations, self.seed + ref.id,
                                                    workspace=self._ws, count_evals=self.count_evals,
                                                    check_valid=False)
            self._prev = (plane_map, ref.pose)
            pano = median_outlier_filter_device(pano, self.median_window, self.median_rel_threshold)
            pole_mask_device(pano, POLE_LAT_LIMIT_DEG)
            image = prep.ref_image
            if image.ndim == 2:
                image = image[..., None].expand(-1, -1, 3).contiguous()
        return DeviceDepthResult(ref.id, pano, ref.pose, image)

    def process(self, group: StereoGroup) -> DepthResult:
        start = time.perf_counter()
        res = self.process_device(group)
        out = DepthResult(res.id, res.pano.to_host(), res.pose, group.reference.image, 0.0)
        out.seconds = time.perf_counter() - start
        return out


# ---------------------------------------------------------------------------------------
# consistency filter
# ---------------------------------------------------------------------------------------

def _frame_args(frames):
    """Host pointer tables + pose blocks for a list of (DeviceDepthPanorama, RigidPose)."""
    n = len(frames)
    if n > _lib.MAX_FRAMES:
        raise ConfigError(f"at most {_lib.MAX_FRAMES} frames per window/buffer are supported, got {n}")
    dptr = (C.c_void_p * max(n, 1))(*[p.depth.data_ptr() for p, _ in frames])
    vptr = (C.c_void_p * max(n, 1))(*[p.valid.data_ptr() for p, _ in frames])
    rot = np.ascontiguousarray(np.stack([q.rotation.reshape(9) for _, q in frames]) if n else np.zeros((1, 9)))
    tr = np.ascontiguousarray(np.stack([q.translation for _, q in frames]) if n else np.zeros((1, 3)))
    return dptr, vptr, rot, tr


def consistency_filter_device(target: DeviceDepthPanorama, target_pose: RigidPose, window,
                              config: ConsistencyConfig) -> DeviceDepthPanorama:
    lib = _lib.load()
    dev = target.depth.device
    cam = DeviceCamera.get(target.camera, dev)
    h, w = target.camera.shape
    out_valid = torch.empty_like(target.valid)
    dptr, vptr, rot, tr = _frame_args(window)
    prot = np.ascontiguousarray(target_pose.rotation.reshape(9))
    ptr_t = np.ascontiguousarray(target_pose.translation)
    with torch.cuda.device(dev):
        _lib.check(lib.d360_consistency_filter(_ptr(target.depth), _ptr(target.valid), prot.ctypes.data,
                                               ptr_t.ctypes.data, C.cast(dptr, C.c_void_p), C.cast(vptr, C.c_void_p),
                                               rot.ctypes.data, tr.ctypes.data, len(window), _ptr(cam.rays64),
                                               int(config.min_support), float(config.rel_depth_tol),
                                               _ptr(out_valid), h, w, _stream()), "consistency_filter")
    return DeviceDepthPanorama(target.camera, target.depth, out_valid)


def consistency_filter(target: DepthPanorama, target_pose: RigidPose, window, config: ConsistencyConfig) -> DepthPanorama:
    """Drop-in for pipeline.consistency_filter: window = [(DepthPanorama, RigidPose), ...]."""
    dev_win = [(DeviceDepthPanorama.from_host(p), q) for p, q in window]
    out = consistency_filter_device(DeviceDepthPanorama.from_host(target), target_pose, dev_win, config)
    return DepthPanorama(target.camera, target.depth.copy(), out.valid.cpu().numpy().astype(bool))


# ---------------------------------------------------------------------------------------
# fusion
# ---------------------------------------------------------------------------------------

class DeviceFusedCloud:
    """Fused batch on the device: points (N,3) f64, colours (N,3) u8, one source id."""

    def __init__(self, points: torch.Tensor, colors: torch.Tensor, source_id: int):
        self.points, self.colors, self.source_id = points, colors, source_id

    def __len__(self) -> int:
        return self.points.shape[0]

    def to_host(self) -> FusedCloud:
        n = len(self)
        return FusedCloud(self.points.cpu().numpy(), self.colors.cpu().numpy(), np.full(n, self.source_id, np.int64))


class FusionBuffer:
    """Fixed-depth FIFO of consistent frames with duplicate erasure."""

    def __init__(self, camera: EquirectCamera, config: FusionConfig, device=None):
        self.camera, self.config = camera, config
        self.device = _device(device)
        self._frames: deque = deque()
        self._scratch = None

    def _buffers(self):
        """Lazily allocated worst-case scratch, reused for every fused frame."""
        if self._scratch is None:
            h, w = self.camera.shape
            dev = self.device
            nblk = _lib.load().d360_fuse_blocks(h, w)
            self._scratch = (torch.empty((h, w), dtype=torch.uint8, device=dev),
                             torch.empty((nblk + 1,), dtype=torch.int32, device=dev),
                             torch.empty((h * w, 3), dtype=torch.float64, device=dev),
                             torch.empty((h * w, 3), dtype=torch.uint8, device=dev))
        return self._scratch

    def push_device(self, frame: DeviceDepthResult):
        self._frames.append(frame)
        if len(self._frames) == self.config.buffer:
            return self._fuse_oldest()
        return None

    def flush_device(self) -> list:
        out = []
        while self._frames:
            out.append(self._fuse_oldest())
        return out

    def push(self, frame: DepthResult):
        got = self.push_device(DeviceDepthResult.from_host(frame, self.device))
        return None if got is None else got.to_host()

    def flush(self) -> list:
        return [b.to_host() for b in self.flush_device()]

    def _fuse_oldest(self) -> DeviceFusedCloud:
        lib = _lib.load()
        oldest = self._frames.popleft()
        newer = [(f.pano, f.pose) for f in self._frames]
        h, w = self.camera.shape
        dev = self.device
        cam = DeviceCamera.get(self.camera, dev)
        dptr, vptr, rot, tr = _frame_args(newer)
        prot = np.ascontiguousarray(oldest.pose.rotation.reshape(9))
        ptr_t = np.ascontiguousarray(oldest.pose.translation)
        n_out = C.c_int64(0)
        with torch.cuda.device(dev):
            keep, counts, points, colors = self._buffers()
            _lib.check(lib.d360_fuse_oldest(_ptr(oldest.pano.depth), _ptr(oldest.pano.valid), prot.ctypes.data,
                                            ptr_t.ctypes.data, _ptr(oldest.image), C.cast(dptr, C.c_void_p),
                                            C.cast(vptr, C.c_void_p), rot.ctypes.data, tr.ctypes.data, len(newer),
                                            _ptr(cam.rays64), float(self.config.reproj_px),
                                            float(self.config.rel_depth_tol), _ptr(keep), _ptr(counts), _ptr(points),
                                            _ptr(colors), C.addressof(n_out), h, w, _stream()), "fuse_oldest")
            n = int(n_out.value)
            return DeviceFusedCloud(points[:n].clone(), colors[:n].clone(), oldest.id)


# ---------------------------------------------------------------------------------------
# streaming driver: keyframes in, filtered depth maps (and fused batches) out
# ---------------------------------------------------------------------------------------

def neighbor_order(n_views: int) -> list:
    """Window offsets of the neighbours of the middle keyframe, nearest first, older before
    newer: V=2 -> (-1, +1), the reference's triple; V=4 -> (-1, +1, -2, +2)."""
    if n_views < 1 or n_views % 2:
        raise ConfigError(f"the sliding keyframe window needs an even number of neighbours, got {n_views}")
    order = []
    for k in range(1, n_views // 2 + 1):
        order += [-k, k]
    return order


@dataclass
class StreamOutput:
    """One finished keyframe of the stream: consistency-filtered depth map on the host, plus
    the fused batch emitted at the same step (if fusion is enabled and its FIFO was full)."""

    id: int
    pano: DepthPanorama
    pose: RigidPose
    cloud: FusedCloud | None = None
    image: np.ndarray | None = None  # the reference keyframe's host image (as given to push)
    cloud_device: "DeviceFusedCloud | None" = None  # the same batch still in HBM (writers and metrics read it there)


class StreamingDensifier:
    """Stages of the reference's ``run_offline`` after the view filter, on one GPU:
    sliding (V+1)-keyframe window with the middle frame as reference (``KeyframeBuffer``,
    P:132-175, generalised from triples), ``DepthStage`` with warp carry-over, the consistency
    window and optionally the fusion FIFO (``_ConsistencyFusion``).

    Each keyframe is uploaded and converted once; depth maps stay in HBM between stages.  Per
    ``push`` the host traffic is one uint8 frame in and (once the windows are full) one filtered
    depth map + mask out.

    ``overlap=True`` takes both copies off the compute stream (the reference overlaps its stages with
    threads and bounded queues; here the stages are CUDA streams and events): the frame goes
    through a pinned staging buffer and an asynchronous copy on a copy stream that the compute stream
    waits for by event, and the finished depth map + mask are copied into pinned buffers on the copy
    stream after an event of the compute stream.  ``push`` then hands out the output of the PREVIOUS
    finished keyframe (its copy is long complete), so the host never waits for the GPU step it has just
    enqueued and the next step's kernels queue up behind the running ones; ``drain()`` returns the last
    output.  Same kernels in the same order on one compute stream: outputs are bit-identical to
    ``overlap=False``.  (With fusion enabled every fused batch still reads its point count back, which
    synchronises; the overlap then only covers the copies.)"""

    def __init__(self, camera: EquirectCamera, spec: PatchSpec, depth_range, iterations: int, seed: int,
                 n_neighbors: int = 2, warp: bool = True, consistency: ConsistencyConfig | None = None,
                 fusion: FusionConfig | None = None, median_window: int = 5, median_rel_threshold: float = 0.2,
                 top_k: int | None = None, precision: str | None = None, init_rng: str = "pcg64", device=None,
                 count_evals: bool = False, overlap: bool = False):
        self.camera = camera
        self.overlap = bool(overlap)
        self.order = neighbor_order(n_neighbors)
        self.consistency = consistency if consistency is not None else ConsistencyConfig()
        self.stage = DepthStage(camera, spec, depth_range, iterations, seed, warp=warp, median_window=median_window,
                                median_rel_threshold=median_rel_threshold, top_k=top_k, precision=precision,
                                init_rng=init_rng, device=device, count_evals=count_evals)
        self.device = self.stage.device
        self._frames: deque = deque(maxlen=n_neighbors + 1)  # (Keyframe, DeviceKeyframe)
        self._window: deque = deque()                        # DeviceDepthResult
        self._fusion = FusionBuffer(camera, fusion, self.device) if fusion is not None else None
        self._last_id = None
        self._group_buffers = {}  # planes of the group in flight, reused from push to push
        self.jobs = 0       # depth jobs run so far
        self._images = {}   # host image of every reference whose output is still pending (<= window entries)
        self._pending: deque = deque()  # overlap mode: (copy-done event, StreamOutput fields, pinned depth, pinned mask)
        if self.overlap:
            with torch.cuda.device(self.device):
                self._copy_stream = torch.cuda.Stream(self.device)
            self._stage_in = []   # two pinned uint8 frames + the event of the last copy out of each
            self._stage_out = []  # three pinned (depth, mask) pairs, rotated
            self._n_in = self._n_out = 0

    def _upload(self, image: np.ndarray) -> torch.Tensor:
        """Host frame -> device through a pinned staging buffer and the copy stream."""
        image = np.ascontiguousarray(image, dtype=np.uint8)
        if len(self._stage_in) < 2:
            self._stage_in.append([torch.empty(image.shape, dtype=torch.uint8).pin_memory(), None])
        slot = self._stage_in[self._n_in % 2]
        self._n_in += 1
        if tuple(slot[0].shape) != image.shape:
            slot[0], slot[1] = torch.empty(image.shape, dtype=torch.uint8).pin_memory(), None
        if slot[1] is not None:
            slot[1].synchronize()  # the copy that last read this buffer (two pushes ago)
        slot[0].numpy()[...] = image
        compute = torch.cuda.current_stream(self.device)
        with torch.cuda.stream(self._copy_stream):
            dev_img = slot[0].to(self.device, non_blocking=True)
            slot[1] = torch.cuda.Event()
            slot[1].record(self._copy_stream)
        compute.wait_event(slot[1])
        dev_img.record_stream(compute)
        return dev_img

    def _download_async(self, pano: DeviceDepthPanorama):
        """Enqueue depth + mask -> pinned host buffers on the copy stream; returns (event, depth, mask)."""
        if len(self._stage_out) < 3:
            h, w = self.camera.shape
            self._stage_out.append((torch.empty((h, w), dtype=torch.float32).pin_memory(),
                                    torch.empty((h, w), dtype=torch.uint8).pin_memory()))
        hd, hv = self._stage_out[self._n_out % 3]
        self._n_out += 1
        compute = torch.cuda.current_stream(self.device)
        ready = torch.cuda.Event()
        ready.record(compute)
        with torch.cuda.stream(self._copy_stream):
            self._copy_stream.wait_event(ready)
            hd.copy_(pano.depth, non_blocking=True)
            hv.copy_(pano.valid, non_blocking=True)
            done = torch.cuda.Event()
            done.record(self._copy_stream)
        pano.depth.record_stream(self._copy_stream)
        pano.valid.record_stream(self._copy_stream)
        return done, hd, hv

    def _collect(self, keep: int) -> list:
        """Outputs whose copies are complete, oldest first, leaving the `keep` newest in flight."""
        outs = []
        while len(self._pending) > keep:
            done, out, hd, hv = self._pending.popleft()
            done.synchronize()
            out.pano = DepthPanorama(self.camera, hd.numpy().copy(), hv.numpy().astype(bool))
            outs.append(out)
        return outs

    def drain(self) -> list:
        """Overlap mode: the outputs still in flight (at most one); empty otherwise."""
        return self._collect(0)

    def push(self, keyframe: Keyframe) -> list:
        """Feed the next keyframe (ids strictly increasing); returns the outputs that
        became final with it (0 or 1)."""
        from .errors import OrderingError

        if self._last_id is not None and keyframe.id <= self._last_id:
            raise OrderingError(f"keyframe id {keyframe.id} arrived after id {self._last_id}; "
                                "ids must be strictly increasing")
        self._last_id = keyframe.id
        image = keyframe.image
        if self.overlap and not isinstance(image, torch.Tensor):
            with torch.cuda.device(self.device):
                image = self._upload(np.asarray(image))
        self._frames.append((keyframe, DeviceKeyframe(image, self.camera, self.device)))
        if len(self._frames) < self._frames.maxlen:
            return []
        mid = len(self._frames) // 2
        picks = [mid] + [mid + o for o in self.order]
        group = StereoGroup(reference=self._frames[mid][0], neighbors=tuple(self._frames[i][0] for i in picks[1:]),
                            camera=self.camera)
        prep = PreparedGroup(group, self.stage.spec, top_k=self.stage.top_k, precision=self.stage.precision,
                             device=self.device, device_keyframes=[self._frames[i][1] for i in picks],
                             buffers=self._group_buffers)
        self._window.append(self.stage.process_device(prep))
        self.jobs += 1
        self._images[group.reference.id] = group.reference.image
        if len(self._window) < self.consistency.window:
            return []
        frames = list(self._window)
        c = len(frames) // 2
        target = frames[c]
        others = [(f.pano, f.pose) for i, f in enumerate(frames) if i != c]
        pano = consistency_filter_device(target.pano, target.pose, others, self.consistency)
        self._window.popleft()
        for old in [k for k in self._images if k < target.id]:
            del self._images[old]  # references the consistency window left behind without an output
        if not self.overlap:
            out = StreamOutput(target.id, pano.to_host(), target.pose, image=self._images.pop(target.id, None))
            if self._fusion is not None:
                batch = self._fusion.push_device(DeviceDepthResult(target.id, pano, target.pose, target.image))
                out.cloud = None if batch is None else batch.to_host()
                out.cloud_device = batch
            return [out]
        with torch.cuda.device(self.device):
            done, hd, hv = self._download_async(pano)
        out = StreamOutput(target.id, None, target.pose, image=self._images.pop(target.id, None))
        if self._fusion is not None:
            batch = self._fusion.push_device(DeviceDepthResult(target.id, pano, target.pose, target.image))
            out.cloud = None if batch is None else batch.to_host()
            out.cloud_device = batch
        self._pending.append((done, out, hd, hv))
        return self._collect(1)

    def finish(self) -> list:
        """Flush the fusion FIFO; frames still inside the consistency window are
        dropped, as in the reference."""
        return [b.to_host() for b in self.finish_device()]

    def finish_device(self) -> list:
        """``finish`` with the batches left in HBM (DeviceFusedCloud)."""
        if self._fusion is None:
            return []
        return self._fusion.flush_device()
