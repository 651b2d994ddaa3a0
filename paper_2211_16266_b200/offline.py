"""Caller of the hot path: ingest -> view filter -> sliding window -> depth -> consistency ->
fusion -> report, i.e. the reference's ``run_offline`` (pipeline.py:402-486) without its dataset
loader and config system.

The compute stages are the device-resident ``StreamingDensifier`` (one keyframe upload per
step, depth maps stay in HBM between stages, completeness on the GPU); the host side keeps the
reference's names, ordering rules, view-filter decisions and report schema:

* ``ViewFilterConfig`` / ``ViewFilterDecision`` / ``view_filter_accept`` — viewfilter.py:19-105,
  O(landmarks) scalar host logic, restated here because ``KeyframeBuffer`` needs its decisions;
* ``KeyframeBuffer`` — pipeline.py:132-175, generalised from triples to (V + 1)-wide windows with
  the middle frame as reference (V = 2 is the reference's triple);
* ``run_offline`` — takes any iterable of ``Keyframe`` (the reference takes a ``Dataset``) and the
  stage configs as keyword arguments (the reference takes an ``EngineConfig``).  ``threaded=True``
  moves ingest + view filter to a producer thread over a bounded queue; GPU work is asynchronous
  on its stream either way, and the results are identical (as the reference guarantees for its
  own threaded mode, tests/test_pipeline.py:344-353).
"""
from __future__ import annotations

import math
import queue
import threading
import time
from collections import deque
from dataclasses import dataclass

import numpy as np
import torch

from .engine import PatchSpec
from .errors import ConfigError, OrderingError
from .geometry import EquirectCamera
from .ingest import resample_keyframe
from .keyframes import Keyframe, StereoGroup
from .pipeline import (ConsistencyConfig, DepthResult, FusedCloud, FusionConfig, StreamingDensifier, neighbor_order)


@dataclass(frozen=True)
class ViewFilterConfig:
    """viewfilter.py:19-35."""

    theta_min: float = 6.0
    theta_max: float = 60.0
    accept_fraction: float = 0.20

    def __post_init__(self) -> None:
        if not (0.0 < self.theta_min < self.theta_max < 180.0):
            raise ConfigError("viewfilter requires 0 < theta_min < theta_max < 180, got "
                              f"theta_min={self.theta_min}, theta_max={self.theta_max}")
        if not (0.0 < self.accept_fraction <= 1.0):
            raise ConfigError(f"viewfilter.accept_fraction must be in (0, 1], got {self.accept_fraction}")


@dataclass(frozen=True)
class ViewFilterDecision:
    """viewfilter.py:38-46."""

    accepted: bool
    fraction: float
    common_points: int
    reason: str

    def __bool__(self) -> bool:
        return self.accepted


def triangulation_angle(point, center_a, center_b) -> float:
    """Angle at ``point`` between the two camera centres in degrees; 0 when the point sits on a
    centre (viewfilter.py:48-62)."""
    u = np.asarray(center_a, np.float64) - point
    v = np.asarray(center_b, np.float64) - point
    nu, nv = float(np.linalg.norm(u)), float(np.linalg.norm(v))
    if nu < 1e-12 or nv < 1e-12:
        return 0.0
    c = float(u @ v) / (nu * nv)
    return math.degrees(math.acos(min(1.0, max(-1.0, c))))


def common_landmarks(a: Keyframe, b: Keyframe) -> np.ndarray:
    """Landmarks of ``a`` that ``b`` observes too, matched by exact coordinates, in ``a``'s order
    (viewfilter.py:65-71)."""
    seen = {tuple(p) for p in b.sparse_points}
    rows = [p for p in a.sparse_points if tuple(p) in seen]
    return np.asarray(rows) if rows else np.zeros((0, 3))


def view_filter_accept(candidate: Keyframe, latest: Keyframe, config: ViewFilterConfig) -> ViewFilterDecision:
    """viewfilter.py:73-105: accept iff the fraction of common landmarks whose triangulation angle
    lies in the closed interval [theta_min, theta_max] reaches ``accept_fraction``."""
    common = common_landmarks(candidate, latest)
    n = common.shape[0]
    if n == 0:
        return ViewFilterDecision(False, 0.0, 0, "no-overlap")
    ta, tb = candidate.pose.translation, latest.pose.translation
    inside = sum(1 for p in common if config.theta_min <= triangulation_angle(p, ta, tb) <= config.theta_max)
    fraction = inside / n
    if fraction >= config.accept_fraction:
        return ViewFilterDecision(True, fraction, n, "ok")
    return ViewFilterDecision(False, fraction, n, "insufficient-parallax")


class KeyframeBuffer:
    """Ingestion state machine (pipeline.py:132-175): ordering check, view filter, stereo groups.
    ``n_neighbors`` = V: a group is emitted for the middle frame of every full (V + 1)-window of
    accepted keyframes, neighbours nearest first."""

    def __init__(self, camera: EquirectCamera, config: ViewFilterConfig, n_neighbors: int = 2):
        self.camera = camera
        self.config = config
        self._order = neighbor_order(n_neighbors)
        self._window: deque = deque(maxlen=n_neighbors + 1)
        self._latest = None
        self._last_id = None
        self.submitted = 0
        self.accepted = 0

    def submit(self, keyframe: Keyframe):
        """-> (ViewFilterDecision, StereoGroup | None)."""
        if self._last_id is not None and keyframe.id <= self._last_id:
            raise OrderingError(f"keyframe id {keyframe.id} arrived after id {self._last_id}; "
                                "ids must be strictly increasing")
        self._last_id = keyframe.id
        self.submitted += 1
        if self._latest is None:
            decision = ViewFilterDecision(True, 1.0, 0, "first-keyframe")
        else:
            decision = view_filter_accept(keyframe, self._latest, self.config)
        if not decision.accepted:
            return decision, None
        self.accepted += 1
        self._latest = keyframe
        self._window.append(keyframe)
        if len(self._window) < self._window.maxlen:
            return decision, None
        frames = list(self._window)
        mid = len(frames) // 2
        group = StereoGroup(reference=frames[mid], neighbors=tuple(frames[mid + o] for o in self._order),
                            camera=self.camera)
        return decision, group


@dataclass
class PipelineResult:
    """pipeline.py:351-356."""

    cloud: FusedCloud
    depths: dict
    report: dict
    camera: EquirectCamera
    device_batches: list = None  # the fused batches as they left the fusion stage, still in HBM (DeviceFusedCloud):
    #                              outputs.write_ply and metrics.completeness take these without a PCIe round trip


def run_offline(keyframes, camera: EquirectCamera, *, viewfilter: ViewFilterConfig | None = None,
                spec: PatchSpec | None = None, depth_range=(0.5, 16.0), iterations: int = 6, seed: int = 0,
                warp: bool = True, median_window: int = 5, median_rel_threshold: float = 0.2,
                consistency: ConsistencyConfig | None = None, fusion: FusionConfig | None = None,
                n_neighbors: int = 2, top_k: int | None = None, precision: str | None = None, init_rng: str = "pcg64",
                threaded: bool = False, queue_size: int = 2, device=None) -> PipelineResult:
    """Process a keyframe sequence through the whole pipeline; deterministic per seed
    (pipeline.py:402-486).  Report keys and meanings are the reference's."""
    from .metrics import completeness

    viewfilter = viewfilter if viewfilter is not None else ViewFilterConfig()
    fusion = fusion if fusion is not None else FusionConfig()
    buffer = KeyframeBuffer(camera, viewfilter, n_neighbors)
    stream = StreamingDensifier(camera, spec if spec is not None else PatchSpec(), depth_range, iterations, seed,
                                n_neighbors=n_neighbors, warp=warp, consistency=consistency, fusion=fusion,
                                median_window=median_window, median_rel_threshold=median_rel_threshold, top_k=top_k,
                                precision=precision, init_rng=init_rng, device=device)
    clock = {"ingest": 0.0, "depth": 0.0, "fuse": 0.0}
    poses, depth_seconds, batches, device_batches, filtered = [], [], [], [], {}
    queue_peaks = {"jobs": 0, "depths": 0}

    def accepted_keyframes():
        for keyframe in keyframes:
            t0 = time.perf_counter()
            if keyframe.image.shape[:2] != camera.shape:  # brought to the working resolution (LANCZOS)
                keyframe = resample_keyframe(keyframe, camera)
            poses.append(keyframe.pose)
            decision, _ = buffer.submit(keyframe)
            clock["ingest"] += time.perf_counter() - t0
            if decision.accepted:
                yield keyframe

    def consume(keyframe):
        t0 = time.perf_counter()
        jobs_before = stream.jobs
        for out in stream.push(keyframe):
            filtered[out.id] = DepthResult(out.id, out.pano, out.pose, out.image, 0.0)
            if out.cloud is not None:
                batches.append(out.cloud)
                device_batches.append(out.cloud_device)
        dt = time.perf_counter() - t0
        if stream.jobs > jobs_before:  # one depth job ran (asynchronously; the time includes the D2H of its output)
            depth_seconds.append(dt)
            clock["depth"] += dt

    if threaded:
        q: queue.Queue = queue.Queue(maxsize=max(1, queue_size))
        errors = []

        def producer():
            try:
                for kf in accepted_keyframes():
                    q.put(kf)
                    queue_peaks["jobs"] = max(queue_peaks["jobs"], q.qsize())
            except BaseException as exc:  # re-raised in the caller's thread, as P:507-511
                errors.append(exc)
            finally:
                q.put(None)

        t = threading.Thread(target=producer, name="densify-ingest")
        t.start()
        try:
            while True:
                kf = q.get()
                if kf is None:
                    break
                consume(kf)
        finally:
            while t.is_alive():
                try:
                    q.get(timeout=0.05)
                except queue.Empty:
                    pass
            t.join()
        if errors:
            raise errors[0]
    else:
        for kf in accepted_keyframes():
            consume(kf)

    t0 = time.perf_counter()
    tail = stream.finish_device()
    device_batches.extend(tail)
    batches.extend(b.to_host() for b in tail)
    clock["fuse"] += time.perf_counter() - t0
    cloud = FusedCloud.concat(batches)
    nonempty = [b.points for b in device_batches if len(b)]
    all_points = torch.cat(nonempty) if nonempty else cloud.points  # the cloud is still in HBM: no re-upload
    comp = completeness(all_points, poses, device=stream.device) if poses else {
        "per_keyframe": [], "mean": 0.0, "point_count": 0, "resolution": [720, 360]}
    report = {
        "keyframes_total": buffer.submitted,
        "keyframes_accepted": buffer.accepted,
        "view_filter_acceptance": buffer.accepted / buffer.submitted if buffer.submitted else 0.0,
        "depth_jobs": len(depth_seconds),
        "fused_points": len(cloud),
        "stage_wall_s": dict(clock),
        "per_keyframe_depth_s": depth_seconds,
        "mean_depth_s": float(np.mean(depth_seconds)) if depth_seconds else 0.0,
        "queue_peak": queue_peaks,
        "completeness": comp,
        "resolution": [camera.width, camera.height],
    }
    return PipelineResult(cloud=cloud, depths=filtered, report=report, camera=camera, device_batches=device_batches)
