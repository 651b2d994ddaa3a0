"""Evaluation metrics (reference metrics.py:1-87): raster completeness, depth accuracy, voxel
coverage, computed on the device.

``completeness`` is the tail of the reference's ``run_offline`` (pipeline.py:459-465): O(points x
poses) numpy work that takes over once densification is fast.  Here the cloud is uploaded once
and every pose costs one splat kernel and one count over a 720 x 360 raster.
No CPU fallback: BackendError without libd360.so / a CUDA device.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .engine import DepthPanorama, DeviceDepthPanorama, _device, _ptr, _stream, _up
from .geometry import EquirectCamera

COMPLETENESS_CAMERA = EquirectCamera(720, 360)


def _points_device(points, device):
    if isinstance(points, torch.Tensor):
        return points.to(torch.float64).reshape(-1, 3).contiguous()
    return _up(np.asarray(points, np.float64).reshape(-1, 3), np.float64, device)


def completeness(points, poses, camera: EquirectCamera = COMPLETENESS_CAMERA, device=None) -> dict:
    """Fraction of raster pixels covered by the projected cloud, per pose (metrics.py:13-49).
    ``points``: (N,3) host array or device tensor."""
    lib = _lib.load()
    dev = points.device if isinstance(points, torch.Tensor) else _device(device)
    pts = _points_device(points, dev)
    n = int(pts.shape[0])
    h, w = camera.shape
    series = []
    with torch.cuda.device(dev):
        raster = torch.empty((h, w), dtype=torch.uint8, device=dev)
        counts = torch.zeros((max(len(poses), 1),), dtype=torch.int64, device=dev)
        for k, pose in enumerate(poses):
            if n == 0:
                continue
            raster.zero_()
            rot = np.ascontiguousarray(pose.rotation, np.float64)
            trans = np.ascontiguousarray(pose.translation, np.float64)
            _lib.check(lib.d360_completeness_splat(_ptr(pts), n, rot.ctypes.data, trans.ctypes.data, _ptr(raster), h, w,
                                                   _stream()), "completeness_splat")
            _lib.check(lib.d360_count_nonzero(_ptr(raster), h * w, _ptr(counts[k:]), _stream()), "count_nonzero")
        hits = counts.tolist()
    for k in range(len(poses)):
        series.append(float(hits[k] / (h * w)) if n else 0.0)
    return {"per_keyframe": series, "mean": float(np.mean(series)) if series else 0.0, "point_count": n,
            "resolution": [camera.width, camera.height]}


def accuracy(prediction, ground_truth, device=None) -> dict:
    """Per-pixel depth error statistics over jointly valid pixels (metrics.py:52-78).
    Panoramas may be host DepthPanorama or DeviceDepthPanorama."""
    if prediction.camera != ground_truth.camera:
        raise ValueError(f"resolution mismatch: prediction {prediction.camera.shape} "
                         f"vs ground truth {ground_truth.camera.shape}")
    lib = _lib.load()
    dev = _device(device)
    for p in (prediction, ground_truth):
        if isinstance(p, DeviceDepthPanorama):
            dev = p.depth.device
    pr = prediction if isinstance(prediction, DeviceDepthPanorama) else DeviceDepthPanorama.from_host(prediction, dev)
    gt = ground_truth if isinstance(ground_truth, DeviceDepthPanorama) else DeviceDepthPanorama.from_host(ground_truth, dev)
    h, w = pr.camera.shape
    with torch.cuda.device(dev):
        scratch = torch.empty((lib.d360_accuracy_scratch_doubles(),), dtype=torch.float64, device=dev)
        out = torch.empty((4,), dtype=torch.float64, device=dev)
        _lib.check(lib.d360_depth_accuracy(_ptr(pr.depth.contiguous()), _ptr(pr.valid.contiguous()),
                                           _ptr(gt.depth.contiguous()), _ptr(gt.valid.contiguous()), h * w,
                                           _ptr(scratch), _ptr(out), _stream()), "depth_accuracy")
        s_rel, s_sq, n_in, n = out.tolist()
    n = int(n)
    if n == 0:
        return {"defined": False, "mean_abs_rel": float("nan"), "rmse_m": float("nan"), "inlier_2pc": float("nan"),
                "valid_pixels": 0}
    return {"defined": True, "mean_abs_rel": float(s_rel / n), "rmse_m": float(np.sqrt(s_sq / n)),
            "inlier_2pc": float(n_in / n), "valid_pixels": n}


def voxel_occupancy(points, voxel: float = 0.1, device=None) -> int:
    """Number of occupied voxels at the given edge length (metrics.py:81-87).  The cell keys are
    computed by d360_voxel_keys; counting the distinct keys uses torch.unique (a library sort)."""
    lib = _lib.load()
    dev = points.device if isinstance(points, torch.Tensor) else _device(device)
    pts = _points_device(points, dev)
    n = int(pts.shape[0])
    if n == 0:
        return 0
    with torch.cuda.device(dev):
        keys = torch.empty((n,), dtype=torch.int64, device=dev)
        overflow = torch.zeros((1,), dtype=torch.int32, device=dev)
        _lib.check(lib.d360_voxel_keys(_ptr(pts), n, float(voxel), _ptr(keys), _ptr(overflow), _stream()), "voxel_keys")
        if int(overflow.item()):
            raise ValueError("voxel_occupancy: cell index outside +-2^20 (points too far for this voxel size)")
        return int(torch.unique(keys).numel())
