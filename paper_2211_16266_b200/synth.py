"""Synthetic scenes rendered on the GPU (benchmark and test input generator).

Re-implements the analytic scenes of the reference's ``densify360.synth`` (SY = synth.py
there): closed axis-aligned box room, long-box corridor and sphere shell viewed from inside
(SY:66-84), textured with 4-octave splitmix-hash value noise (SY:101-151) or the deliberately
ambiguous checker (SY:88-92).  The kernel follows the float64 numpy code operation by operation
(the two BLAS statements as the reference's numpy rounds them), so the images are bit-identical to
``render_scene`` (SY:154-169) for any pose; the reference's CPU render takes ~11 s per 1920x960 frame.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .engine import DepthPanorama, DeviceCamera, _device, _ptr, _stream
from .errors import ConfigError
from .geometry import EquirectCamera, GeometryError, RigidPose
from .keyframes import Keyframe, StereoGroup

SCENE_KINDS = ("box", "corridor", "sphere")


@dataclass(frozen=True)
class SyntheticScene:
    """Closed analytic scene (SY:27-64): full box extents in metres for box / corridor, ``(diameter,) * 3``
    for the sphere shell; value-noise texture parameters, or the checker of ``noise_scale``-sized cells."""

    kind: str = "box"
    size: tuple = (4.0, 3.0, 5.0)
    texture_seed: int = 7
    noise_scale: float = 0.6
    octaves: int = 4
    checker: bool = False
    trajectory: tuple = ()

    def __post_init__(self) -> None:
        if self.kind not in SCENE_KINDS:
            raise ConfigError(f"scene kind must be one of {SCENE_KINDS}, got {self.kind!r}")
        if min(self.size) <= 0:
            raise ConfigError(f"scene size must be positive, got {self.size}")
        if self.octaves < 1:
            raise ConfigError(f"texture octaves must be >= 1, got {self.octaves}")
        for pose in self.trajectory:
            if not self.contains(pose.translation):
                raise GeometryError(f"trajectory pose at {pose.translation} lies outside the scene")

    @property
    def radius(self) -> float:
        return self.size[0] / 2.0

    def contains(self, point, margin: float = 0.05) -> bool:
        pt = np.asarray(point, dtype=np.float64)
        if self.kind == "sphere":
            return float(np.linalg.norm(pt)) < self.radius - margin
        half = np.asarray(self.size, dtype=np.float64) / 2.0
        return bool(np.all(np.abs(pt) < half - margin))

    def cast(self, origin, directions) -> np.ndarray:
        """Distance from ``origin`` (inside the scene) to the surface along unit ``directions`` (..., 3), on the host
        (SY:66-84): used for the few hundred sparse landmarks of ``make_sequence``; images go through the GPU kernel.
        Same float64 operations per element as the reference, so the landmarks come out bit for bit."""
        o = np.asarray(origin, dtype=np.float64)
        d = np.asarray(directions, dtype=np.float64)
        if self.kind == "sphere":
            # |o + t d| = radius, positive root; d @ o stays a matrix-vector product (its BLAS rounding is part of
            # what the reference computes)
            along = d @ o
            return np.sqrt(np.maximum(along * along - (o @ o - self.radius**2), 0.0)) - along
        # box / corridor: the ray leaves through the nearest of the three far slab faces
        half = np.asarray(self.size) / 2.0
        face = np.where(d > 0, half, -half)
        with np.errstate(divide="ignore", invalid="ignore"):
            t = np.where(d != 0.0, (face - o) / np.where(d == 0, 1, d), np.inf)
        return np.where(t > 0, t, np.inf).min(axis=-1)


def straight_line_trajectory(scene: SyntheticScene, keyframes: int, span_fraction: float = 0.7) -> tuple:
    """In-and-out flight along the scene's long axis with identity orientation (SY:172-200): a triangle
    wave whose fold sits half a step past the apex, so the return leg interleaves the outbound grid (all poses
    distinct, consecutive baselines never vanish)."""
    if keyframes < 1:
        raise ConfigError(f"keyframes must be >= 1, got {keyframes}")
    if scene.kind == "sphere":
        long_axis, length = 2, scene.radius
    else:
        long_axis = int(np.argmax(np.asarray(scene.size)))
        length = np.asarray(scene.size)[long_axis]
    reach = length * span_fraction / 2.0
    step = 4.0 / keyframes
    ramp = step * np.arange(keyframes) - 1.0            # -1 ... 3
    folded = np.where(ramp > 1.0 + step / 4.0, 2.0 + step / 2.0 - ramp, ramp)
    poses = []
    for fraction in folded:
        centre = np.zeros(3)
        centre[long_axis] = 1.0
        poses.append(RigidPose(np.eye(3), centre * (fraction * reach)))
    return tuple(poses)


def default_scene(kind: str, keyframes: int = 0, checker: bool = False) -> SyntheticScene:
    """Presets of SY:203-224."""
    sizes = {"box": (4.0, 3.0, 5.0), "corridor": (4.0, 3.0, 20.0), "sphere": (4.0, 4.0, 4.0)}
    if kind not in sizes:
        raise ConfigError(f"scene kind must be one of {SCENE_KINDS}, got {kind!r}")
    scene = SyntheticScene(kind, sizes[kind], checker=checker)
    if keyframes:
        scene = SyntheticScene(kind, sizes[kind], checker=checker, trajectory=straight_line_trajectory(scene, keyframes))
    return scene


def render_scene_device(scene: SyntheticScene, camera: EquirectCamera, pose: RigidPose, device=None):
    """(image (H,W,3) u8, depth (H,W) f32) as CUDA tensors."""
    if not scene.contains(pose.translation):
        raise GeometryError(f"camera at {pose.translation} lies outside the scene")
    dev = _device(device)
    lib = _lib.load()
    cam = DeviceCamera.get(camera, dev)
    h, w = camera.shape
    size = np.ascontiguousarray(scene.size, dtype=np.float64)
    rot = np.ascontiguousarray(pose.rotation.reshape(9), dtype=np.float64)
    tr = np.ascontiguousarray(pose.translation, dtype=np.float64)
    o = np.asarray(pose.translation, dtype=np.float64)
    oo_minus_r2 = float(o @ o - scene.radius**2)  # SY:73, evaluated by numpy as the reference does
    with torch.cuda.device(dev):
        image = torch.empty((h, w, 3), dtype=torch.uint8, device=dev)
        depth = torch.empty((h, w), dtype=torch.float32, device=dev)
        _lib.check(lib.d360_render_scene(1 if scene.kind == "sphere" else 0, int(bool(scene.checker)), size.ctypes.data,
                                         oo_minus_r2, int(scene.texture_seed), float(scene.noise_scale),
                                         int(scene.octaves), rot.ctypes.data, tr.ctypes.data, _ptr(cam.rays64),
                                         _ptr(image), _ptr(depth), h, w, _stream()), "render_scene")
    return image, depth


def render_scene(scene: SyntheticScene, camera: EquirectCamera, pose: RigidPose):
    """Drop-in for synth.render_scene: (uint8 image, DepthPanorama) on the host."""
    image, depth = render_scene_device(scene, camera, pose)
    return image.cpu().numpy(), DepthPanorama(camera, depth.cpu().numpy(), np.ones(camera.shape, bool))


def neighbor_offsets(n_views: int, step: float = 0.15):
    """Signed baselines of SURVEY.md §8d: ±step, ±2 step, ... (V even) along one axis."""
    offs = []
    for k in range(1, n_views // 2 + 1):
        offs += [-k * step, k * step]
    if n_views % 2:
        offs.append((n_views // 2 + 1) * step)
    return offs


def make_group(scene: SyntheticScene, camera: EquirectCamera, center=(0.0, 0.0, 0.0), n_views: int = 2,
               step: float = 0.15, axis: int = 2, ref_id: int = 0, device=None):
    """Reference keyframe at ``center`` plus ``n_views`` neighbours displaced along ``axis``.

    Returns (StereoGroup, ground-truth depth (H,W) f32 numpy).  V=2 reproduces the layout of
    the reference's test fixture (tests/scenes.py:11-29): neighbours at -step and +step."""
    frames = []
    gt = None
    for k, off in enumerate([0.0] + neighbor_offsets(n_views, step)):
        t = np.array(center, dtype=np.float64)
        t[axis] += off
        pose = RigidPose(np.eye(3), t)
        image, pano = render_scene(scene, camera, pose)
        frames.append(Keyframe(id=ref_id + k, image=image, pose=pose))
        if k == 0:
            gt = pano.depth
    return StereoGroup(reference=frames[0], neighbors=tuple(frames[1:]), camera=camera), gt


def scene_to_dict(scene: SyntheticScene) -> dict:
    """The manifest's optional scene descriptor (SY:227-235)."""
    return {"kind": scene.kind, "size": list(scene.size), "texture_seed": scene.texture_seed,
            "noise_scale": scene.noise_scale, "octaves": scene.octaves, "checker": scene.checker}


def make_sequence(scene: SyntheticScene, keyframes: int, sparse_density: int, camera: EquirectCamera = EquirectCamera(512, 256),
                  seed: int = 11, device=None) -> list:
    """The keyframes ``make_dataset`` (SY:252-330) writes, kept in memory: trajectory poses (the scene's, or
    ``straight_line_trajectory``), GPU-rendered images, and the sliding window over one global landmark pool
    (surface hits of random directions, cast from a camera near each landmark's window) that the view filter
    keys on.  Same NumPy draws in the same order as the reference, so ids, poses and landmarks are identical."""
    if keyframes < 3:
        raise ConfigError(f"make_dataset needs keyframes >= 3, got {keyframes}")
    if sparse_density < 1:
        raise ConfigError(f"sparse_density must be >= 1, got {sparse_density}")
    poses = scene.trajectory
    if len(poses) != keyframes:
        poses = straight_line_trajectory(scene, keyframes)
    rng = np.random.default_rng(seed)
    stride = max(1, sparse_density // 3)
    pool_size = sparse_density + stride * (keyframes - 1)
    dirs = rng.standard_normal((pool_size, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    src = np.clip(np.arange(pool_size) // stride - 1, 0, keyframes - 1)
    pool = np.empty((pool_size, 3))
    for k in np.unique(src):
        sel = src == k
        origin = poses[k].translation
        pool[sel] = origin + dirs[sel] * scene.cast(origin, dirs[sel])[:, None]
    out = []
    for k, pose in enumerate(poses):
        image, _ = render_scene_device(scene, camera, pose, device)
        out.append(Keyframe(id=k, image=image.cpu().numpy(), pose=pose,
                            sparse_points=pool[k * stride: k * stride + sparse_density]))
    return out


def make_dataset(scene: SyntheticScene, keyframes: int, sparse_density: int, out_dir, camera: EquirectCamera = EquirectCamera(512, 256),
                 seed: int = 11):
    """Drop-in for synth.make_dataset (SY:252-330): the sequence of ``make_sequence`` written in the pipeline's
    dataset directory format (``kfNNNN.png`` + ``dataset.json`` with the field names of dataset.py:40)."""
    import json
    from pathlib import Path

    from PIL import Image

    from .errors import DatasetError

    frames = make_sequence(scene, keyframes, sparse_density, camera, seed)
    out = Path(out_dir)
    try:
        out.mkdir(parents=True, exist_ok=True)
    except OSError as exc:
        raise DatasetError(f"cannot create dataset directory {out}: {exc}") from exc
    entries = []
    for kf in frames:
        name = f"kf{kf.id:04d}.png"
        try:
            Image.fromarray(kf.image).save(out / name)
        except OSError as exc:
            raise DatasetError(f"cannot write image {out / name}: {exc}") from exc
        entries.append({"id": kf.id, "image": name, "rotation": [float(v) for v in kf.pose.rotation.reshape(-1)],
                        "translation": [float(v) for v in kf.pose.translation],
                        "sparse_points": [[float(c) for c in pt] for pt in kf.sparse_points]})
    manifest = {"camera": {"width": camera.width, "height": camera.height}, "keyframes": entries,
                "synthetic": scene_to_dict(scene)}
    try:
        with open(out / "dataset.json", "w", encoding="utf-8") as fh:
            json.dump(manifest, fh, indent=1)
    except OSError as exc:
        raise DatasetError(f"cannot write manifest {out / 'dataset.json'}: {exc}") from exc
    return out
