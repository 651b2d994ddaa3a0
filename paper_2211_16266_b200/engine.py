"""Plane-hypothesis stereo for one equirectangular reference keyframe — host side.

Mirrors the public surface of the reference's ``densify360.engine`` (E = engine.py there):
``PatchSpec``, ``PlaneMap``, ``DepthPanorama``, ``prepare_group``, ``random_init``,
``warp_plane_map``, ``red_black_iteration``, ``run_patchmatch``, ``median_outlier_filter``.
The numpy-facing functions keep the reference's argument meaning and error behaviour; every
per-pixel computation is a CUDA kernel behind the C ABI of ``include/d360.h``.  State can
also stay on the device between calls (``DevicePlaneMap`` and the ``*_device`` functions),
which is what ``DepthStage`` and the benchmark use.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import BackendError, ConfigError
from .geometry import EquirectCamera, RigidPose, relative_transform, trig_tables
from .keyframes import StereoGroup

DEFAULT_REFINE_THETA_DEG = 60.0  # E:29
DEFAULT_REFINE_DEPTH_FRACTION = 0.25  # E:30
REFINE_CANDIDATES = 6  # E:31

PRECISIONS = {"exact": _lib.PREC_EXACT, "mixed": _lib.PREC_MIXED}
DEFAULT_PRECISION = "mixed"


def default_top_k(n_views: int) -> int:
    """V <= 2: every view (the reference's plain mean, K:297); V > 2: the better half."""
    return n_views if n_views <= 2 else max(2, n_views // 2)


# ---------------------------------------------------------------------------------------
# device plumbing
# ---------------------------------------------------------------------------------------

def _device(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise BackendError("no CUDA device is visible; this package has no CPU fallback")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(device)
    if dev.type != "cuda":
        raise BackendError(f"device must be a CUDA device, got {dev}; this package has no CPU fallback")
    if dev.index is None:  # "cuda" == the current device; tensors report an index, so carry one too
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t) -> int:
    return 0 if t is None else t.data_ptr()


def _up(a: np.ndarray, dtype, device) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=dtype)).to(device, non_blocking=False)


def _image_on_device(image, device) -> torch.Tensor:
    """uint8 image as a tensor on ``device``.  CUDA tensors pass through; a CPU tensor in pinned memory is copied
    asynchronously on the current stream (the caller keeps it alive and unchanged until that copy has run - the
    contract of every pinned staging buffer), so the host does not wait for the kernels already queued; numpy
    arrays and pageable tensors take the blocking copy."""
    if isinstance(image, torch.Tensor):
        if image.device.type == "cuda":
            return image
        return image.contiguous().to(device, non_blocking=image.is_pinned())
    return _up(np.asarray(image), np.uint8, device)


class DeviceCamera:
    """Per-(camera, device) constants: trig tables and pixel rays in f32 and f64."""

    _cache: dict = {}

    def __init__(self, camera: EquirectCamera, device: torch.device):
        lib = _lib.load()
        self.camera = camera
        self.device = device
        h, w = camera.shape
        with torch.cuda.device(device):
            tabs = [_up(t, np.float64, device) for t in trig_tables(camera)]
            self.rays32 = torch.empty((h, w, 3), dtype=torch.float32, device=device)
            self.rays64 = torch.empty((h, w, 3), dtype=torch.float64, device=device)
            _lib.check(lib.d360_camera_rays(_ptr(tabs[0]), _ptr(tabs[1]), _ptr(tabs[2]), _ptr(tabs[3]),
                                            _ptr(self.rays32), _ptr(self.rays64), h, w, _stream()),
                       "camera_rays")
            torch.cuda.current_stream().synchronize()

    @classmethod
    def get(cls, camera: EquirectCamera, device=None) -> "DeviceCamera":
        dev = _device(device)
        key = (camera.width, camera.height, dev.index)
        if key not in cls._cache:
            cls._cache[key] = cls(camera, dev)
        return cls._cache[key]


# ---------------------------------------------------------------------------------------
# value types (reference E:34-134)
# ---------------------------------------------------------------------------------------

@dataclass(frozen=True)
class PatchSpec:
    """Patch sampling grid and cost truncation (E:34-65)."""

    half_window: int = 5
    sample_stride: int = 2
    cost_truncation: float = 1.2

    def __post_init__(self) -> None:
        if self.half_window < 1:
            raise ConfigError(f"patchmatch.half_window must be >= 1, got {self.half_window}")
        if self.sample_stride < 1:
            raise ConfigError(f"patchmatch.sample_stride must be >= 1, got {self.sample_stride}")
        if not self.cost_truncation > 0:
            raise ConfigError(f"patchmatch.cost_truncation must be > 0, got {self.cost_truncation}")

    def sample_offsets(self) -> np.ndarray:
        """(S, 2) int32 (dx, dy), dy outer / dx inner (E:60-65)."""
        reach = (self.half_window // self.sample_stride) * self.sample_stride
        steps = np.arange(-reach, reach + 1, self.sample_stride, dtype=np.int32)
        grid_y, grid_x = np.meshgrid(steps, steps, indexing="ij")
        return np.stack([grid_x.ravel(), grid_y.ravel()], axis=1).astype(np.int32)


@dataclass
class PlaneMap:
    """Host (numpy) plane hypotheses + cost + validity (E:68-118)."""

    camera: EquirectCamera
    depth: np.ndarray
    normal: np.ndarray
    cost: np.ndarray
    valid: np.ndarray
    depth_range: tuple

    @classmethod
    def empty(cls, camera: EquirectCamera, depth_range) -> "PlaneMap":
        h, w = camera.shape
        return cls(camera, np.zeros((h, w), np.float32), np.zeros((h, w, 3), np.float32),
                   np.full((h, w), np.inf, np.float32), np.zeros((h, w), bool), tuple(depth_range))

    @property
    def width(self) -> int:
        return self.camera.width

    @property
    def height(self) -> int:
        return self.camera.height

    def copy(self) -> "PlaneMap":
        return PlaneMap(self.camera, self.depth.copy(), self.normal.copy(), self.cost.copy(),
                        self.valid.copy(), self.depth_range)

    def hypothesis(self, x: int, y: int):
        from .geometry import PlaneHypothesis

        return PlaneHypothesis(depth=float(self.depth[y, x]), normal=self.normal[y, x].astype(np.float64))


@dataclass
class DepthPanorama:
    """Dense depth + validity (E:121-134)."""

    camera: EquirectCamera
    depth: np.ndarray
    valid: np.ndarray

    def copy(self) -> "DepthPanorama":
        return DepthPanorama(self.camera, self.depth.copy(), self.valid.copy())

    @property
    def valid_count(self) -> int:
        return int(self.valid.sum())


class DevicePlaneMap:
    """PlaneMap whose arrays live in HBM: depth (H,W) f32, normal (H,W,3) f32, cost (H,W) f32,
    valid (H,W) u8 — the same layouts as the numpy type, 21 B per pixel."""

    def __init__(self, camera, depth, normal, cost, valid, depth_range):
        self.camera = camera
        self.depth, self.normal, self.cost, self.valid = depth, normal, cost, valid
        self.depth_range = tuple(depth_range)

    @classmethod
    def empty(cls, camera: EquirectCamera, depth_range, device=None) -> "DevicePlaneMap":
        dev = _device(device)
        h, w = camera.shape
        return cls(camera, torch.zeros((h, w), dtype=torch.float32, device=dev),
                   torch.zeros((h, w, 3), dtype=torch.float32, device=dev),
                   torch.full((h, w), float("inf"), dtype=torch.float32, device=dev),
                   torch.zeros((h, w), dtype=torch.uint8, device=dev), depth_range)

    @classmethod
    def from_host(cls, pm: PlaneMap, device=None) -> "DevicePlaneMap":
        dev = _device(device)
        return cls(pm.camera, _up(pm.depth, np.float32, dev), _up(pm.normal, np.float32, dev),
                   _up(pm.cost, np.float32, dev), _up(pm.valid.astype(np.uint8), np.uint8, dev), pm.depth_range)

    def to_host(self) -> PlaneMap:
        return PlaneMap(self.camera, self.depth.cpu().numpy(), self.normal.cpu().numpy(), self.cost.cpu().numpy(),
                        self.valid.cpu().numpy().astype(bool), self.depth_range)

    def clone(self) -> "DevicePlaneMap":
        return DevicePlaneMap(self.camera, self.depth.clone(), self.normal.clone(), self.cost.clone(),
                              self.valid.clone(), self.depth_range)

    @property
    def device(self):
        return self.depth.device


class DeviceDepthPanorama:
    def __init__(self, camera, depth, valid):
        self.camera, self.depth, self.valid = camera, depth, valid

    def to_host(self) -> DepthPanorama:
        return DepthPanorama(self.camera, self.depth.cpu().numpy(), self.valid.cpu().numpy().astype(bool))

    @classmethod
    def from_host(cls, p: DepthPanorama, device=None) -> "DeviceDepthPanorama":
        dev = _device(device)
        return cls(p.camera, _up(p.depth, np.float32, dev), _up(p.valid.astype(np.uint8), np.uint8, dev))


# ---------------------------------------------------------------------------------------
# PreparedGroup (E:137-160): images -> luma on the device, rays, relative poses, offsets
# ---------------------------------------------------------------------------------------

NB_PAD_X = 4  # wrapped columns each side of a neighbour plane (keeps rows 16-byte aligned)
NB_PAD_Y = 1  # replicated rows above / below
REF_CTX_PAD = 8  # wrapped columns / replicated rows of the reference context plane (>= any patch reach)


def to_gray_device(image, device=None, out: torch.Tensor | None = None, pad=(0, 0),
                   out64: torch.Tensor | None = None) -> torch.Tensor:
    """uint8 (H,W) / (H,W,3) numpy array or CUDA tensor -> float32 luma on the device
    (keyframes.py:64-72, float32 arithmetic).

    ``pad=(px, py)`` writes the padded plane layout of ``d360_group.nb``: shape
    (H + 2 py, W + 2 px) with wrapped columns and replicated rows.  ``out``: optional
    contiguous float32 target of that shape; ``out64``: optional float64 target of shape
    (..., 2) that receives, per texel, the exactly widened value and the difference to its right
    neighbour (layout of ``d360_group.nb64``)."""
    dev = _device(device)
    lib = _lib.load()
    img = _image_on_device(image, dev)
    if img.dtype != torch.uint8:
        raise ValueError(f"expected a uint8 image, got {img.dtype}")
    if img.ndim == 2:
        ch = 1
    elif img.ndim == 3 and img.shape[2] == 3:
        ch = 3
    else:
        raise ValueError(f"expected (H, W) or (H, W, 3) image, got {tuple(img.shape)}")
    img = img.contiguous()
    h, w = img.shape[:2]
    px, py = int(pad[0]), int(pad[1])
    shape = (h + 2 * py, w + 2 * px)
    if out is None:
        out = torch.empty(shape, dtype=torch.float32, device=dev)
    elif tuple(out.shape) != shape or out.dtype != torch.float32 or not out.is_contiguous():
        raise ValueError(f"out must be a contiguous float32 {shape} tensor")
    if out64 is not None and (tuple(out64.shape) != (*shape, 2) or out64.dtype != torch.float64 or
                              not out64.is_contiguous()):
        raise ValueError(f"out64 must be a contiguous float64 {(*shape, 2)} tensor")
    for name, t in (("image", img), ("out", out), ("out64", out64)):
        if t is not None and t.device != dev:
            raise ValueError(f"{name} lives on {t.device}, the launch device is {dev}")
    with torch.cuda.device(dev):
        _lib.check(lib.d360_to_gray_padded(_ptr(img), ch, _ptr(out), _ptr(out64), h, w, px, py, _stream()),
                   "to_gray")
    return out


def to_gray(image: np.ndarray) -> np.ndarray:
    """Drop-in for keyframes.to_gray (computed on the GPU)."""
    return to_gray_device(image).cpu().numpy()


class DeviceKeyframe:
    """One keyframe's device-side planes, computed once and shared by every stereo group the
    keyframe takes part in (as the reference or as a neighbour): uint8 image, dense f32 luma,
    padded f32 luma and its f64 widening (layout of ``d360_group.nb`` / ``nb64``)."""

    def __init__(self, image, camera: EquirectCamera, device=None):
        self.device = _device(device)
        h, w = camera.shape
        with torch.cuda.device(self.device):
            img = _image_on_device(image, self.device)
            if tuple(img.shape[:2]) != (h, w):
                raise ValueError(f"image {tuple(img.shape[:2])} does not match camera {(h, w)}")
            self.image = img
            self.gray = to_gray_device(img, self.device)
            shape = (h + 2 * NB_PAD_Y, w + 2 * NB_PAD_X)
            self.padded32 = torch.empty(shape, dtype=torch.float32, device=self.device)
            self.padded64 = torch.empty((*shape, 2), dtype=torch.float64, device=self.device)
            to_gray_device(img, self.device, out=self.padded32, pad=(NB_PAD_X, NB_PAD_Y), out64=self.padded64)


class PreparedGroup:
    """Stereo group unpacked into the kernel layout, resident on one GPU.

    ``device_images``: optional uint8 CUDA tensors (reference first) instead of the keyframes'
    host images; ``device_keyframes``: optional ``DeviceKeyframe`` list (reference first) whose
    cached planes are gathered instead of recomputing the luma; ``buffers``: optional dict a
    per-keyframe loop passes again and again — the group's planes (180 MB at 1920x960, V = 4) then
    live in the same memory for every group of the stream instead of going through the allocator
    (the previous group must no longer be in use; work on one stream is ordered anyway)."""

    def __init__(self, group: StereoGroup, spec: PatchSpec, top_k: int | None = None,
                 precision: str | None = None, device=None, device_images=None, device_keyframes=None,
                 buffers: dict | None = None):
        self.group = group
        self.spec = spec
        self.camera = group.camera
        self.device = _device(device)
        self.n_views = len(group.neighbors)
        self.top_k = default_top_k(self.n_views) if top_k is None else int(top_k)
        if not 1 <= self.top_k <= self.n_views:
            raise ConfigError(f"patchmatch.top_k must be in [1, {self.n_views}], got {self.top_k}")
        self.precision = DEFAULT_PRECISION if precision is None else precision
        if self.precision not in PRECISIONS:
            raise ConfigError(f"patchmatch.precision must be one of {sorted(PRECISIONS)}, got {self.precision!r}")
        self.offsets = spec.sample_offsets()
        if len(self.offsets) > _lib.MAX_SAMPLES:
            raise ConfigError(f"patch has {len(self.offsets)} samples; at most {_lib.MAX_SAMPLES} are supported")
        with torch.cuda.device(self.device):
            self.cam_dev = DeviceCamera.get(self.camera, self.device)
            h, w = self.camera.shape
            # neighbour luma planes, padded so that every bilinear footprint is in-plane (d360.h),
            # and the same planes widened to f64: the reference interpolates in f64 (K:134-153)
            def plane(name, shape, dtype):
                if buffers is None:
                    return torch.empty(shape, dtype=dtype, device=self.device)
                t = buffers.get(name)
                if t is None or tuple(t.shape) != tuple(shape) or t.dtype != dtype or t.device != self.device:
                    t = buffers[name] = torch.empty(shape, dtype=dtype, device=self.device)
                return t

            self.nb_padded = plane("nb32", (self.n_views, h + 2 * NB_PAD_Y, w + 2 * NB_PAD_X), torch.float32)
            self.nb64_padded = plane("nb64", (*self.nb_padded.shape, 2), torch.float64)
            if device_keyframes is not None:
                if len(device_keyframes) != self.n_views + 1:
                    raise ValueError("device_keyframes must list the reference and every neighbour")
                self.ref_image = device_keyframes[0].image
                self.ref_gray = device_keyframes[0].gray
                for v, dk in enumerate(device_keyframes[1:]):
                    self.nb_padded[v].copy_(dk.padded32)
                    self.nb64_padded[v].copy_(dk.padded64)
            else:
                imgs = device_images if device_images is not None else (
                    [group.reference.image] + [nb.image for nb in group.neighbors])
                ref_img = imgs[0] if isinstance(imgs[0], torch.Tensor) else _up(np.asarray(imgs[0]), np.uint8,
                                                                                 self.device)
                self.ref_image = ref_img  # u8 (H,W) / (H,W,3) on the device; fusion reads its colours
                self.ref_gray = to_gray_device(ref_img, self.device)
                for v, im in enumerate(imgs[1:]):
                    to_gray_device(im, self.device, out=self.nb_padded[v], pad=(NB_PAD_X, NB_PAD_Y),
                                   out64=self.nb64_padded[v])
            # (ray, luma) of the reference as one padded float4 plane: the TMA source of the patch windows
            self.ref_ctx = None
            if self.precision == "mixed":
                self.ref_ctx = plane("ctx", (h + 2 * REF_CTX_PAD, w + 2 * REF_CTX_PAD, 4), torch.float32)
                _lib.check(_lib.load().d360_build_ref_context(_ptr(self.cam_dev.rays32), _ptr(self.ref_gray),
                                                              _ptr(self.ref_ctx), h, w, REF_CTX_PAD, _stream()),
                           "build_ref_context")
        rel = [relative_transform(group.reference.pose, nb.pose) for nb in group.neighbors]
        self.rel_r = np.ascontiguousarray(np.stack([r for r, _ in rel]), dtype=np.float32)
        self.rel_t = np.ascontiguousarray(np.stack([t for _, t in rel]), dtype=np.float32)
        self._struct = _lib.Group(
            width=self.camera.width, height=self.camera.height, n_views=self.n_views,
            n_samples=len(self.offsets), top_k=self.top_k, precision=PRECISIONS[self.precision],
            rays=_ptr(self.cam_dev.rays32), ref_gray=_ptr(self.ref_gray), nb=_ptr(self.nb_padded), nb_pad_x=NB_PAD_X, nb_pad_y=NB_PAD_Y, nb64=_ptr(self.nb64_padded),
            rel_r=self.rel_r.ctypes.data, rel_t=self.rel_t.ctypes.data, offsets=self.offsets.ctypes.data,
            trunc=float(spec.cost_truncation),
            ref_ctx=_ptr(self.ref_ctx) if self.ref_ctx is not None else 0, ref_ctx_pad=REF_CTX_PAD)

    @property
    def nb(self) -> torch.Tensor:
        """(V, H, W) view of the neighbour luma planes without the padding."""
        return self.nb_padded[:, NB_PAD_Y:-NB_PAD_Y, NB_PAD_X:-NB_PAD_X]

    @property
    def struct(self):
        return C.byref(self._struct)


def prepare_group(group: StereoGroup, spec: PatchSpec, **kw) -> PreparedGroup:
    return PreparedGroup(group, spec, **kw)


def _as_prepared(group, spec: PatchSpec) -> PreparedGroup:
    return group if isinstance(group, PreparedGroup) else PreparedGroup(group, spec)


# ---------------------------------------------------------------------------------------
# random_init (E:244-283)
# ---------------------------------------------------------------------------------------

def _check_depth_range(depth_range):
    dmin, dmax = float(depth_range[0]), float(depth_range[1])
    if not (dmin > 0.0 and dmax > dmin):
        raise ConfigError(f"patchmatch.depth_range must satisfy 0 < min < max, got [{dmin}, {dmax}]")
    return dmin, dmax


def random_init_device(pm: DevicePlaneMap, depth_range, seed: int, rng: str = "pcg64") -> DevicePlaneMap:
    """Fill every invalid pixel in place with a random plane; mark everything valid.

    rng="pcg64": the reference's NumPy draws are generated on the host and injected, so the
    hypotheses are the reference's.  rng="philox": counter-based Philox4x32-10 on the device
    (same distributions, no host work)."""
    dmin, dmax = _check_depth_range(depth_range)
    lib = _lib.load()
    cam = DeviceCamera.get(pm.camera, pm.device)
    h, w = pm.camera.shape
    with torch.cuda.device(pm.device):
        if rng == "pcg64":
            gen = np.random.default_rng(seed)
            inv = _up(gen.uniform(1.0 / dmax, 1.0 / dmin, size=(h, w)), np.float64, pm.device)
            g = _up(gen.standard_normal((h, w, 3)), np.float64, pm.device)
        elif rng == "philox":
            inv = g = None
        else:
            raise ConfigError(f"rng must be 'pcg64' or 'philox', got {rng!r}")
        _lib.check(lib.d360_random_init(_ptr(pm.depth), _ptr(pm.normal), _ptr(pm.cost), _ptr(pm.valid), _ptr(inv),
                                        _ptr(g), int(seed) & 0xFFFFFFFFFFFFFFFF, dmin, dmax, _ptr(cam.rays64),
                                        h, w, _stream()), "random_init")
    pm.depth_range = (dmin, dmax)
    return pm


def random_init(plane_map: PlaneMap, depth_range, seed: int, rng: str = "pcg64") -> PlaneMap:
    _check_depth_range(depth_range)
    dev = DevicePlaneMap.from_host(plane_map)
    return random_init_device(dev, depth_range, seed, rng).to_host()


# ---------------------------------------------------------------------------------------
# warp_plane_map (E:286-355)
# ---------------------------------------------------------------------------------------

def warp_plane_map_device(previous: DevicePlaneMap, pose_prev: RigidPose, pose_cur: RigidPose,
                          camera: EquirectCamera, winner: torch.Tensor | None = None) -> DevicePlaneMap:
    """``winner``: optional (H, W) int64 scratch (the packed (cost, source) of the scatter); pass a
    persistent one in a per-keyframe loop — a fresh 8 B/pixel allocation every call can miss the
    caching allocator and cost a cudaMalloc (tens of ms) in the middle of a step."""
    if previous.camera != camera:
        raise ConfigError(f"plane map camera {previous.camera} does not match target camera {camera}")
    lib = _lib.load()
    dev = previous.device
    cam = DeviceCamera.get(camera, dev)
    h, w = camera.shape
    out = DevicePlaneMap(camera, torch.empty_like(previous.depth), torch.empty_like(previous.normal),
                         torch.empty_like(previous.cost), torch.empty_like(previous.valid), previous.depth_range)
    r_rel, t_rel = relative_transform(pose_prev, pose_cur)
    r_rel = np.ascontiguousarray(r_rel, np.float64)
    t_rel = np.ascontiguousarray(t_rel, np.float64)
    with torch.cuda.device(dev):
        if winner is None:
            winner = torch.empty((h, w), dtype=torch.int64, device=dev)
        _lib.check(lib.d360_warp_plane_map(_ptr(previous.depth), _ptr(previous.normal), _ptr(previous.cost),
                                           _ptr(previous.valid), _ptr(cam.rays64), r_rel.ctypes.data,
                                           t_rel.ctypes.data, float(previous.depth_range[0]),
                                           float(previous.depth_range[1]), _ptr(out.depth), _ptr(out.normal),
                                           _ptr(out.cost), _ptr(out.valid), _ptr(winner), h, w, _stream()),
                   "warp_plane_map")
    return out


def warp_plane_map(previous: PlaneMap, pose_prev: RigidPose, pose_cur: RigidPose, camera: EquirectCamera) -> PlaneMap:
    return warp_plane_map_device(DevicePlaneMap.from_host(previous), pose_prev, pose_cur, camera).to_host()


# ---------------------------------------------------------------------------------------
# cost evaluation / propagation / refinement
# ---------------------------------------------------------------------------------------

def _check_initialized(valid_all: bool) -> None:
    if not valid_all:
        raise ConfigError("run_patchmatch requires a fully initialized plane map; "
                          "fill unfilled pixels with random_init first")


def evaluate_costs_device(prep: PreparedGroup, pm: DevicePlaneMap) -> None:
    """cost <- matching cost of every pixel's hypothesis (kernels.eval_costs, K:300-349)."""
    lib = _lib.load()
    with torch.cuda.device(prep.device):
        _lib.check(lib.d360_eval_costs(prep.struct, _ptr(pm.depth), _ptr(pm.normal), _ptr(pm.cost), _stream()),
                   "eval_costs")


def red_black_pass_device(prep: PreparedGroup, parity: int, src: DevicePlaneMap, dst: DevicePlaneMap,
                          n_evals: torch.Tensor | None = None) -> None:
    """One pass of K:352-473.  ``src.cost`` must hold the true costs of ``src``'s hypotheses (as after
    ``evaluate_costs_device`` or an earlier pass): the mixed policy's duplicate rule relies on it, see
    include/d360.h."""
    lib = _lib.load()
    with torch.cuda.device(prep.device):
        _lib.check(lib.d360_red_black_pass(prep.struct, int(parity), _ptr(src.depth), _ptr(src.normal),
                                           _ptr(src.cost), _ptr(dst.depth), _ptr(dst.normal), _ptr(dst.cost),
                                           _ptr(n_evals), _stream()), "red_black_pass")


def refine_pass_device(prep: PreparedGroup, pm: DevicePlaneMap, table, depth_range) -> None:
    lib = _lib.load()
    dd, sa, ca, caz, saz = (np.ascontiguousarray(t, np.float32) for t in table)
    with torch.cuda.device(prep.device):
        _lib.check(lib.d360_refine_pass(prep.struct, _ptr(pm.depth), _ptr(pm.normal), _ptr(pm.cost),
                                        dd.ctypes.data, sa.ctypes.data, ca.ctypes.data, caz.ctypes.data,
                                        saz.ctypes.data, len(dd), float(depth_range[0]), float(depth_range[1]),
                                        _stream()), "refine_pass")


def red_black_iteration(plane_map: PlaneMap, group, spec: PatchSpec, parity) -> PlaneMap:
    """One checkerboard pass on a host plane map (E:382-421)."""
    parity_idx = {"red": 0, "black": 1, 0: 0, 1: 1}.get(parity)
    if parity_idx is None:
        raise ConfigError(f"parity must be 'red' or 'black', got {parity!r}")
    _check_initialized(bool(plane_map.valid.all()))
    prep = _as_prepared(group, spec)
    cur = DevicePlaneMap.from_host(plane_map, prep.device)
    if not np.isfinite(plane_map.cost).all():
        evaluate_costs_device(prep, cur)
    out = cur.clone()
    red_black_pass_device(prep, parity_idx, cur, out)
    return out.to_host()


def refinement_draw_tables(seed: int, iterations: int, delta_d: float, theta: float) -> np.ndarray:
    """(iterations, 5, 6) f32: rows (dd, sin ang, cos ang, cos az, sin az), drawn with NumPy
    PCG64 in the reference's order so both paths share one schedule (E:495-526)."""
    rng = np.random.default_rng(seed)
    out = np.empty((iterations, 5, REFINE_CANDIDATES), np.float32)
    for it in range(iterations):
        draws = np.empty((REFINE_CANDIDATES, 3), np.float64)
        for i in range(REFINE_CANDIDATES):
            shrink = 0.5**i
            draws[i, 0] = rng.uniform(-1.0, 1.0) * delta_d * shrink
            draws[i, 1] = rng.uniform(0.0, 1.0) * theta * shrink
            draws[i, 2] = rng.uniform(0.0, 2.0 * math.pi)
        out[it, 0] = draws[:, 0].astype(np.float32)
        out[it, 1] = np.sin(draws[:, 1]).astype(np.float32)
        out[it, 2] = np.cos(draws[:, 1]).astype(np.float32)
        out[it, 3] = np.cos(draws[:, 2]).astype(np.float32)
        out[it, 4] = np.sin(draws[:, 2]).astype(np.float32)
    return out


class PatchMatchWorkspace:
    """Ping-pong buffers and the evaluation counter reused across keyframes of one size."""

    def __init__(self, camera: EquirectCamera, device):
        h, w = camera.shape
        self.depth = torch.empty((h, w), dtype=torch.float32, device=device)
        self.normal = torch.empty((h, w, 3), dtype=torch.float32, device=device)
        self.cost = torch.empty((h, w), dtype=torch.float32, device=device)
        self.flags = torch.empty((3, h, w), dtype=torch.uint8, device=device)    # changed (x2), memo validity
        self.memo = torch.empty((h, w, 8), dtype=torch.float64, device=device)  # memoised candidate costs
        self.n_evals = torch.zeros((2,), dtype=torch.int64, device=device)  # [evaluations, cut short]
        self.winner = torch.empty((h, w), dtype=torch.int64, device=device)  # scratch of warp_plane_map


def run_patchmatch_device(prep: PreparedGroup, pm: DevicePlaneMap, iterations: int, seed: int,
                          refine_theta_deg: float = DEFAULT_REFINE_THETA_DEG,
                          refine_depth_fraction: float = DEFAULT_REFINE_DEPTH_FRACTION,
                          workspace: PatchMatchWorkspace | None = None, count_evals: bool = False,
                          check_valid: bool = True, skip_unchanged: bool = True, probes: bool | None = None):
    """Optimise ``pm`` in place on the device; returns (pm, DeviceDepthPanorama).

    ``probes`` (default: environment variable D360_PROBES=1): the reference's monotonicity spot checks
    (E:567-570, E:596-598, E:622-624) - the cost at 8 fixed probe pixels is read back after every pass and
    must not have increased, else AssertionError with the reference's message.  The passes are then
    enqueued one C-ABI call at a time with a read-back in between (a debugging mode: same results, bit
    for bit, without the memoised candidate costs and with 1 + 3 x iterations synchronisations).

    One C-ABI call (d360_run_patchmatch) enqueues eval + iterations x (red, black, refine).
    With ``count_evals`` the executed propagation/refinement cost evaluations are ADDED to
    ``workspace.n_evals[0]`` and the refinement evaluations decided after V - 1 views to
    ``workspace.n_evals[1]`` (zero it yourself; reading it synchronises).  ``skip_unchanged`` lets
    the propagation reuse the cost of a neighbour's hypothesis for as long as that hypothesis does
    not change (memoised, bit-identical results, see include/d360.h); switch it off to count the
    reference's evaluations."""
    if iterations < 1:
        raise ConfigError(f"patchmatch.iterations must be >= 1, got {iterations}")
    if prep.camera != pm.camera:
        raise ConfigError(f"plane map camera {pm.camera} does not match group camera {prep.camera}")
    if check_valid:
        _check_initialized(bool(pm.valid.all().item()))
    lib = _lib.load()
    dmin, dmax = pm.depth_range
    tables = refinement_draw_tables(seed, iterations, refine_depth_fraction * (dmax - dmin),
                                    math.radians(refine_theta_deg))
    ws = workspace if workspace is not None else PatchMatchWorkspace(prep.camera, prep.device)
    if probes is None:
        probes = os.environ.get("D360_PROBES") == "1"
    if probes:
        return _run_patchmatch_probed(prep, pm, iterations, tables, ws, count_evals)
    with torch.cuda.device(prep.device):
        valid = torch.empty(prep.camera.shape, dtype=torch.uint8, device=prep.device)
        _lib.check(lib.d360_run_patchmatch(prep.struct, _ptr(pm.depth), _ptr(pm.normal), _ptr(pm.cost),
                                           _ptr(ws.depth), _ptr(ws.normal), _ptr(ws.cost),
                                           _ptr(ws.flags) if skip_unchanged else 0,
                                           _ptr(ws.memo) if skip_unchanged else 0, tables.ctypes.data,
                                           int(iterations), REFINE_CANDIDATES, float(dmin), float(dmax),
                                           _ptr(valid), _ptr(ws.n_evals) if count_evals else 0, _stream()),
                   "run_patchmatch")
    pano = DeviceDepthPanorama(prep.camera, pm.depth.clone(), valid)
    return pm, pano


def _run_patchmatch_probed(prep: PreparedGroup, pm: DevicePlaneMap, iterations: int, tables: np.ndarray,
                           ws: "PatchMatchWorkspace", count_evals: bool):
    """run_patchmatch pass by pass with the reference's probe-pixel assertions (E:567-624)."""
    h, w = prep.camera.shape
    dev = prep.device
    probe_y = torch.as_tensor(np.linspace(0, h - 1, 8).astype(np.int64), device=dev)
    probe_x = torch.as_tensor(np.linspace(0, w - 1, 8).astype(np.int64), device=dev)
    n_evals = ws.n_evals if count_evals else None
    cur = pm
    nxt = DevicePlaneMap(pm.camera, ws.depth, ws.normal, ws.cost, pm.valid, pm.depth_range)
    evaluate_costs_device(prep, cur)
    for it in range(iterations):
        for parity in (0, 1):
            red_black_pass_device(prep, parity, cur, nxt, n_evals)
            ok = bool((nxt.cost[probe_y, probe_x] <= cur.cost[probe_y, probe_x]).all().item())
            assert ok, "propagation increased a probe pixel's cost"
            cur, nxt = nxt, cur
        before = cur.cost[probe_y, probe_x].clone()
        refine_pass_device(prep, cur, tables[it], pm.depth_range)
        ok = bool((cur.cost[probe_y, probe_x] <= before).all().item())
        assert ok, "refinement increased a probe pixel's cost"
    if cur is not pm:  # never the case: two swaps per iteration
        pm.depth.copy_(cur.depth); pm.normal.copy_(cur.normal); pm.cost.copy_(cur.cost)
    valid = (pm.cost < float(prep.spec.cost_truncation)).to(torch.uint8)
    return pm, DeviceDepthPanorama(prep.camera, pm.depth.clone(), valid)


def run_patchmatch(group, init: PlaneMap, spec: PatchSpec, iterations: int, seed: int, workers: int | None = None,
                   refine_theta_deg: float = DEFAULT_REFINE_THETA_DEG,
                   refine_depth_fraction: float = DEFAULT_REFINE_DEPTH_FRACTION):
    """Drop-in for engine.run_patchmatch (E:529-631): host arrays in, host arrays out.

    ``workers`` is accepted for signature compatibility and ignored (results never depended
    on it, T/test_engine.py:478-488)."""
    if iterations < 1:
        raise ConfigError(f"patchmatch.iterations must be >= 1, got {iterations}")
    _check_initialized(bool(np.asarray(init.valid).all()))
    prep = _as_prepared(group, spec)
    if prep.camera != init.camera:
        raise ConfigError(f"plane map camera {init.camera} does not match group camera {prep.camera}")
    pm = DevicePlaneMap.from_host(init, prep.device)
    pm, pano = run_patchmatch_device(prep, pm, iterations, seed, refine_theta_deg, refine_depth_fraction,
                                     check_valid=False)
    return pm.to_host(), pano.to_host()


# ---------------------------------------------------------------------------------------
# median outlier filter (E:634-648)
# ---------------------------------------------------------------------------------------

def median_outlier_filter_device(pano: DeviceDepthPanorama, window: int = 5,
                                 rel_threshold: float = 0.2) -> DeviceDepthPanorama:
    if window < 3 or window % 2 == 0:
        raise ConfigError(f"median filter window must be odd and >= 3, got {window}")
    lib = _lib.load()
    h, w = pano.camera.shape
    out_valid = torch.empty_like(pano.valid)
    with torch.cuda.device(pano.depth.device):
        _lib.check(lib.d360_median_support_mask(_ptr(pano.depth), _ptr(pano.valid), window // 2,
                                                float(rel_threshold), _ptr(out_valid), h, w, _stream()),
                   "median_support_mask")
    return DeviceDepthPanorama(pano.camera, pano.depth, out_valid)


def median_outlier_filter(depth: DepthPanorama, window: int = 5, rel_threshold: float = 0.2) -> DepthPanorama:
    if window < 3 or window % 2 == 0:
        raise ConfigError(f"median filter window must be odd and >= 3, got {window}")
    out = median_outlier_filter_device(DeviceDepthPanorama.from_host(depth), window, rel_threshold)
    return DepthPanorama(depth.camera, depth.depth.copy(), out.valid.cpu().numpy().astype(bool))


def pole_mask_device(pano: DeviceDepthPanorama, limit_deg: float) -> None:
    """Invalidate rows beyond ``limit_deg`` of latitude in place."""
    lib = _lib.load()
    h, w = pano.camera.shape
    with torch.cuda.device(pano.depth.device):
        _lib.check(lib.d360_pole_mask(_ptr(pano.valid), float(limit_deg), h, w, _stream()), "pole_mask")
