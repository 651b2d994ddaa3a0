"""Image ingest on the device: ``resample_keyframe`` of the reference's ``dataset.py`` (lines 146-157).

The reference resizes with ``PIL.Image.resize((W, H), Image.LANCZOS)``.  Pillow is a third-party
dependency that is not under /root/reference (pinned by this image: Pillow 12.2.0); its algorithm is
the one published in ``src/libImaging/Resample.c``: ``precompute_coeffs`` builds, per output pixel, a
window of source pixels and double-precision Lanczos-3 weights normalised to sum 1,
``normalize_coeffs_8bpc`` rounds them to 22-bit fixed point, and two separable passes (horizontal
first, through a uint8 intermediate) accumulate in int32.  The windows and integer weights (a few
hundred numbers per axis) are computed here on the host with the same statements; the byte work is
``d360_resample_u8``.  Integer arithmetic throughout the passes, so the result equals Pillow's bit for
bit (``tests/test_gpu_parity.py::test_resample_keyframe_equals_pillow_lanczos``).

The dataset directory loader itself (manifest JSON, PNG decode) stays host code and out of scope.
"""
from __future__ import annotations

import math

import numpy as np
import torch

from . import _lib
from .engine import _device, _ptr, _stream, _up
from .geometry import EquirectCamera
from .keyframes import Keyframe

PRECISION_BITS = 32 - 8 - 2  # Resample.c
LANCZOS_SUPPORT = 3.0


def _sinc(x: float) -> float:
    if x == 0.0:
        return 1.0
    x = x * math.pi
    return math.sin(x) / x


def _lanczos(x: float) -> float:
    """Resample.c lanczos_filter: truncated sinc(x) sinc(x / 3)."""
    if -3.0 <= x < 3.0:
        return _sinc(x) * _sinc(x / 3)
    return 0.0


def lanczos_coefficients(in_size: int, out_size: int):
    """Resample.c precompute_coeffs + normalize_coeffs_8bpc for the full-image box (in0 = 0, in1 = in_size).

    Returns (bounds int32 (out_size, 2) = (first source index, tap count), kk int32 (out_size, ksize))."""
    scale = filterscale = float(in_size) / out_size
    if filterscale < 1.0:
        filterscale = 1.0
    support = LANCZOS_SUPPORT * filterscale
    ksize = int(math.ceil(support)) * 2 + 1
    bounds = np.zeros((out_size, 2), np.int32)
    kk = np.zeros((out_size, ksize), np.int32)
    ss = 1.0 / filterscale
    for xx in range(out_size):
        center = 0.0 + (xx + 0.5) * scale
        xmin = int(center - support + 0.5)
        if xmin < 0:
            xmin = 0
        xmax = int(center + support + 0.5)
        if xmax > in_size:
            xmax = in_size
        xmax -= xmin
        w = [_lanczos((x + xmin - center + 0.5) * ss) for x in range(xmax)]
        ww = 0.0
        for v in w:
            ww += v
        for x in range(xmax):
            k = w[x] / ww if ww != 0.0 else w[x]
            kk[xx, x] = int(-0.5 + k * (1 << PRECISION_BITS)) if k < 0 else int(0.5 + k * (1 << PRECISION_BITS))
        bounds[xx] = (xmin, xmax)
    return bounds, kk


def _identity_coefficients(size: int):
    """The pass Pillow skips when an axis keeps its size: one tap of weight 1."""
    bounds = np.stack([np.arange(size, dtype=np.int32), np.ones(size, np.int32)], axis=1)
    return bounds, np.full((size, 1), 1 << PRECISION_BITS, np.int32)


_COEFF_CACHE: dict = {}


def _coefficients(in_size: int, out_size: int, device, relative: bool):
    """Windows and weights of one axis, on the host and (cached per size pair and device) on the device.
    ``relative``: windows counted from the first source row the axis reads (the vertical pass reads the
    intermediate, which starts there)."""
    key = (in_size, out_size, str(device), relative)
    hit = _COEFF_CACHE.get(key)
    if hit is None:
        bounds, kk = _identity_coefficients(in_size) if in_size == out_size else lanczos_coefficients(in_size, out_size)
        first = int(bounds[0, 0])
        span = int(bounds[-1, 0] + bounds[-1, 1]) - first
        dev_bounds = bounds.copy()
        if relative:
            dev_bounds[:, 0] -= first
        hit = _COEFF_CACHE[key] = (_up(dev_bounds, np.int32, device), _up(kk, np.int32, device), kk.shape[1], first, span)
    return hit


def resample_image_device(image, width: int, height: int, device=None) -> torch.Tensor:
    """uint8 (H, W) or (H, W, 3) numpy array or CUDA tensor -> uint8 CUDA tensor of (height, width[, 3]),
    equal to ``PIL.Image.fromarray(image).resize((width, height), Image.LANCZOS)``."""
    dev = _device(device)
    img = image if isinstance(image, torch.Tensor) else _up(np.asarray(image), np.uint8, dev)
    if img.dtype != torch.uint8 or not (img.ndim == 2 or (img.ndim == 3 and img.shape[2] == 3)):
        raise ValueError(f"expected a uint8 (H, W) or (H, W, 3) image, got {img.dtype} {tuple(img.shape)}")
    if img.device != dev:
        raise ValueError(f"image lives on {img.device}, the launch device is {dev}")
    img = img.contiguous()
    sh, sw = img.shape[:2]
    ch = 1 if img.ndim == 2 else 3
    if (sh, sw) == (height, width):
        return img
    lib = _lib.load()
    with torch.cuda.device(dev):
        d_bx, d_kx, ksize_x, _, _ = _coefficients(sw, width, dev, relative=False)
        # Resample.c: the horizontal pass covers source rows ybox_first .. ybox_last only
        d_by, d_ky, ksize_y, row0, rows = _coefficients(sh, height, dev, relative=True)
        tmp = torch.empty((rows, width, ch), dtype=torch.uint8, device=dev)
        out = torch.empty((height, width) if ch == 1 else (height, width, 3), dtype=torch.uint8, device=dev)
        _lib.check(lib.d360_resample_u8(_ptr(img), sh, sw, ch, _ptr(tmp), _ptr(out), height, width, _ptr(d_bx),
                                        _ptr(d_kx), ksize_x, _ptr(d_by), _ptr(d_ky), ksize_y, row0, rows,
                                        _stream()), "resample_u8")
    return out


def resample_keyframe(keyframe: Keyframe, camera: EquirectCamera) -> Keyframe:
    """Drop-in for dataset.resample_keyframe (dataset.py:146-157): the keyframe at another resolution."""
    if tuple(keyframe.image.shape[:2]) == tuple(camera.shape):
        return keyframe
    resized = resample_image_device(keyframe.image, camera.width, camera.height).cpu().numpy()
    return Keyframe(id=keyframe.id, image=resized, pose=keyframe.pose, sparse_points=keyframe.sparse_points)
