"""ctypes binding of libd360.so — the C ABI declared in include/d360.h.

The library is the product: if it is missing or cannot be loaded this module raises
BackendError.  Nothing here (or anywhere in the package) falls back to a CPU path.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

from .errors import BackendError

PREC_EXACT = 0
PREC_MIXED = 1

MAX_VIEWS = 8
MAX_SAMPLES = 128
MAX_REFINE = 16
MAX_FRAMES = 8

import os

# D360_LIB_PATH selects another build of the same ABI (kernel-variant experiments only)
_LIB_PATH = Path(os.environ.get("D360_LIB_PATH") or Path(__file__).resolve().parent / "libd360.so")
_lib = None

c_void = C.c_void_p


class Group(C.Structure):
    """struct d360_group"""

    _fields_ = [
        ("width", C.c_int32), ("height", C.c_int32), ("n_views", C.c_int32), ("n_samples", C.c_int32),
        ("top_k", C.c_int32), ("precision", C.c_int32),
        ("rays", c_void), ("ref_gray", c_void), ("nb", c_void), ("nb_pad_x", C.c_int32), ("nb_pad_y", C.c_int32),
        ("nb64", c_void),
        ("rel_r", c_void), ("rel_t", c_void), ("offsets", c_void),
        ("trunc", C.c_double),
        ("ref_ctx", c_void), ("ref_ctx_pad", C.c_int32),
    ]


_SIGNATURES = {
    "d360_last_error": (C.c_char_p, []),
    "d360_version": (C.c_int, []),
    "d360_launch_count": (C.c_ulonglong, []),
    "d360_generic_fallbacks": (C.c_ulonglong, []),
    "d360_trace_enable": (C.c_int, [C.c_int]),
    "d360_trace_summary": (C.c_int, [C.c_char_p, C.c_int]),
    "d360_eval_costs": (C.c_int, [C.POINTER(Group), c_void, c_void, c_void, c_void]),
    "d360_red_black_pass": (C.c_int, [C.POINTER(Group), C.c_int] + [c_void] * 8),
    "d360_refine_pass": (C.c_int, [C.POINTER(Group)] + [c_void] * 8 + [C.c_int, C.c_double, C.c_double, c_void]),
    "d360_run_patchmatch": (C.c_int, [C.POINTER(Group)] + [c_void] * 9 + [C.c_int, C.c_int, C.c_double,
                                                                         C.c_double, c_void, c_void, c_void]),
    "d360_build_ref_context": (C.c_int, [c_void, c_void, c_void, C.c_int, C.c_int, C.c_int, c_void]),
    "d360_median_support_mask": (C.c_int, [c_void, c_void, C.c_int, C.c_double, c_void, C.c_int, C.c_int, c_void]),
    "d360_to_gray": (C.c_int, [c_void, C.c_int, c_void, C.c_int, C.c_int, c_void]),
    "d360_to_gray_padded": (C.c_int, [c_void, C.c_int, c_void, c_void, C.c_int, C.c_int, C.c_int, C.c_int, c_void]),
    "d360_camera_rays": (C.c_int, [c_void] * 6 + [C.c_int, C.c_int, c_void]),
    "d360_random_init": (C.c_int, [c_void] * 6 + [C.c_uint64, C.c_double, C.c_double, c_void, C.c_int, C.c_int,
                                                  c_void]),
    "d360_warp_plane_map": (C.c_int, [c_void] * 7 + [C.c_double, C.c_double] + [c_void] * 5 + [C.c_int, C.c_int,
                                                                                              c_void]),
    "d360_pole_mask": (C.c_int, [c_void, C.c_double, C.c_int, C.c_int, c_void]),
    "d360_consistency_filter": (C.c_int, [c_void] * 8 + [C.c_int, c_void, C.c_int, C.c_double, c_void, C.c_int,
                                                         C.c_int, c_void]),
    "d360_fuse_blocks": (C.c_int, [C.c_int, C.c_int]),
    "d360_fuse_oldest": (C.c_int, [c_void] * 9 + [C.c_int, c_void, C.c_double, C.c_double] + [c_void] * 5 +
                         [C.c_int, C.c_int, c_void]),
    "d360_resample_u8": (C.c_int, [c_void, C.c_int, C.c_int, C.c_int, c_void, c_void, C.c_int, C.c_int, c_void, c_void,
                                   C.c_int, c_void, c_void, C.c_int, C.c_int, C.c_int, c_void]),
    "d360_render_scene": (C.c_int, [C.c_int, C.c_int, c_void, C.c_double, C.c_int, C.c_double, C.c_int, c_void, c_void,
                                    c_void, c_void, c_void, C.c_int, C.c_int, c_void]),
    "d360_render_box_scene": (C.c_int, [c_void, C.c_int, C.c_double, C.c_int, c_void, c_void, c_void, c_void,
                                        c_void, C.c_int, C.c_int, c_void]),
    "d360_measure_fma_peak": (C.c_double, [C.c_int, C.c_int]),
    "d360_pack_ply_records": (C.c_int, [c_void, c_void, c_void, C.c_int64, c_void]),
    "d360_depth_to_mm16": (C.c_int, [c_void, c_void, c_void, c_void, C.c_int, C.c_int, c_void]),
    "d360_completeness_splat": (C.c_int, [c_void, C.c_int64, c_void, c_void, c_void, C.c_int, C.c_int, c_void]),
    "d360_count_nonzero": (C.c_int, [c_void, C.c_int64, c_void, c_void]),
    "d360_accuracy_scratch_doubles": (C.c_int, []),
    "d360_depth_accuracy": (C.c_int, [c_void, c_void, c_void, c_void, C.c_int64, c_void, c_void, c_void]),
    "d360_voxel_keys": (C.c_int, [c_void, C.c_int64, C.c_double, c_void, c_void, c_void]),
}

EXPORTED_SYMBOLS = tuple(_SIGNATURES)


def lib_path() -> Path:
    return _LIB_PATH


def load():
    """Load libd360.so once; raise BackendError if it is absent (no fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists():
        raise BackendError(
            f"{_LIB_PATH} is missing: build it with `python -m paper_2211_16266_b200._build` "
            "(nvcc, sm_100a).  This package has no CPU fallback."
        )
    try:
        lib = C.CDLL(str(_LIB_PATH))
    except OSError as exc:
        raise BackendError(f"cannot load {_LIB_PATH}: {exc}") from exc
    for name, (restype, argtypes) in _SIGNATURES.items():
        try:
            fn = getattr(lib, name)
        except AttributeError as exc:
            raise BackendError(f"{_LIB_PATH} does not export {name}") from exc
        fn.restype = restype
        fn.argtypes = argtypes
    _lib = lib
    return lib


def launch_count() -> int:
    """Kernels launched by libd360 since it was loaded."""
    return int(load().d360_launch_count())


def generic_fallbacks() -> int:
    """Launches that fell off the throughput kernels onto the generic ones (include/d360.h)."""
    return int(load().d360_generic_fallbacks())


def trace_enable(on: bool) -> None:
    """Start (and clear) or stop per-launch CUDA-event timing inside the library."""
    load().d360_trace_enable(1 if on else 0)


def trace_summary() -> dict:
    """{kernel kind: (launches, total device ms)} since trace_enable(True)."""
    buf = C.create_string_buffer(1 << 16)
    n = load().d360_trace_summary(buf, len(buf))
    if n < 0:
        check(1, "trace_summary")
    out = {}
    for line in buf.raw[:n].decode().splitlines():
        kind, cnt, ms = line.split()
        out[kind] = (int(cnt), float(ms))
    return out


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().d360_last_error()
        raise BackendError(f"{what} failed (status {rc}): {msg.decode() if msg else 'unknown error'}")
