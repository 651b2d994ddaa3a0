"""ctypes front-end of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this module.  The product package
``paper_2211_16266_b200`` never does; it fails loudly when its CUDA library is missing.

Everything here works on plain numpy arrays (no product types) so that the oracle and
the product share no code.  Reference shorthand: K = kernels.py, E = engine.py,
P = pipeline.py, G = geometry.py under /root/reference/pkg/src/densify360/.

Parity status: pinned at V=2 by tests/golden/*.npz (produced by oracle/gen_golden.py
from the reference itself); unpinned for V>2 / top-k (no reference implementation).
"""

from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "libd360_oracle.so"

REFINE_CANDIDATES = 6  # E:31
DEFAULT_REFINE_THETA_DEG = 60.0  # E:29
DEFAULT_REFINE_DEPTH_FRACTION = 0.25  # E:30
POLE_LAT_LIMIT_DEG = 85.0


_FAST_LIB_PATH = _HERE / "libd360_oracle_fast.so"
_timing_build = False


def build(force: bool = False) -> Path:
    """Compile the C restatement (gcc, seconds)."""
    src = _HERE / "d360_oracle.c"
    if force or not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-C", str(_HERE), "-B"], check=True, capture_output=True)
    return _LIB_PATH


def use_timing_build() -> Path:
    """bench.py's CPU arm only: switch this process to the -O3 -march=native build (compiled here, for
    this host; FMA contraction allowed like the reference's fastmath numba kernels).  Never used as
    the checker.  Always rebuilt: the library must match the CPU it runs on."""
    global _lib, _timing_build
    subprocess.run(["make", "-C", str(_HERE), "-B", "fast"], check=True, capture_output=True)
    _timing_build, _lib = True, None
    return _FAST_LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if _timing_build:
            _lib = C.CDLL(str(_FAST_LIB_PATH))
        else:
            build()
            _lib = C.CDLL(str(_LIB_PATH))
        _lib.d360o_get_threads.restype = C.c_int
    return _lib


def set_threads(n: int) -> None:
    lib().d360o_set_threads(C.c_int(int(n)))


def get_threads() -> int:
    return int(lib().d360o_get_threads())


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _u8(a):
    return np.ascontiguousarray(a).astype(np.uint8, copy=False)


# --------------------------------------------------------------------------------------
# Host-side geometry restated with numpy exactly as the reference writes it.
# --------------------------------------------------------------------------------------

def camera_tables(width: int, height: int):
    """Row/column trig tables of G:81-86 (float64)."""
    xs = np.arange(width, dtype=np.float64)
    ys = np.arange(height, dtype=np.float64)
    lam = (2.0 * np.pi) * ((xs + 0.5) / width) - np.pi
    phi = np.pi / 2.0 - np.pi * ((ys + 0.5) / height)
    return np.sin(lam), np.cos(lam), np.sin(phi), np.cos(phi)


def camera_rays64(width: int, height: int) -> np.ndarray:
    """G:117-122 → (H, W, 3) float64."""
    sl, cl, sp, cp = camera_tables(width, height)
    out = np.empty((height, width, 3), np.float64)
    out[..., 0] = cp[:, None] * sl[None, :]
    out[..., 1] = -sp[:, None]
    out[..., 2] = cp[:, None] * cl[None, :]
    return out


def relative_transform(r_src, t_src, r_dst, t_dst):
    """G:182-188: x_dst = R x_src + t with poses camera→world."""
    r_src, t_src, r_dst, t_dst = map(_f64, (r_src, t_src, r_dst, t_dst))
    rt = r_dst.T
    return rt @ r_src, rt @ t_src + (-rt @ t_dst)


def sample_offsets(half_window: int = 5, sample_stride: int = 2) -> np.ndarray:
    """E:60-65, dy outer / dx inner, rows are (dx, dy)."""
    reach = (half_window // sample_stride) * sample_stride
    steps = np.arange(-reach, reach + 1, sample_stride, dtype=np.int32)
    return np.array([(dx, dy) for dy in steps for dx in steps], dtype=np.int32)


def to_gray(image: np.ndarray) -> np.ndarray:
    """keyframes.py:64-72."""
    img = np.asarray(image)
    if img.ndim == 2:
        return img.astype(np.float32) / np.float32(255.0)
    h, w = img.shape[:2]
    out = np.empty((h, w), np.float32)
    lib().d360o_to_gray_rgb(_p(np.ascontiguousarray(img, np.uint8)), _p(out), h, w)
    return out


def refinement_draw_tables(seed: int, iterations: int, depth_range, theta_deg=DEFAULT_REFINE_THETA_DEG,
                           depth_fraction=DEFAULT_REFINE_DEPTH_FRACTION):
    """E:495-526 / E:558-561 (NumPy PCG64 scalar draws, shared by all pixels)."""
    dmin, dmax = depth_range
    delta_d = depth_fraction * (dmax - dmin)
    theta = math.radians(theta_deg)
    rng = np.random.default_rng(seed)
    tables = []
    for _ in range(iterations):
        dd = np.empty(REFINE_CANDIDATES, np.float64)
        ang = np.empty(REFINE_CANDIDATES, np.float64)
        az = np.empty(REFINE_CANDIDATES, np.float64)
        for i in range(REFINE_CANDIDATES):
            scale = 0.5**i
            dd[i] = rng.uniform(-1.0, 1.0) * delta_d * scale
            ang[i] = rng.uniform(0.0, 1.0) * theta * scale
            az[i] = rng.uniform(0.0, 2.0 * math.pi)
        tables.append((dd.astype(np.float32), np.sin(ang).astype(np.float32),
                       np.cos(ang).astype(np.float32), np.cos(az).astype(np.float32),
                       np.sin(az).astype(np.float32)))
    return tables


class Group:
    """Plain-array stereo group in the kernel layout of E:137-156, V views."""

    def __init__(self, ref_image, nb_images, ref_pose, nb_poses, half_window=5, sample_stride=2,
                 trunc=1.2, top_k=None):
        self.ref_gray = to_gray(ref_image)
        self.h, self.w = self.ref_gray.shape
        self.nb = np.stack([to_gray(im) for im in nb_images])
        self.n_views = len(nb_images)
        self.rays64 = camera_rays64(self.w, self.h)
        self.rays = self.rays64.astype(np.float32)
        rel = [relative_transform(ref_pose[0], ref_pose[1], p[0], p[1]) for p in nb_poses]
        self.rel_r = np.stack([r for r, _ in rel]).astype(np.float32)
        self.rel_t = np.stack([t for _, t in rel]).astype(np.float32)
        self.offsets = sample_offsets(half_window, sample_stride)
        self.trunc = float(trunc)
        self.top_k = default_top_k(self.n_views) if top_k is None else int(top_k)


def default_top_k(n_views: int) -> int:
    """V<=2: all views (the reference's mean, K:297); V>2: best half."""
    return n_views if n_views <= 2 else max(2, n_views // 2)


# --------------------------------------------------------------------------------------
# Kernels
# --------------------------------------------------------------------------------------

def _group_args(g: Group):
    return (_p(g.rays), _p(g.ref_gray), _p(g.nb), C.c_int(g.n_views), _p(g.rel_r), _p(g.rel_t),
            _p(g.offsets), C.c_int(len(g.offsets)), C.c_int(g.h), C.c_int(g.w),
            C.c_double(g.trunc), C.c_int(g.top_k))


def eval_costs(g: Group, depth, normal) -> np.ndarray:
    depth, normal = _f32(depth), _f32(normal)
    cost = np.empty((g.h, g.w), np.float32)
    rc = lib().d360o_eval_costs(_p(depth), _p(normal), _p(cost), *_group_args(g))
    assert rc == 0
    return cost


def red_black_pass(g: Group, parity: int, depth, normal, cost):
    """Returns (depth, normal, cost, n_evals); inputs untouched (pre-copy of E:575-577 here)."""
    depth, normal, cost = _f32(depth), _f32(normal), _f32(cost)
    od, on, oc = depth.copy(), normal.copy(), cost.copy()
    n = C.c_int64(0)
    rc = lib().d360o_red_black_pass(C.c_int(parity), _p(depth), _p(normal), _p(cost), _p(od), _p(on),
                                    _p(oc), *_group_args(g), C.byref(n))
    assert rc == 0
    return od, on, oc, int(n.value)


def refine_pass(g: Group, depth, normal, cost, table, depth_range):
    """Returns new (depth, normal, cost); K:476-610."""
    d, n, c = _f32(depth).copy(), _f32(normal).copy(), _f32(cost).copy()
    dd, sa, ca, caz, saz = (_f32(t) for t in table)
    rc = lib().d360o_refine_pass(_p(d), _p(n), _p(c), _p(dd), _p(sa), _p(ca), _p(caz), _p(saz),
                                 C.c_int(len(dd)), C.c_double(depth_range[0]),
                                 C.c_double(depth_range[1]), *_group_args(g))
    assert rc == 0
    return d, n, c


def median_support_mask(depth, valid, half: int, rel_threshold: float) -> np.ndarray:
    depth = _f32(depth)
    v = _u8(valid)
    h, w = depth.shape
    out = np.zeros((h, w), np.uint8)
    lib().d360o_median_support_mask(_p(depth), _p(v), C.c_int(half), C.c_double(rel_threshold),
                                    _p(out), C.c_int(h), C.c_int(w))
    return out.astype(bool)


def random_init(depth, normal, cost, valid, depth_range, seed: int):
    """E:244-283 with NumPy PCG64 draws; returns new (depth, normal, cost, valid)."""
    h, w = depth.shape
    dmin, dmax = float(depth_range[0]), float(depth_range[1])
    rng = np.random.default_rng(seed)
    inv = rng.uniform(1.0 / dmax, 1.0 / dmin, size=(h, w))
    g = rng.standard_normal((h, w, 3))
    return random_init_apply(depth, normal, cost, valid, inv, g)


def random_init_apply(depth, normal, cost, valid, inv, g):
    h, w = depth.shape
    d, n, c = _f32(depth).copy(), _f32(normal).copy(), _f32(cost).copy()
    v = _u8(valid).copy()
    rays64 = camera_rays64(w, h)
    lib().d360o_random_init_apply(_p(_f64(inv)), _p(_f64(g)), _p(rays64), _p(d), _p(n), _p(c), _p(v),
                                  C.c_int(h), C.c_int(w))
    return d, n, c, v.astype(bool)


def warp_plane_map(depth, normal, cost, valid, pose_prev, pose_cur, depth_range):
    """E:286-355; poses are (R, t) camera→world."""
    h, w = depth.shape
    r_rel, t_rel = relative_transform(pose_prev[0], pose_prev[1], pose_cur[0], pose_cur[1])
    od = np.zeros((h, w), np.float32)
    on = np.zeros((h, w, 3), np.float32)
    oc = np.full((h, w), np.inf, np.float32)
    ov = np.zeros((h, w), np.uint8)
    rays64 = camera_rays64(w, h)
    lib().d360o_warp_plane_map(_p(_f32(depth)), _p(_f32(normal)), _p(_f32(cost)), _p(_u8(valid)),
                               _p(rays64), _p(_f64(r_rel)), _p(_f64(t_rel)),
                               C.c_double(depth_range[0]), C.c_double(depth_range[1]), _p(od), _p(on),
                               _p(oc), _p(ov), C.c_int(h), C.c_int(w))
    return od, on, oc, ov.astype(bool)


def consistency_filter(depth, valid, pose, window, min_support=2, rel_tol=0.01) -> np.ndarray:
    """P:246-281.  window: list of (depth, valid, (R, t)).  Returns the surviving mask."""
    h, w = depth.shape
    wd = _f32(np.stack([f[0] for f in window]))
    wv = _u8(np.stack([f[1] for f in window]))
    wr = _f64(np.stack([np.asarray(f[2][0]).reshape(9) for f in window]))
    wt = _f64(np.stack([f[2][1] for f in window]))
    out = np.zeros((h, w), np.uint8)
    lib().d360o_consistency_filter(_p(_f32(depth)), _p(_u8(valid)), _p(_f64(pose[0]).reshape(9)),
                                   _p(_f64(pose[1])), _p(wd), _p(wv), _p(wr), _p(wt),
                                   C.c_int(len(window)), _p(camera_rays64(w, h)),
                                   C.c_int(min_support), C.c_double(rel_tol), _p(out), C.c_int(h),
                                   C.c_int(w))
    return out.astype(bool)


def fuse_oldest(depth, valid, pose, image, newer, reproj_px=1.0, rel_tol=0.01):
    """P:310-348.  newer: list of (depth, valid, (R, t)).  Returns (points f64, colors u8)."""
    h, w = depth.shape
    n_new = len(newer)
    if n_new:
        nd = _f32(np.stack([f[0] for f in newer]))
        nv = _u8(np.stack([f[1] for f in newer]))
        nr = _f64(np.stack([np.asarray(f[2][0]).reshape(9) for f in newer]))
        nt = _f64(np.stack([f[2][1] for f in newer]))
    else:
        nd = np.zeros((1, h, w), np.float32)
        nv = np.zeros((1, h, w), np.uint8)
        nr = np.zeros((1, 9))
        nt = np.zeros((1, 3))
    img = np.asarray(image)
    if img.ndim == 2:
        img = np.repeat(img[..., None], 3, axis=2)
    pts = np.empty((h * w, 3), np.float64)
    col = np.empty((h * w, 3), np.uint8)
    n = C.c_int64(0)
    lib().d360o_fuse_oldest(_p(_f32(depth)), _p(_u8(valid)), _p(_f64(pose[0]).reshape(9)),
                            _p(_f64(pose[1])), _p(np.ascontiguousarray(img, np.uint8)), _p(nd), _p(nv),
                            _p(nr), _p(nt), C.c_int(n_new), _p(camera_rays64(w, h)),
                            C.c_double(reproj_px), C.c_double(rel_tol), _p(pts), _p(col), C.byref(n),
                            C.c_int(h), C.c_int(w))
    k = int(n.value)
    return pts[:k].copy(), col[:k].copy()


def philox4x32_10(ctr, key) -> np.ndarray:
    c = np.asarray(ctr, np.uint32)
    k = np.asarray(key, np.uint32)
    out = np.zeros(4, np.uint32)
    lib().d360o_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def pole_rows(height: int) -> np.ndarray:
    """P:214 with G:125-128."""
    ys = np.arange(height, dtype=np.float64) + 0.5
    lat = np.pi / 2.0 - np.pi * (ys / height)
    return np.abs(np.degrees(lat)) > POLE_LAT_LIMIT_DEG


def run_patchmatch(g: Group, depth, normal, depth_range, iterations: int, seed: int,
                   trace: list | None = None):
    """E:529-631 on plain arrays.  Returns (depth, normal, cost, valid_pano).

    ``trace`` (optional list) receives a copy of (depth, normal, cost) after the initial
    evaluation and after every pass, for per-iteration parity checks.
    """
    tables = refinement_draw_tables(seed, iterations, depth_range)
    d, n = _f32(depth).copy(), _f32(normal).copy()
    c = eval_costs(g, d, n)
    if trace is not None:
        trace.append(("eval", d.copy(), n.copy(), c.copy()))
    for it in range(iterations):
        for parity in (0, 1):
            d, n, c, _ = red_black_pass(g, parity, d, n, c)
            if trace is not None:
                trace.append((f"rb{it}.{parity}", d.copy(), n.copy(), c.copy()))
        d, n, c = refine_pass(g, d, n, c, tables[it], depth_range)
        if trace is not None:
            trace.append((f"refine{it}", d.copy(), n.copy(), c.copy()))
    return d, n, c, c < np.float32(g.trunc)  # E:629 on the f32-stored cost


def depth_stage(g: Group, ref_id: int, depth_range, iterations: int, seed: int, prev=None,
                ref_pose=None, median_window=5, median_rel_threshold=0.2):
    """warp-or-random init → run_patchmatch → median → pole mask."""
    h, w = g.h, g.w
    d = np.zeros((h, w), np.float32)
    n = np.zeros((h, w, 3), np.float32)
    c = np.full((h, w), np.inf, np.float32)
    v = np.zeros((h, w), bool)
    if prev is not None:
        pd, pn, pc, pv, ppose = prev
        d, n, c, v = warp_plane_map(pd, pn, pc, pv, ppose, ref_pose, depth_range)
    d, n, c, v = random_init(d, n, c, v, depth_range, seed + ref_id)
    d, n, c, valid = run_patchmatch(g, d, n, depth_range, iterations, seed + ref_id)
    plane = (d, n, c, np.ones((h, w), bool))
    valid = median_support_mask(d, valid, median_window // 2, median_rel_threshold)
    valid[pole_rows(h), :] = False
    return plane, d, valid
