"""Timing of the f3 / f4 kernels at C3 size next to a numpy restatement of the reference's
statements (outputs.py:43-51, 84-87; metrics.py:31-45, 66-77) on the host — not the benchmark."""
import sys, os, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, torch
import paper_2211_16266_b200 as p
from paper_2211_16266_b200 import engine, metrics, outputs, _lib

_lib.load()
W, H = 1920, 960
n = W * H
rng = np.random.default_rng(0)
pts = rng.normal(size=(n, 3)) * 3.0
cols = rng.integers(0, 256, size=(n, 3), dtype=np.uint8)
depth = rng.uniform(0.5, 16.0, size=(H, W)).astype(np.float32)
valid = rng.uniform(size=(H, W)) > 0.2
dev = torch.device("cuda")
d_pts, d_cols = torch.from_numpy(pts).to(dev), torch.from_numpy(cols).to(dev)
cam = p.EquirectCamera(W, H)
d_pano = engine.DeviceDepthPanorama.from_host(engine.DepthPanorama(cam, depth, valid), dev)
d_gt = engine.DeviceDepthPanorama.from_host(engine.DepthPanorama(cam, depth * 1.01, valid), dev)
pose = p.RigidPose(np.eye(3), np.zeros(3))


def gpu_ms(fn, reps=20):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def cpu_ms(fn, reps=3):
    fn()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t) / reps * 1e3


def np_pack():
    rec = np.empty(n, outputs.PLY_DTYPE)
    f = pts.astype(np.float32)
    rec["x"], rec["y"], rec["z"] = f[:, 0], f[:, 1], f[:, 2]
    rec["red"], rec["green"], rec["blue"] = cols[:, 0], cols[:, 1], cols[:, 2]
    return rec.tobytes()


def np_mm():
    mm = np.clip(np.rint(depth.astype(np.float64) * 1000.0), 0, 65535).astype(np.uint16)
    mm[~valid] = 0
    return mm


def np_comp():
    h, w = 360, 720
    local = (pts - pose.translation) @ pose.rotation
    r = np.linalg.norm(local, axis=1)
    keep = r > 1e-12
    local, rr = local[keep], r[keep]
    lon = np.arctan2(local[:, 0], local[:, 2])
    u = (lon + np.pi) * (w / (2.0 * np.pi)) - 0.5
    v = np.arccos(np.clip(-local[:, 1] / rr, -1.0, 1.0)) * (h / np.pi) - 0.5
    raster = np.zeros((h, w), bool)
    raster[np.clip(np.rint(v).astype(np.int64), 0, h - 1), np.rint(u).astype(np.int64) % w] = True
    return raster.mean()


def np_acc():
    joint = valid
    pr, gt = depth[joint].astype(np.float64), (depth * 1.01)[joint].astype(np.float64)
    rel = np.abs(pr - gt) / gt
    return rel.mean(), np.sqrt(np.mean((pr - gt) ** 2)), (rel <= 0.02).mean()


rows = [("pack_ply_records", lambda: outputs.pack_ply_records_device(d_pts, d_cols), n * (24 + 3 + 15), np_pack),
        ("depth_to_mm16", lambda: outputs.depth_to_mm16_device(d_pano), n * (4 + 1 + 2), np_mm),
        ("completeness (1 pose, 720x360)", lambda: metrics.completeness(d_pts, [pose]), n * 24, np_comp),
        ("depth_accuracy", lambda: metrics.accuracy(d_pano, d_gt), n * 10, np_acc)]
for name, g, nbytes, c in rows:
    gm, cm = gpu_ms(g), cpu_ms(c)
    _lib.trace_enable(True)
    g(); torch.cuda.synchronize()
    tr = _lib.trace_summary()
    _lib.trace_enable(False)
    km = sum(ms for _, ms in tr.values())
    print(f"{name:32s} kernels {km:7.4f} ms ({nbytes / km / 1e6:7.1f} GB/s algorithmic), call incl. host wrapper "
          f"{gm:7.3f} ms   numpy on host {cm:8.1f} ms   {tr}")
