"""Why the projection runs on the FP64 pipe: the same CPU restatement compiled
twice - as the checker is (f64 after lam = num / dn, K:244-251) and with every projection operation in
float32 (-DD360O_F32_PROJECTION, an experiment build that never serves as the checker) - evaluates one
full-size C3 keyframe (1920x960, near-ground-truth hypotheses, the regime of converged maps) and the
costs are compared under the parity gate |dc| <= 1e-4 c + 1e-7.  CPU only:
    python tools/f32_projection.py [width] > profiles/f32_projection_r2.txt"""
import ctypes as C, importlib.util, os, subprocess, sys, tempfile
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np
import bench
from oracle import d360_oracle as O


def main():
    W = int(sys.argv[1]) if len(sys.argv) > 1 else 1920
    H = W // 2
    V = int(os.environ.get("VIEWS", "4"))
    O.build()
    tmp = Path(tempfile.mkdtemp())
    f32_lib = tmp / "libd360_oracle_f32proj.so"
    subprocess.run(["gcc", "-O2", "-fPIC", "-ffp-contract=off", "-fno-fast-math", "-std=gnu11", "-DD360O_F32_PROJECTION",
                    "-shared", "-o", str(f32_lib), str(ROOT / "oracle" / "d360_oracle.c"), "-lm", "-lpthread"], check=True)
    spec = importlib.util.spec_from_file_location("d360_oracle_f32proj", ROOT / "oracle" / "d360_oracle.py")
    O32 = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(O32)
    O32._lib = C.CDLL(str(f32_lib))
    O32._lib.d360o_get_threads.restype = C.c_int

    nb_order = []
    for k in range(1, V // 2 + 1):
        nb_order += [-k, k]
    i = 11
    idx = sorted({i + o for o in [0] + nb_order})
    imgs, how = bench.render_cpu_inputs(W, H, idx)
    pos = bench.sequence_positions(0)
    eye = np.eye(3)
    # ground-truth depth of the 4 x 3 x 5 m box from pos[i] (ray / axis-aligned slab intersection)
    ys, xs = np.mgrid[0:H, 0:W]
    lam = 2 * np.pi * (xs + 0.5) / W - np.pi
    phi = np.pi / 2 - np.pi * (ys + 0.5) / H
    rays = np.stack([np.cos(phi) * np.sin(lam), -np.sin(phi), np.cos(phi) * np.cos(lam)], -1)
    half = np.array([2.0, 1.5, 2.5])
    with np.errstate(divide="ignore", invalid="ignore"):
        tt = np.where(rays > 0, (half - pos[i]) / rays, (-half - pos[i]) / rays)
    gt = tt.min(-1)
    rng = np.random.default_rng(0)
    n = -rays + rng.normal(0, 0.15, rays.shape)
    n = (n / np.linalg.norm(n, axis=-1, keepdims=True)).astype(np.float32)
    d = (gt * (1 + rng.normal(0, 0.01, gt.shape))).astype(np.float32)
    res = {}
    for name, mod in (("f64 projection (the checker)", O), ("f32 projection (experiment build)", O32)):
        g = mod.Group(imgs[i], [imgs[i + o] for o in nb_order], (eye, pos[i]), [(eye, pos[i + o]) for o in nb_order], 5, 2, 1.2)
        res[name] = mod.eval_costs(g, d, n).astype(np.float64)
    a, b = res.values()
    rel = np.abs(a - b) / np.maximum(a, 1e-12)
    inside = np.abs(a - b) <= 1e-4 * a + 1e-7
    low = a < 0.05
    print(f"{W}x{H}, {V} neighbour views, 25 samples, frames by {how}; near-ground-truth hypotheses on every pixel")
    print(f"median cost {np.median(a):.4f}; pixels with cost < 0.05: {low.mean():.3f}")
    print(f"relative cost difference f32-projection vs f64-projection: p50 {np.percentile(rel, 50):.2e}  p90 {np.percentile(rel, 90):.2e}  "
          f"p99 {np.percentile(rel, 99):.2e}  max {rel.max():.2e}")
    print(f"inside the parity gate |dc| <= 1e-4 c + 1e-7: {inside.mean():.4f} of all pixels, {inside[low].mean():.4f} of the low-cost pixels")
    print(f"north_star asks for every per-iteration cost within 1e-4 relative: an all-f32 projection leaves {1 - inside.mean():.1%} of the pixels outside.")


if __name__ == "__main__":  # render_cpu_inputs spawns worker processes that re-import this file
    main()
