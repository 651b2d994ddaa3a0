"""Debug: fast (mixed) vs literal (exact) eval_costs on a golden scene; where do they differ?"""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, torch
import paper_2211_16266_b200 as p
from paper_2211_16266_b200 import engine
from paper_2211_16266_b200.engine import PatchSpec
name = sys.argv[1] if len(sys.argv) > 1 else "hot_256x128_c1"
z = np.load(f"tests/golden/{name}.npz")
cam = p.EquirectCamera(z["images"].shape[2], z["images"].shape[1])
kfs = [p.Keyframe(id=k, image=z["images"][k], pose=p.RigidPose(z["rotations"][k], z["translations"][k])) for k in range(3)]
spec = PatchSpec(int(z["half_window"]), int(z["sample_stride"]), float(z["trunc"]))
group = p.StereoGroup(reference=kfs[1], neighbors=(kfs[0], kfs[2]), camera=cam)
out = {}
for prec in ("mixed", "exact"):
    prep = engine.prepare_group(group, spec, precision=prec)
    pm = engine.DevicePlaneMap.from_host(engine.PlaneMap(cam, z["init_depth"], z["init_normal"], np.full(cam.shape, np.inf, np.float32), np.ones(cam.shape, bool), tuple(z["depth_range"])))
    engine.evaluate_costs_device(prep, pm)
    out[prec] = pm.cost.cpu().numpy()
d = np.abs(out["mixed"] - out["exact"])
tol = 1e-4 * np.abs(out["exact"]) + 1e-7
bad = d > tol
print("bad pixels", bad.sum(), "of", bad.size, "max", d.max())
ys, xs = np.nonzero(bad)
print("rows hist", np.bincount(ys // 8)[:40]); print("per-row", np.bincount(ys, minlength=128)[:12], np.bincount(ys, minlength=128)[-12:])
print("cols hist", np.bincount(xs // 16)[:40])
for y, x in list(zip(ys, xs))[:12]:
    print(y, x, out["mixed"][y, x], out["exact"][y, x])
