"""SHA-256 of the depth / normal / cost maps of the benchmark's warp-initialised chain (C3 by default),
one line per keyframe: the bit-identity check between builds of the library (D360_LIB_PATH)."""
import hashlib, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, torch
import paper_2211_16266_b200 as p
from paper_2211_16266_b200 import engine, pipeline, synth
import bench

W, H, V, hw, stride, iters = bench.WORKLOADS[os.environ.get("WORKLOAD", "c3")]
dev = torch.device("cuda", 0)
cam = p.EquirectCamera(W, H)
spec = engine.PatchSpec(hw, stride, 1.2)
scene = synth.default_scene("box")
poses = [p.RigidPose(np.eye(3), t) for t in bench.sequence_positions(0)]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
nb_order = []
for k in range(1, V // 2 + 1):
    nb_order += [-k, k]
order = bench.walk(n)
need = sorted({i + o for i in order for o in [0] + nb_order})
imgs = {k: synth.render_scene_device(scene, cam, poses[k], dev)[0] for k in need}
kfs = {k: p.Keyframe(id=k, image=imgs[k].cpu().numpy(), pose=poses[k]) for k in need}
stage = pipeline.DepthStage(cam, spec, bench.DEPTH_RANGE, iters, 0, warp=True, precision="mixed", init_rng="philox",
                            device=dev)
save = os.environ.get("SAVE")
for step, i in enumerate(order):
    g = p.StereoGroup(reference=kfs[i], neighbors=tuple(kfs[i + o] for o in nb_order), camera=cam)
    prep = engine.PreparedGroup(g, spec, precision="mixed", device=dev)
    res = stage.process_device(prep)
    pm = stage._prev[0] if isinstance(stage._prev, tuple) else stage._prev
    arrs = [pm.depth.cpu().numpy(), pm.normal.cpu().numpy(), pm.cost.cpu().numpy()]
    print(step, " ".join(hashlib.sha256(a.tobytes()).hexdigest()[:16] for a in arrs), flush=True)
    if save:
        np.savez(f"{save}_{step}.npz", depth=arrs[0], normal=arrs[1], cost=arrs[2])
