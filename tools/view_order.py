"""Experiment: which view should refine_pass leave for its second pass?  The V-1 lower bound (DESIGN.md
section 4.4) holds for any V-1 views, and the per-view costs and their sorted aggregate do not depend on the
order of the neighbours, so the order only changes how many evaluations are decided early.
python tools/view_order.py "-1,1,-2,2" [n_keyframes]  ->  ms per keyframe, evaluations, early cuts."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, torch
import paper_2211_16266_b200 as p
from paper_2211_16266_b200 import engine, pipeline, synth, _lib
import bench

W, H, V, hw, stride, iters = bench.WORKLOADS["c3"]
dev = torch.device("cuda", 0)
cam = p.EquirectCamera(W, H)
spec = engine.PatchSpec(hw, stride, 1.2)
scene = synth.default_scene("box")
poses = [p.RigidPose(np.eye(3), t) for t in bench.sequence_positions(0)]
nb_order = [int(x) for x in sys.argv[1].split(",")]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
order = bench.walk(n)
need = sorted({i + o for i in order for o in [0] + nb_order})
imgs = {k: synth.render_scene_device(scene, cam, poses[k], dev)[0] for k in need}
kfs = {k: p.Keyframe(id=k, image=imgs[k].cpu().numpy(), pose=poses[k]) for k in need}
stage = pipeline.DepthStage(cam, spec, bench.DEPTH_RANGE, iters, 0, warp=True, precision="mixed", init_rng="philox",
                            device=dev, count_evals=True)
import hashlib
h = hashlib.sha256()
for step, i in enumerate(order):
    g = p.StereoGroup(reference=kfs[i], neighbors=tuple(kfs[i + o] for o in nb_order), camera=cam)
    prep = engine.PreparedGroup(g, spec, precision="mixed", device=dev)
    if step == 2:
        torch.cuda.synchronize(); stage.workspace.n_evals.zero_()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True); e0.record()
    res = stage.process_device(prep)
    h.update(res.pano.depth.cpu().numpy().tobytes())
e1.record(); torch.cuda.synchronize()
ev, cut = (int(x) for x in stage.workspace.n_evals.tolist())
print(f"order {nb_order}: {e0.elapsed_time(e1) / (n - 2):.2f} ms/keyframe, evals {ev / (n - 2) / 1e6:.2f} M, "
      f"cut {cut / (n - 2) / 1e6:.2f} M, depth hash {h.hexdigest()[:16]}")
