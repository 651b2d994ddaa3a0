"""Experiment: potential of an approximate reject-filter in refine_pass (needs a -DD360_REFINE_STATS build,
D360_LIB_PATH=tools/variants/libd360_stats.so).  Runs the benchmark's warp-initialised chain."""
import ctypes, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, torch
import paper_2211_16266_b200 as p
from paper_2211_16266_b200 import _lib, engine, pipeline, synth
import bench

W, H, V, hw, stride, iters = bench.WORKLOADS["c3"]
dev = torch.device("cuda", 0)
cam = p.EquirectCamera(W, H)
spec = engine.PatchSpec(hw, stride, 1.2)
scene = synth.default_scene("box")
poses = [p.RigidPose(np.eye(3), t) for t in bench.sequence_positions(0)]
imgs = [synth.render_scene_device(scene, cam, pose, dev)[0] for pose in poses]
kfs = [p.Keyframe(id=k, image=imgs[k].cpu().numpy(), pose=poses[k]) for k in range(len(poses))]
nb_order = [-1, 1, -2, 2]
stage = pipeline.DepthStage(cam, spec, bench.DEPTH_RANGE, iters, 0, warp=True, precision="mixed", init_rng="philox",
                            device=dev, count_evals=True)
lib = _lib.load()
out = (ctypes.c_ulonglong * 96)()
n = int(os.environ.get("N", "6"))
for step, i in enumerate(bench.walk(n)):
    g = p.StereoGroup(reference=kfs[i], neighbors=tuple(kfs[i + o] for o in nb_order), camera=cam)
    prep = engine.PreparedGroup(g, spec, precision="mixed", device=dev)
    stage.process_device(prep)
    torch.cuda.synchronize()
    lib.d360_debug_refine_stats(out, 1)
    s = list(out)
    tot = max(s[0], 1)
    print(f"step {step}: evals {s[0]}  accepted {s[1]/tot:.4f}  not-cut-by-3-views {s[2]/tot:.4f}  unresolved@delta[0,1e-5,3e-5,1e-4,3e-4] "
          + " ".join(f"{x/tot:.4f}" for x in s[3:8]))
    for k in range(6):
        print(f"   k={k}: unresolved@delta[0,1e-5,3e-5,1e-4,3e-4]", " ".join(f"{s[32+5*k+i]/max(s[8+k],1):.4f}" for i in range(5)))
    print("   bound hist [<.01,.02,.05,.1,.2,.5,1,inf]:", " ".join(f"{x/tot:.3f}" for x in s[64:72]))
    print("   min-sigma hist [<1e-3,2e-3,5e-3,1e-2,2e-2,5e-2,1e-1,inf]:", " ".join(f"{x/tot:.3f}" for x in s[72:80]))
    print("   per-candidate accept rate:", " ".join(f"{s[16+k]/max(s[8+k],1):.4f}" for k in range(6)), flush=True)
