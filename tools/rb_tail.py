"""Per-iteration cost of the propagation on a steady-state keyframe of the benchmark chain: evaluations and
CUDA-event time of the red-black launch of every iteration (differences between runs of 1..6 iterations from the
same warp-initialised start).  python tools/rb_tail.py"""
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
nb_order = [-1, 1, -2, 2]
order = bench.walk(3)
need = sorted({i + o for i in order for o in [0] + nb_order})
kfs = {k: p.Keyframe(id=k, image=synth.render_scene_device(scene, cam, poses[k], dev)[0].cpu().numpy(), pose=poses[k]) for k in need}
stage = pipeline.DepthStage(cam, spec, bench.DEPTH_RANGE, iters, 0, warp=True, precision="mixed", init_rng="philox", device=dev)
for i in order[:2]:
    g = p.StereoGroup(reference=kfs[i], neighbors=tuple(kfs[i + o] for o in nb_order), camera=cam)
    stage.process_device(engine.PreparedGroup(g, spec, precision="mixed", device=dev))
i = order[2]
g = p.StereoGroup(reference=kfs[i], neighbors=tuple(kfs[i + o] for o in nb_order), camera=cam)
prep = engine.PreparedGroup(g, spec, precision="mixed", device=dev)
prev_map, prev_pose = stage._prev
init = engine.warp_plane_map_device(prev_map, prev_pose, kfs[i].pose, cam)
init = engine.random_init_device(init, bench.DEPTH_RANGE, i, "philox")
ws = engine.PatchMatchWorkspace(cam, dev)
res = []
for k in range(1, iters + 1):
    for rep in range(2):
        pm = init.clone()
        ws.n_evals.zero_()
        _lib.trace_enable(True)
        engine.run_patchmatch_device(prep, pm, k, i, workspace=ws, count_evals=True, check_valid=False)
        torch.cuda.synchronize()
        tr = _lib.trace_summary()
        _lib.trace_enable(False)
    ev, cut = (int(x) for x in ws.n_evals.tolist())
    res.append((k, ev - 6 * W * H * k, tr["red_black"][1], tr["refine"][1], cut))
prev = (0, 0, 0.0, 0.0, 0)
print("iteration  rb_evals(M)  rb_ms  us_per_1000_evals  refine_ms  refine_cut_share")
for r in res:
    de, dt, dr, dc = r[1] - prev[1], r[2] - prev[2], r[3] - prev[3], r[4] - prev[4]
    print(f"{r[0]:9d} {de / 1e6:11.3f} {dt:6.3f} {1e3 * dt / (de / 1e3):18.3f} {dr:10.3f} {dc / (6 * W * H):17.3f}")
    prev = r
