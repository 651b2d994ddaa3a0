import sys, time, json
sys.path.insert(0, '/root/repo')
import torch, numpy as np
import paper_2211_16266_b200 as p
from paper_2211_16266_b200 import engine, synth, _lib
lib=_lib.load()
print("fp32 peak TF", lib.d360_measure_fma_peak(0, 20000), "fp64 peak TF", lib.d360_measure_fma_peak(1, 20000))
cam = p.EquirectCamera(1920, 960)
scene = synth.default_scene("box")
t0=time.time(); group, gt = synth.make_group(scene, cam, n_views=4); print("render s", time.time()-t0)
spec = engine.PatchSpec(); dr=(0.5,16.0)
for prec in ("mixed","exact"):
    prep = engine.prepare_group(group, spec, precision=prec)
    ws = engine.PatchMatchWorkspace(cam, prep.device)
    for it in (1, 6):
        pm = engine.DevicePlaneMap.empty(cam, dr); engine.random_init_device(pm, dr, 0, "philox")
        torch.cuda.synchronize(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
        e0.record(); engine.run_patchmatch_device(prep, pm, it, 0, workspace=ws, count_evals=True, check_valid=False); e1.record(); torch.cuda.synchronize()
        print(prec, "iters", it, "ms", e0.elapsed_time(e1), "evals", int(ws.n_evals.item()), flush=True)
    if prec=="exact": break
