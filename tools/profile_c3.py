"""One C3-sized PatchMatch iteration for ncu captures (not a benchmark)."""
import sys
sys.path.insert(0, '/root/repo')
import torch
import paper_2211_16266_b200 as p
from paper_2211_16266_b200 import engine, synth
prec = sys.argv[1] if len(sys.argv) > 1 else "mixed"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cam = p.EquirectCamera(1920, 960)
group, gt = synth.make_group(synth.default_scene("box"), cam, n_views=4)
prep = engine.prepare_group(group, engine.PatchSpec(), precision=prec)
dr = (0.5, 16.0)
pm = engine.DevicePlaneMap.empty(cam, dr)
engine.random_init_device(pm, dr, 0, "philox")
engine.run_patchmatch_device(prep, pm, iters, 0, check_valid=False)
torch.cuda.synchronize()
