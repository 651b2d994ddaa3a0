"""Time one C3-sized PatchMatch run (kernel-variant experiments; not the benchmark)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
import paper_2211_16266_b200 as p
from paper_2211_16266_b200 import engine, synth, _lib

cam = p.EquirectCamera(1920, 960)
group, gt = synth.make_group(synth.default_scene("box"), cam, n_views=int(os.environ.get("NV", "4")))
prep = engine.prepare_group(group, engine.PatchSpec(), precision="mixed")
dr = (0.5, 16.0)
ws = engine.PatchMatchWorkspace(cam, prep.device)
for rep in range(2):
    pm = engine.DevicePlaneMap.empty(cam, dr)
    engine.random_init_device(pm, dr, 0, "philox")
    ws.n_evals.zero_()
    _lib.trace_enable(True)
    engine.run_patchmatch_device(prep, pm, 6, 0, workspace=ws, count_evals=True, check_valid=False)
    torch.cuda.synchronize()
    tr = _lib.trace_summary()
    _lib.trace_enable(False)
gt_t = torch.from_numpy(gt).cuda()
ok = ((pm.depth - gt_t).abs() / gt_t < 0.02).float().mean().item()
tot = sum(ms for _, ms in tr.values())
print(os.environ.get("D360_LIB_PATH", "default"), "total ms %.2f" % tot,
      {k: round(ms / n, 3) for k, (n, ms) in tr.items() if k in ("red_black", "refine", "eval_costs")},
      "evals", ws.n_evals.tolist(), "within2pct %.4f" % ok, "cost sum %.6f" % pm.cost.double().sum().item())
