"""Run every BASELINE.json config once (functional check + timing; not the benchmark)."""
import sys, os, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, torch
import paper_2211_16266_b200 as p
from paper_2211_16266_b200 import engine, synth, _lib

CONFIGS = {"c1": (256, 128, 2, 5, 2, 3, "box"), "c2": (960, 480, 4, 3, 1, 6, "box"), "c3": (1920, 960, 4, 5, 2, 6, "box"),
           "c4": (3840, 1920, 6, 5, 2, 6, "corridor"), "c4s1": (3840, 1920, 6, 5, 1, 1, "corridor"),
           "quality": (5760, 2880, 4, 5, 2, 6, "box")}  # the paper's quality-mode resolution: planes > 2^23 texels
for name in sys.argv[1:] or list(CONFIGS):
    W, H, V, hw, st, it, kind = CONFIGS[name]
    cam = p.EquirectCamera(W, H)
    group, gt = synth.make_group(synth.default_scene(kind), cam, n_views=V)
    spec = engine.PatchSpec(hw, st, 1.2)
    prep = engine.prepare_group(group, spec)
    dr = (0.5, 16.0)
    ws = engine.PatchMatchWorkspace(cam, prep.device)
    for rep in range(2):
        pm = engine.DevicePlaneMap.empty(cam, dr)
        engine.random_init_device(pm, dr, 0, "philox")
        ws.n_evals.zero_()
        _lib.trace_enable(True)
        pm, pano = engine.run_patchmatch_device(prep, pm, it, 0, workspace=ws, count_evals=True, check_valid=False)
        torch.cuda.synchronize()
        tr = _lib.trace_summary()
        _lib.trace_enable(False)
    gt_t = torch.from_numpy(gt).cuda()
    ok = (((pm.depth - gt_t).abs() / gt_t < 0.02) & (pano.valid > 0)).float().mean().item()
    tot = sum(ms for _, ms in tr.values())
    print(name, f"{W}x{H} V={V} S={len(prep.offsets)} I={it}: total {tot:.2f} ms",
          {k: round(ms / n, 3) for k, (n, ms) in tr.items() if k in ("red_black", "refine", "eval_costs")},
          "evals", ws.n_evals.tolist(), f"within2pct&valid {ok:.3f}", flush=True)
