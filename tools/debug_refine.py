import sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, torch
import paper_2211_16266_b200 as p
from paper_2211_16266_b200 import engine
from oracle import d360_oracle as O
from conftest import golden_group, load_golden
from test_gpu_parity import make_group, host_map
for name in ("hot_64x32_ident", "hot_64x32_rot", "hot_256x128_c1"):
    z = load_golden(name)
    group, spec, cam = make_group(p, z)
    og = golden_group(O, z)
    names = [str(s) for s in z["step_names"]]
    dr = tuple(z["depth_range"])
    for prec in ("exact", "mixed"):
        prep = engine.prepare_group(group, spec, precision=prec)
        for i in range(1, len(names)):
            if not names[i].startswith("refine") or not names[i-1].startswith("rb"): continue
            src = engine.DevicePlaneMap.from_host(host_map(engine, cam, z, i - 1))
            prev = (z["step_depth"][i - 1], z["step_normal"][i - 1], z["step_cost"][i - 1])
            tab = tuple(z["tables"][int(names[i][6:])])
            engine.refine_pass_device(prep, src, tab, dr)
            od, on, oc = O.refine_pass(og, *prev, tab, dr)
            gd, gn, gc = src.depth.cpu().numpy(), src.normal.cpu().numpy(), src.cost.cpu().numpy()
            diff = (gd != od) | (gn != on).any(-1)
            e = np.abs(gc.astype(np.float64) - oc)
            rel = e / np.maximum(oc, 1e-12)
            print(name, prec, names[i], "hyp mismatch px", int(diff.sum()), "max abs", e.max(), "max rel(all)", rel.max(),
                  "max rel(same hyp)", rel[~diff].max() if (~diff).any() else None, "exact cost frac", (gc == oc).mean())
            ys, xs = np.nonzero(diff)
            for y, x in list(zip(ys, xs))[:4]:
                print("   px", x, y, "gpu d", gd[y, x], "orc d", od[y, x], "gpu c", gc[y, x], "orc c", oc[y, x], "prev c", prev[2][y, x])
