"""Generate golden vectors from the REFERENCE implementation (build container only).

Runs /root/reference/pkg/src/densify360 (numba) on small synthetic scenes and stores
inputs + outputs of every hot-path function under tests/golden/*.npz.  The reference
cannot travel to the GPU box, these fixtures can.  Re-run:

    NUMBA_CACHE_DIR=/tmp/numba_cache python oracle/gen_golden.py

Nothing under tests/, bench.py or the package reads /root/reference at run time.
"""
import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
os.environ.setdefault("NUMBA_NUM_THREADS", "8")
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")

import numpy as np

from densify360 import engine, kernels, pipeline  # noqa: E402
from densify360.engine import PatchSpec, PlaneMap  # noqa: E402
from densify360.geometry import EquirectCamera, RigidPose, camera_rays  # noqa: E402
from densify360.keyframes import Keyframe, StereoGroup, to_gray  # noqa: E402
from densify360.synth import default_scene, render_scene  # noqa: E402

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"
OUT.mkdir(parents=True, exist_ok=True)
DEPTH_RANGE = (0.5, 16.0)


def rot(axis, deg):
    a = np.radians(deg)
    c, s = np.cos(a), np.sin(a)
    m = {0: [[1, 0, 0], [0, c, -s], [0, s, c]], 1: [[c, 0, s], [0, 1, 0], [-s, 0, c]],
         2: [[c, -s, 0], [s, c, 0], [0, 0, 1]]}[axis]
    return np.array(m, np.float64)


def make_frames(cam, poses, scene_kind="box"):
    scene = default_scene(scene_kind)
    frames, gts = [], []
    for k, pose in enumerate(poses):
        image, pano = render_scene(scene, cam, pose)
        frames.append(Keyframe(id=k, image=image, pose=pose))
        gts.append(pano.depth)
    return frames, gts


def pose_arrays(frames):
    return (np.stack([f.pose.rotation for f in frames]),
            np.stack([f.pose.translation for f in frames]))


def hot_path_case(name, width, iterations, poses, spec, seed, full_trace):
    """eval → (red, black, refine)*I with the state after every pass."""
    cam = EquirectCamera(width, width // 2)
    frames, gts = make_frames(cam, poses)
    group = StereoGroup(reference=frames[1], neighbors=(frames[0], frames[2]), camera=cam)
    prep = engine.prepare_group(group, spec)
    init = engine.random_init(PlaneMap.empty(cam, DEPTH_RANGE), DEPTH_RANGE, seed=seed)
    rng = np.random.default_rng(seed)
    tables = engine._refinement_draw_tables(
        rng, iterations, engine.DEFAULT_REFINE_DEPTH_FRACTION * (DEPTH_RANGE[1] - DEPTH_RANGE[0]),
        np.radians(engine.DEFAULT_REFINE_THETA_DEG))
    trunc = spec.cost_truncation
    out = {
        "images": np.stack([f.image for f in frames]),
        "rotations": pose_arrays(frames)[0], "translations": pose_arrays(frames)[1],
        "gt_depth": gts[1].astype(np.float32),
        "half_window": spec.half_window, "sample_stride": spec.sample_stride, "trunc": trunc,
        "depth_range": np.array(DEPTH_RANGE), "seed": seed, "iterations": iterations,
        "init_depth": init.depth, "init_normal": init.normal,
        "ref_gray": prep.ref_gray, "rays": prep.rays, "rel_r": prep.rel_r, "rel_t": prep.rel_t,
        "offsets": prep.offsets,
        "tables": np.stack([np.stack(t) for t in tables]),
    }
    cur = init.copy()
    engine._evaluate_all(prep, cur.depth, cur.normal, cur.cost)
    steps = [("eval", cur.copy())]
    nxt = cur.copy()
    for it in range(iterations):
        for parity in (0, 1):
            np.copyto(nxt.depth, cur.depth); np.copyto(nxt.normal, cur.normal); np.copyto(nxt.cost, cur.cost)
            kernels.red_black_pass(parity, kernels.NEIGHBOR_OFFSETS, cur.depth, cur.normal, cur.cost,
                                   nxt.depth, nxt.normal, nxt.cost, prep.rays, prep.ref_gray,
                                   prep.nb0, prep.nb1, prep.rel_r, prep.rel_t, prep.offsets, trunc)
            cur, nxt = nxt, cur
            steps.append((f"rb{it}.{parity}", cur.copy()))
        dd, sa, ca, caz, saz = tables[it]
        kernels.refine_pass(cur.depth, cur.normal, cur.cost, dd, sa, ca, caz, saz, DEPTH_RANGE[0],
                            DEPTH_RANGE[1], prep.rays, prep.ref_gray, prep.nb0, prep.nb1, prep.rel_r,
                            prep.rel_t, prep.offsets, trunc)
        steps.append((f"refine{it}", cur.copy()))
    # cross-check against the reference's own driver
    pm, pano = engine.run_patchmatch(group, init, spec, iterations=iterations, seed=seed, workers=8)
    assert np.array_equal(pm.depth, cur.depth) and np.array_equal(pm.cost, cur.cost)
    keep = steps if full_trace else [steps[0], steps[1], steps[2], steps[3], steps[-1]]
    out["step_names"] = np.array([s[0] for s in keep])
    out["step_depth"] = np.stack([s[1].depth for s in keep])
    out["step_normal"] = np.stack([s[1].normal for s in keep])
    out["step_cost"] = np.stack([s[1].cost for s in keep])
    out["pano_valid"] = pano.valid
    med = engine.median_outlier_filter(pano, window=5, rel_threshold=0.2)
    out["median_valid"] = med.valid
    # float64 reference cost (E:169-224) at a few pixels of the final map
    from densify360.geometry import PlaneHypothesis
    pr = np.random.default_rng(1)
    px = np.stack([pr.integers(0, cam.width, 40), pr.integers(0, cam.height, 40)], 1)
    pc = []
    for x, y in px:
        n = init.normal[y, x].astype(np.float64)
        n /= np.linalg.norm(n)
        pc.append(engine.patch_cost(prep, (x, y), PlaneHypothesis(float(init.depth[y, x]), n), spec))
    out["patch_cost_px"] = px
    out["patch_cost"] = np.array(pc)
    np.savez_compressed(OUT / f"{name}.npz", **out)
    print(name, "steps", len(keep), "final mean cost", float(cur.cost.mean()), "valid", float(pano.valid.mean()))


def stage_case():
    """DepthStage chain (warp + random init), consistency filter, fusion on 64x32."""
    cam = EquirectCamera(64, 32)
    spec = PatchSpec()
    n_kf = 9
    poses = [RigidPose(rotation=rot(1, 2.0 * k) @ rot(0, 1.0 * k),
                       translation=np.array([0.02 * k, 0.01 * k, -0.6 + 0.15 * k])) for k in range(n_kf)]
    frames, gts = make_frames(cam, poses)
    stage = pipeline.DepthStage(cam, spec, DEPTH_RANGE, iterations=2, seed=3, warp=True, workers=8)
    results = []
    warp_io = None
    for k in range(1, n_kf - 1):
        group = StereoGroup(reference=frames[k], neighbors=(frames[k - 1], frames[k + 1]), camera=cam)
        if k == 2:
            prev_map, prev_pose = stage._prev
            w = engine.warp_plane_map(prev_map, prev_pose, frames[k].pose, cam)
            warp_io = (prev_map.copy(), w)
        results.append(stage.process(group))
    out = {
        "images": np.stack([f.image for f in frames]),
        "rotations": pose_arrays(frames)[0], "translations": pose_arrays(frames)[1],
        "depth_range": np.array(DEPTH_RANGE), "seed": 3, "iterations": 2,
        "stage_ids": np.array([r.id for r in results]),
        "stage_depth": np.stack([r.pano.depth for r in results]),
        "stage_valid": np.stack([r.pano.valid for r in results]),
        "warp_src_depth": warp_io[0].depth, "warp_src_normal": warp_io[0].normal,
        "warp_src_cost": warp_io[0].cost, "warp_src_valid": warp_io[0].valid,
        "warp_out_depth": warp_io[1].depth, "warp_out_normal": warp_io[1].normal,
        "warp_out_cost": warp_io[1].cost, "warp_out_valid": warp_io[1].valid,
    }
    # consistency + fusion on ground-truth panoramas with a sprinkling of outliers
    rng = np.random.default_rng(5)
    panos = []
    for k in range(5):
        d = gts[k + 1].astype(np.float32).copy()
        v = rng.uniform(size=d.shape) > 0.1
        bad = rng.uniform(size=d.shape) < 0.2
        d[bad] *= rng.uniform(0.7, 1.3, size=int(bad.sum())).astype(np.float32)
        panos.append(engine.DepthPanorama(cam, d, v))
    ccfg = pipeline.ConsistencyConfig()
    target = panos[2]
    others = [(panos[i], poses[i + 1]) for i in (0, 1, 3, 4)]
    filt = pipeline.consistency_filter(target, poses[3], others, ccfg)
    out.update(cons_depth=np.stack([p.depth for p in panos]), cons_valid=np.stack([p.valid for p in panos]),
               cons_out_valid=filt.valid)
    fcfg = pipeline.FusionConfig()
    fb = pipeline.FusionBuffer(cam, fcfg)
    cloud = None
    for k in range(4):
        res = pipeline.DepthResult(id=k + 1, pano=panos[k], pose=poses[k + 1], image=frames[k + 1].image, seconds=0.0)
        got = fb.push(res)
        if got is not None:
            cloud = got
    out.update(fuse_points=cloud.points, fuse_colors=cloud.colors, fuse_ids=cloud.source_ids)
    np.savez_compressed(OUT / "stage_64x32.npz", **out)
    print("stage", [float(r.pano.valid.mean()) for r in results], "warp fill", float(warp_io[1].valid.mean()),
          "cons survive", float(filt.valid.mean()), "fused", len(cloud.points))


def misc_case():
    """random_init known answers (PCG64), to_gray, rays, median edge cases."""
    cam = EquirectCamera(32, 16)
    pm = PlaneMap.empty(cam, (0.5, 8.0))
    pm.depth[3, 7] = 2.25
    pm.normal[3, 7] = (0, 0, -1)
    pm.valid[3, 7] = True
    ri = engine.random_init(pm, (0.5, 8.0), seed=42)
    rng = np.random.default_rng(9)
    img = rng.integers(0, 256, size=(16, 32, 3), dtype=np.uint8)
    depth = rng.uniform(0.5, 8.0, size=(16, 32)).astype(np.float32)
    valid = rng.uniform(size=(16, 32)) > 0.3
    med3 = engine.median_outlier_filter(engine.DepthPanorama(cam, depth, valid), 3, 0.2).valid
    med7 = engine.median_outlier_filter(engine.DepthPanorama(cam, depth, valid), 7, 0.35).valid
    np.savez_compressed(OUT / "misc_32x16.npz", ri_depth=ri.depth, ri_normal=ri.normal, ri_cost=ri.cost,
                        ri_valid=ri.valid, gray_in=img, gray_out=to_gray(img), gray2_out=to_gray(img[..., 0]),
                        rays32=camera_rays(cam).astype(np.float32), med_depth=depth, med_valid=valid,
                        med3=med3, med7=med7)
    print("misc ok")


def io_metrics_case():
    """Output writers (outputs.py) and metrics (metrics.py): bytes / numbers of the reference."""
    import tempfile

    from densify360 import metrics, outputs
    from densify360.pipeline import FusedCloud

    rng = np.random.default_rng(31)
    n = 257
    pts = rng.normal(size=(n, 3)) * np.array([2.0, 1.0, 3.0]) + np.array([0.1, -0.2, 0.3])
    pts[5] = (0.1, -0.2, 0.3)  # coincides with the first pose centre: dropped by completeness (r <= 1e-12)
    cols = rng.integers(0, 256, size=(n, 3), dtype=np.uint8)
    cloud = FusedCloud(pts, cols, np.zeros(n, np.int64))
    cam = EquirectCamera(32, 16)
    depth = rng.uniform(0.2, 70.0, size=(16, 32)).astype(np.float32)  # > 65.535 m clips
    depth[2, 3] = 1.0005  # rint half-to-even candidates in millimetres
    depth[2, 4] = 2.0015
    valid = rng.uniform(size=(16, 32)) > 0.25
    pano = engine.DepthPanorama(cam, depth, valid)
    with tempfile.TemporaryDirectory() as d:
        outputs.write_ply(Path(d) / "c.ply", cloud)
        ply = np.frombuffer((Path(d) / "c.ply").read_bytes(), np.uint8)
        outputs.write_depth_png(Path(d) / "d.png", pano)
        png = np.frombuffer((Path(d) / "d.png").read_bytes(), np.uint8)
        sidecar = (Path(d) / "d.json").read_text()
        back = outputs.read_depth_png(Path(d) / "d.png")
    poses = [RigidPose(np.eye(3), np.array([0.1, -0.2, 0.3])),
             RigidPose(rot(1, 33.0) @ rot(0, -12.0), np.array([-0.5, 0.1, 0.9])),
             RigidPose(rot(2, 80.0), np.array([1.5, 0.4, -2.0]))]
    comp_cam = EquirectCamera(72, 36)
    comp = metrics.completeness(pts, poses, comp_cam)
    comp_default = metrics.completeness(pts, poses[:2])
    gt = engine.DepthPanorama(cam, (depth * rng.uniform(0.97, 1.03, size=depth.shape)).astype(np.float32),
                              rng.uniform(size=(16, 32)) > 0.2)
    acc = metrics.accuracy(pano, gt)
    vox = [metrics.voxel_occupancy(pts, v) for v in (0.1, 0.5, 2.0)]
    np.savez_compressed(OUT / "io_metrics.npz", points=pts, colors=cols, ply=ply, depth=depth, valid=valid, png=png,
                        sidecar=np.array(sidecar), back_depth=back.depth, back_valid=back.valid,
                        pose_r=np.stack([p.rotation for p in poses]), pose_t=np.stack([p.translation for p in poses]),
                        comp_series=np.array(comp["per_keyframe"]), comp_mean=comp["mean"],
                        comp_default_series=np.array(comp_default["per_keyframe"]), gt_depth=gt.depth,
                        gt_valid=gt.valid, acc=np.array([acc["mean_abs_rel"], acc["rmse_m"], acc["inlier_2pc"],
                                                          acc["valid_pixels"]]), vox=np.array(vox))
    print("io/metrics ok", len(ply), len(png), comp["per_keyframe"], acc, vox)


def offline_case():
    """run_offline on the 20-keyframe 64x32 room of the reference's own pipeline test
    (tests/test_pipeline.py:279-296): inputs, every view-filter decision, report, filtered maps."""
    import tempfile

    from densify360.config import load_config
    from densify360.dataset import load_dataset
    from densify360.pipeline import run_offline
    from densify360.synth import make_dataset
    from densify360.viewfilter import view_filter_accept

    with tempfile.TemporaryDirectory() as d:
        make_dataset(default_scene("box"), keyframes=20, sparse_density=150, out_dir=d, camera=EquirectCamera(64, 32),
                     seed=5)
        ds = load_dataset(d)
        cfg = load_config(overrides={"patchmatch.iterations": 4, "patchmatch.depth_max": 8.0,
                                     "consistency.rel_depth_tol": 0.05, "processing.threaded": False})
        kfs = list(ds.keyframes())
        # a second landmark layout that makes the view filter reject: drop most shared landmarks of some frames
        res = run_offline(ds, cfg)
        latest, decisions = None, []
        for kf in kfs:
            if latest is None:
                decisions.append((1, 1.0, 0))
                latest = kf
                continue
            dec = view_filter_accept(kf, latest, cfg.viewfilter)
            decisions.append((int(dec.accepted), dec.fraction, dec.common_points))
            if dec.accepted:
                latest = kf
    rep = res.report
    ids = sorted(res.depths)
    np.savez_compressed(
        OUT / "offline_64x32.npz", images=np.stack([k.image for k in kfs]),
        rotations=np.stack([k.pose.rotation for k in kfs]), translations=np.stack([k.pose.translation for k in kfs]),
        sparse=np.stack([k.sparse_points for k in kfs]), decisions=np.array(decisions),
        vf=np.array([cfg.viewfilter.theta_min, cfg.viewfilter.theta_max, cfg.viewfilter.accept_fraction]),
        keyframes_total=rep["keyframes_total"], keyframes_accepted=rep["keyframes_accepted"],
        depth_jobs=rep["depth_jobs"], fused_points=rep["fused_points"],
        comp_series=np.array(rep["completeness"]["per_keyframe"]), comp_mean=rep["completeness"]["mean"],
        depth_ids=np.array(ids), depths=np.stack([res.depths[i].pano.depth for i in ids]),
        valids=np.stack([res.depths[i].pano.valid for i in ids]), cloud_ids=res.cloud.source_ids,
        report_keys=np.array(sorted(rep)))
    print("offline ok", rep["keyframes_total"], rep["keyframes_accepted"], rep["depth_jobs"], rep["fused_points"],
          rep["completeness"]["mean"], ids, decisions[:4])


def render_case():
    """synth.render_scene (SY:154-169) for every scene kind, with rotated poses and the checker texture."""
    cam = EquirectCamera(64, 32)
    cases = [("sphere", False, RigidPose(np.eye(3), np.array([0.31, -0.27, 0.45]))),
             ("sphere", False, RigidPose(rot(1, 33.0) @ rot(0, -12.0), np.array([-0.5, 0.2, 0.1]))),
             ("box", True, RigidPose(rot(2, 8.0) @ rot(1, -21.0), np.array([0.4, -0.3, 0.9]))),
             ("corridor", False, RigidPose(rot(0, 5.0) @ rot(1, 170.0), np.array([0.7, 0.4, -6.5]))),
             ("box", False, RigidPose(rot(1, 91.0) @ rot(2, 45.0) @ rot(0, -30.0), np.array([-1.1, 0.9, 1.7])))]
    out = {"kinds": np.array([c[0] for c in cases]), "checker": np.array([c[1] for c in cases]),
           "rotations": np.stack([c[2].rotation for c in cases]), "translations": np.stack([c[2].translation for c in cases])}
    imgs, depths = [], []
    for kind, checker, pose in cases:
        image, pano = render_scene(default_scene(kind, checker=checker), cam, pose)
        imgs.append(image)
        depths.append(pano.depth)
    # a larger frame too: the BLAS kernels behind rays @ R.T may differ with the matrix size
    big = EquirectCamera(512, 256)
    image, pano = render_scene(default_scene("sphere"), big, cases[1][2])
    from densify360.synth import straight_line_trajectory
    traj = straight_line_trajectory(default_scene("corridor"), 9)
    np.savez_compressed(OUT / "render_64x32.npz", images=np.stack(imgs), depths=np.stack(depths), big_image=image,
                        big_depth=pano.depth, traj=np.stack([q.translation for q in traj]), **out)
    print("render ok", [int(i.mean()) for i in imgs])


def resample_case():
    """dataset.resample_keyframe (dataset.py:146-157, Pillow LANCZOS): down, up, one axis only, gray."""
    from densify360.dataset import resample_keyframe
    cam = EquirectCamera(128, 64)
    image, _ = render_scene(default_scene("box"), cam, RigidPose(np.eye(3), np.zeros(3)))
    rng = np.random.default_rng(3)
    noise = rng.integers(0, 256, (50, 100, 3), dtype=np.uint8)
    out = {"src_box": image, "src_noise": noise}
    for name, src, (w, h) in (("box_down", image, (64, 32)), ("box_up", image, (192, 96)), ("noise_to_64", noise, (64, 32)),
                              ("noise_up", noise, (256, 128))):
        kf = Keyframe(id=0, image=src, pose=RigidPose(np.eye(3), np.zeros(3)))
        out[name] = resample_keyframe(kf, EquirectCamera(w, h)).image
    np.savez_compressed(OUT / "resample_128x64.npz", **out)
    print("resample ok", {k: v.shape for k, v in out.items()})


def dataset_case():
    """synth.make_dataset (SY:252-330): manifest text and PNG bytes of a 5-keyframe corridor dataset."""
    import hashlib
    import tempfile
    from densify360.synth import make_dataset
    with tempfile.TemporaryDirectory() as tmp:
        root = make_dataset(default_scene("corridor", keyframes=5), 5, 7, tmp, EquirectCamera(64, 32), seed=5)
        manifest = (root / "dataset.json").read_bytes()
        pngs = [np.frombuffer((root / f"kf{k:04d}.png").read_bytes(), np.uint8) for k in range(5)]
    np.savez_compressed(OUT / "dataset_64x32.npz", manifest=np.frombuffer(manifest, np.uint8),
                        **{f"png{k}": a for k, a in enumerate(pngs)})
    print("dataset ok", hashlib.sha256(manifest).hexdigest()[:12], [len(a) for a in pngs])


if __name__ == "__main__":
    if sys.argv[1:] == ["dataset"]:
        dataset_case()
        sys.exit(0)
    if sys.argv[1:] == ["resample"]:
        resample_case()
        sys.exit(0)
    if sys.argv[1:] == ["render"]:
        render_case()
        sys.exit(0)
    if sys.argv[1:] == ["io"]:
        io_metrics_case()
        sys.exit(0)
    if sys.argv[1:] == ["offline"]:
        offline_case()
        sys.exit(0)
    ident = lambda z: RigidPose(rotation=np.eye(3), translation=np.array([0.0, 0.0, z]))
    hot_path_case("hot_64x32_ident", 64, 3, [ident(-0.15), ident(0.0), ident(0.15)], PatchSpec(), 7, True)
    rposes = [RigidPose(rot(1, -7.0) @ rot(0, 3.0), np.array([0.05, -0.02, -0.17])),
              RigidPose(rot(2, 4.0), np.array([0.0, 0.0, 0.0])),
              RigidPose(rot(1, 9.0) @ rot(2, -5.0), np.array([-0.04, 0.03, 0.16]))]
    hot_path_case("hot_64x32_rot", 64, 2, rposes, PatchSpec(half_window=3, sample_stride=1), 11, True)
    hot_path_case("hot_256x128_c1", 256, 3, [ident(-0.15), ident(0.0), ident(0.15)], PatchSpec(), 0, False)
    stage_case()
    misc_case()
    io_metrics_case()
    offline_case()
    render_case()
    resample_case()
    dataset_case()
