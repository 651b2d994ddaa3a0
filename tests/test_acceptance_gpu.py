"""The reference's acceptance criteria that concern the hot path (tests/test_acceptance.py there,
SPEC.md:446-457), run through this package on the GPU with the reference's own bars."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def pkg():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2211_16266_b200 as p
    from paper_2211_16266_b200 import engine, metrics, offline, pipeline, synth

    return p, engine, pipeline, synth, offline, metrics


def test_acceptance_3_depth_accuracy_on_ground_truth(pkg):
    """Criterion 3: on the synthetic box room the filtered depth maps have mean |rel| error <= 5 %
    and >= 70 % of the pixels within 2 % of ground truth (test_acceptance.py:133-151)."""
    p, engine, pipeline, synth, offline, metrics = pkg
    cam = p.EquirectCamera(512, 256)
    scene = synth.default_scene("box")
    landmarks = np.random.default_rng(2).uniform(-1.0, 1.0, size=(60, 3)) * np.array([1.9, 1.4, 2.4])
    kfs = []
    for k in range(12):
        pose = p.RigidPose(np.eye(3), np.array([0.3, -0.1, -0.9 + 0.15 * k]))
        img, _ = synth.render_scene(scene, cam, pose)
        kfs.append(p.Keyframe(id=k, image=img, pose=pose, sparse_points=landmarks))
    res = offline.run_offline(kfs, cam, viewfilter=offline.ViewFilterConfig(theta_min=1.0), depth_range=(0.5, 16.0),
                              iterations=6, seed=0)
    assert res.report["keyframes_accepted"] == 12 and res.report["depth_jobs"] == 10 and len(res.depths) == 6
    rels, inliers = [], []
    for _, dr in sorted(res.depths.items()):
        _, gt = synth.render_scene(scene, cam, dr.pose)
        m = metrics.accuracy(dr.pano, gt)
        assert m["defined"]
        rels.append(m["mean_abs_rel"])
        inliers.append(m["inlier_2pc"])
    assert np.mean(rels) <= 0.05 and np.mean(inliers) >= 0.70, (rels, inliers)
    assert res.report["fused_points"] > 0 and 0 < res.report["completeness"]["mean"] <= 1


def test_acceptance_6_wraparound_equivariance(pkg):
    """Criterion 6: rolling every image by a quarter turn and yawing every pose by 90 degrees rolls
    the depth map: >= 99.9 % of the valid pixels within 1e-6 (test_acceptance.py:223-278).
    Exercises the column wrap of the patch window, of the propagation and of the bilinear taps."""
    p, engine, pipeline, synth, _, _ = pkg
    cam = p.EquirectCamera(128, 64)
    spec, dr = engine.PatchSpec(), (0.5, 16.0)
    group, _ = synth.make_group(synth.default_scene("box"), cam, (0.0, 0.0, 0.0), n_views=2, step=0.15, axis=1)
    shift = cam.width // 4
    yaw90 = np.array([[0.0, 0.0, -1.0], [0.0, 1.0, 0.0], [1.0, 0.0, 0.0]])

    def rolled(kf):
        return p.Keyframe(id=kf.id, image=np.roll(kf.image, shift, axis=1),
                          pose=p.RigidPose(kf.pose.rotation @ yaw90, kf.pose.translation))

    rgroup = p.StereoGroup(reference=rolled(group.reference), neighbors=tuple(rolled(n) for n in group.neighbors),
                           camera=cam)
    init = engine.random_init(engine.PlaneMap.empty(cam, dr), dr, seed=3)
    rinit = engine.PlaneMap(cam, np.roll(init.depth, shift, axis=1),
                            np.ascontiguousarray(np.roll(init.normal, shift, axis=1) @ yaw90).astype(np.float32),
                            np.roll(init.cost, shift, axis=1), np.roll(init.valid, shift, axis=1), init.depth_range)

    def densify(grp, ini):
        _, pano = engine.run_patchmatch(grp, ini, spec, 6, 3)
        pano = engine.median_outlier_filter(pano)
        pano.valid[np.abs(np.degrees(p.row_latitudes(cam))) > 85.0, :] = False
        return pano

    pano, rpano = densify(group, init), densify(rgroup, rinit)
    rolled_depth, rolled_valid = np.roll(pano.depth, shift, axis=1), np.roll(pano.valid, shift, axis=1)
    joint = rolled_valid & rpano.valid
    assert joint.sum() >= 0.99 * rolled_valid.sum()
    diff = np.abs(rpano.depth[joint].astype(np.float64) - rolled_depth[joint].astype(np.float64))
    assert (diff <= 1e-6).mean() >= 0.999, ((diff <= 1e-6).mean(), diff.max())


def test_acceptance_4_consistency_filter_behaviour(pkg):
    """Criterion 4: ground-truth maps of a five-frame window survive the geometric-consistency
    filter (>= 99 %), random depths do not (<= 1 %), and the filter never validates a pixel
    (test_acceptance.py:154-190; the box room at 512x256 stands in for the reference's sphere
    scene, which this package does not render)."""
    p, engine, pipeline, synth, _, _ = pkg
    cam = p.EquirectCamera(512, 256)
    scene = synth.default_scene("box")
    frames = []
    for k in range(5):
        pose = p.RigidPose(np.eye(3), np.array([0.0, 0.0, (k - 2) * 0.1]))
        _, pano = synth.render_scene(scene, cam, pose)
        frames.append((pano, pose))
    target, target_pose = frames[2]
    window = frames[:2] + frames[3:]
    cfg = pipeline.ConsistencyConfig()
    gt_out = pipeline.consistency_filter(target, target_pose, window, cfg)
    assert gt_out.valid.mean() >= 0.99, gt_out.valid.mean()
    assert np.array_equal(gt_out.depth, target.depth)  # depths untouched
    rng = np.random.default_rng(20240817)
    rnd = engine.DepthPanorama(cam, rng.uniform(0.5, 8.0, cam.shape).astype(np.float32), np.ones(cam.shape, bool))
    assert pipeline.consistency_filter(rnd, target_pose, window, cfg).valid.mean() <= 0.01
    for _ in range(3):
        partial = engine.DepthPanorama(cam, target.depth, target.valid & (rng.random(cam.shape) > rng.uniform(0.2, 0.8)))
        out = pipeline.consistency_filter(partial, target_pose, window, cfg)
        assert not (out.valid & ~partial.valid).any()


def test_acceptance_1_matches_exhaustive_plane_search(pkg):
    """Criterion 1 (test_acceptance.py:75-96): after 6 iterations from a random start >= 90 % of the pixels sit
    within 5 % of the exhaustive minimum over 96 inverse-depth levels x fronto-parallel normals.  The exhaustive
    search is 96 eval_costs launches here (the reference loops 96 x H x W oracle_patch_cost calls)."""
    p, engine, pipeline, synth, offline, metrics = pkg
    cam = p.EquirectCamera(64, 32)
    dr = (0.5, 8.0)
    group, _ = synth.make_group(synth.default_scene("box"), cam, n_views=2)
    spec = engine.PatchSpec()
    prep = engine.prepare_group(group, spec)
    init = engine.random_init(engine.PlaneMap.empty(cam, dr), dr, seed=7)
    pm, _ = engine.run_patchmatch(prep, init, spec, iterations=6, seed=7)
    final = torch.from_numpy(pm.cost.astype(np.float64)).cuda()
    rays = p.camera_rays(cam)
    best = torch.full(cam.shape, float("inf"), dtype=torch.float64, device="cuda")
    probe = engine.DevicePlaneMap.from_host(engine.PlaneMap(cam, np.zeros(cam.shape, np.float32), (-rays).astype(np.float32),
                                                            np.full(cam.shape, np.inf, np.float32), np.ones(cam.shape, bool), dr))
    for inv in np.linspace(1.0 / dr[1], 1.0 / dr[0], 96):
        probe.depth.fill_(float(1.0 / inv))
        engine.evaluate_costs_device(prep, probe)
        best = torch.minimum(best, probe.cost.double())
    good = final <= best * 1.05 + 1e-6
    assert good.double().mean().item() >= 0.90, good.double().mean().item()


def test_acceptance_2_warping_improves_corridor_coverage(pkg):
    """Criterion 2 (test_acceptance.py:99-130): at a single-sweep budget (one iteration per keyframe) warping
    carries converged planes from keyframe to keyframe, so the run with warp keeps more of the corridor than the
    run without: higher completeness and more fused points."""
    p, engine, pipeline, synth, offline, metrics = pkg
    cam = p.EquirectCamera(512, 256)
    kfs = synth.make_sequence(synth.default_scene("corridor"), 30, 200, cam, seed=5)
    reports = {}
    for warp in (True, False):
        reports[warp] = offline.run_offline(kfs, cam, iterations=1, warp=warp, seed=0).report
    assert reports[True]["depth_jobs"] == reports[False]["depth_jobs"] > 0
    assert reports[True]["completeness"]["mean"] > reports[False]["completeness"]["mean"], reports
    assert reports[True]["fused_points"] > reports[False]["fused_points"]
