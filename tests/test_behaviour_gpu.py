"""Behaviour tests in the style of the reference's test_engine.py classes that the parity files do not
already cover (TestPatchCost 198-243, TestRandomInit 244-282, TestWarp 285-329, TestRefinement 420-462,
TestMedianFilter 519-572), through this package's host API.  The parity tests pin the numbers; these pin
what the numbers mean."""
import math

import numpy as np
import pytest

from test_engine_gpu import box_normals

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

DEPTH_RANGE = (0.5, 8.0)


@pytest.fixture(scope="module")
def pkg():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2211_16266_b200 as p
    from paper_2211_16266_b200 import engine, synth

    return p, engine, synth


def gt_map(p, engine, cam, gt, normals, cost):
    return engine.PlaneMap(cam, gt.astype(np.float32), normals.astype(np.float32),
                           np.full(cam.shape, cost, np.float32), np.ones(cam.shape, bool), DEPTH_RANGE)


def costs_of(engine, prep, pm):
    d = engine.DevicePlaneMap.from_host(pm)
    engine.evaluate_costs_device(prep, d)
    return d.cost.cpu().numpy()


# ---- matching cost (TestPatchCost)

def test_ground_truth_plane_scores_low_and_beats_doubled_depth(pkg):
    p, engine, synth = pkg
    cam = p.EquirectCamera(64, 32)
    scene = synth.default_scene("box")
    group, gt = synth.make_group(scene, cam, n_views=2, step=0.02)  # tiny baseline: near-identical images
    normals = box_normals(scene, p.camera_rays(cam), gt)
    prep = engine.prepare_group(group, engine.PatchSpec())
    good = costs_of(engine, prep, gt_map(p, engine, cam, gt, normals, np.inf))
    inner = good[4:-4]
    assert np.median(inner) < 0.05
    group, gt = synth.make_group(scene, cam, n_views=2, step=0.15)
    prep = engine.prepare_group(group, engine.PatchSpec())
    good = costs_of(engine, prep, gt_map(p, engine, cam, gt, normals, np.inf))[4:-4]
    bad = costs_of(engine, prep, gt_map(p, engine, cam, np.minimum(2 * gt, 7.9), normals, np.inf))[4:-4]
    assert (good < bad).mean() >= 0.95


def test_unrelated_noise_images_cost_near_truncation(pkg):
    p, engine, _ = pkg
    cam = p.EquirectCamera(64, 32)
    rng = np.random.default_rng(0)
    kfs = [p.Keyframe(id=k, image=rng.integers(0, 256, (*cam.shape, 3), dtype=np.uint8),
                      pose=p.RigidPose(np.eye(3), np.array([0.0, 0.0, z]))) for k, z in enumerate((-0.1, 0.0, 0.1))]
    group = p.StereoGroup(reference=kfs[1], neighbors=(kfs[0], kfs[2]), camera=cam)
    spec = engine.PatchSpec()
    rays = p.camera_rays(cam)
    pm = engine.PlaneMap(cam, np.full(cam.shape, 2.0, np.float32), (-rays).astype(np.float32),
                         np.full(cam.shape, np.inf, np.float32), np.ones(cam.shape, bool), DEPTH_RANGE)
    c = costs_of(engine, engine.prepare_group(group, spec), pm)[4:-4]
    assert np.median(c) == pytest.approx(spec.cost_truncation, rel=0.25)  # 1 - NCC of noise is about 1


# ---- random initialisation (TestRandomInit)

def test_random_init_determinism_constraints_and_preserved_pixels(pkg):
    p, engine, _ = pkg
    cam = p.EquirectCamera(64, 32)
    a = engine.random_init(engine.PlaneMap.empty(cam, DEPTH_RANGE), DEPTH_RANGE, seed=42)
    b = engine.random_init(engine.PlaneMap.empty(cam, DEPTH_RANGE), DEPTH_RANGE, seed=42)
    c = engine.random_init(engine.PlaneMap.empty(cam, DEPTH_RANGE), DEPTH_RANGE, seed=43)
    assert np.array_equal(a.depth, b.depth) and np.array_equal(a.normal, b.normal)
    assert not np.array_equal(a.depth, c.depth)
    assert a.valid.all() and np.isinf(a.cost).all()
    assert (a.depth >= DEPTH_RANGE[0]).all() and (a.depth <= DEPTH_RANGE[1]).all()
    assert np.allclose(np.linalg.norm(a.normal, axis=-1), 1.0, atol=1e-5)
    assert (np.einsum("ijk,ijk->ij", a.normal.astype(np.float64), p.camera_rays(cam)) < 0).all()  # facing the camera
    pm = engine.PlaneMap.empty(cam, DEPTH_RANGE)
    pm.depth[3, 7], pm.normal[3, 7], pm.valid[3, 7], pm.cost[3, 7] = 2.25, (0, 0, -1), True, 0.125
    out = engine.random_init(pm, DEPTH_RANGE, seed=9)
    assert out.depth[3, 7] == np.float32(2.25) and tuple(out.normal[3, 7]) == (0, 0, -1) and out.cost[3, 7] == 0.125
    from paper_2211_16266_b200.errors import ConfigError
    for bad in ((0.0, 1.0), (2.0, 1.0), (-1.0, 3.0)):
        with pytest.raises(ConfigError):
            engine.random_init(engine.PlaneMap.empty(cam, DEPTH_RANGE), bad, seed=1)


@pytest.mark.parametrize("rng_kind", ["pcg64", "philox"])
def test_random_init_is_uniform_in_inverse_depth(pkg, rng_kind):
    p, engine, _ = pkg
    cam = p.EquirectCamera(1536, 768)  # > 1e6 pixels
    pm = engine.DevicePlaneMap.empty(cam, DEPTH_RANGE)
    engine.random_init_device(pm, DEPTH_RANGE, 3, rng_kind)
    inv = 1.0 / pm.depth.double().cpu().numpy().ravel()
    lo, hi = 1.0 / DEPTH_RANGE[1], 1.0 / DEPTH_RANGE[0]
    bins = 16
    counts, _ = np.histogram(inv, bins=bins, range=(lo, hi))
    n = inv.size
    sigma = math.sqrt(n * (1 / bins) * (1 - 1 / bins))
    assert np.all(np.abs(counts - n / bins) <= 4 * sigma), counts


# ---- plane-map warp (TestWarp)

def test_warp_identity_empty_and_forward_motion(pkg):
    p, engine, synth = pkg
    cam = p.EquirectCamera(64, 32)
    scene = synth.default_scene("box")
    ident = p.RigidPose.identity()
    pm = engine.random_init(engine.PlaneMap.empty(cam, DEPTH_RANGE), DEPTH_RANGE, seed=2)
    pm.cost[:] = 0.5
    same = engine.warp_plane_map(pm, ident, ident, cam)
    assert same.valid.mean() > 0.99
    assert np.allclose(same.depth[same.valid], pm.depth[same.valid], rtol=1e-4)
    assert (same.cost[same.valid] == 0.5).all()  # the source cost travels with the plane
    empty = engine.warp_plane_map(engine.PlaneMap.empty(cam, DEPTH_RANGE), ident, ident, cam)
    assert not empty.valid.any()
    _, gt = synth.make_group(scene, cam, n_views=2)
    normals = box_normals(scene, p.camera_rays(cam), gt)
    moved = p.RigidPose(np.eye(3), np.array([0.0, 0.0, 0.3]))
    warped = engine.warp_plane_map(gt_map(p, engine, cam, gt, normals, 0.1), ident, moved, cam)
    assert warped.valid.mean() >= 0.70  # reference baseline: 0.87 fill on this room
    _, pano = synth.render_scene(scene, cam, moved)
    ok = warped.valid
    rel = np.abs(warped.depth[ok] - pano.depth[ok]) / pano.depth[ok]
    assert np.quantile(rel, 0.9) < 0.05  # the re-anchored planes are the room seen from the new pose


# ---- refinement (TestRefinement)

def test_refinement_is_monotone_and_leaves_a_strict_optimum_alone(pkg):
    p, engine, synth = pkg
    cam = p.EquirectCamera(64, 32)
    scene = synth.default_scene("box")
    group, gt = synth.make_group(scene, cam, n_views=2, step=0.02)
    spec = engine.PatchSpec()
    prep = engine.prepare_group(group, spec)
    pm = engine.DevicePlaneMap.from_host(engine.random_init(engine.PlaneMap.empty(cam, DEPTH_RANGE), DEPTH_RANGE, seed=4))
    engine.evaluate_costs_device(prep, pm)
    ws_evals = torch.zeros(2, dtype=torch.int64, device=pm.depth.device)
    for seed in (0, 1, 2):
        before = pm.cost.clone()
        table = engine.refinement_draw_tables(seed, 1, 0.25 * (DEPTH_RANGE[1] - DEPTH_RANGE[0]), math.radians(60.0))[0]
        engine.refine_pass_device(prep, pm, table, DEPTH_RANGE)
        assert (pm.cost <= before).all()  # a candidate is adopted only if it is strictly better (K:600)
        assert (pm.depth >= DEPTH_RANGE[0]).all() and (pm.depth <= DEPTH_RANGE[1]).all()
        assert torch.allclose(pm.normal.norm(dim=-1), torch.ones_like(pm.depth), atol=1e-5)
    # from the true planes: a pixel either keeps its plane and its cost, bit for bit, or moves to a strictly
    # cheaper one - nothing is adopted on a tie (the reference's convex-cost test, T/test_engine.py:436-462)
    normals = box_normals(scene, p.camera_rays(cam), gt)
    opt = engine.DevicePlaneMap.from_host(gt_map(p, engine, cam, gt, normals, np.inf))
    engine.evaluate_costs_device(prep, opt)
    d0, c0 = opt.depth.clone(), opt.cost.clone()
    engine.refine_pass_device(prep, opt, engine.refinement_draw_tables(5, 1, 1.875, math.radians(60.0))[0], DEPTH_RANGE)
    kept = opt.depth == d0
    assert (opt.cost[~kept] < c0[~kept]).all() and (opt.cost[kept] == c0[kept]).all()


# ---- median outlier filter (TestMedianFilter)

def test_median_filter_removes_spikes_and_never_smooths(pkg):
    p, engine, synth = pkg
    cam = p.EquirectCamera(64, 32)
    flat = engine.DepthPanorama(cam, np.full(cam.shape, 2.0, np.float32), np.ones(cam.shape, bool))
    out = engine.median_outlier_filter(flat, window=5, rel_threshold=0.1)
    assert out.valid.all() and np.array_equal(out.depth, flat.depth)
    spike = flat.copy()
    spike.depth[10, 20] = 20.0
    out = engine.median_outlier_filter(spike, window=5, rel_threshold=0.1)
    assert not out.valid[10, 20] and out.valid.sum() == spike.valid.sum() - 1
    assert np.array_equal(out.depth, spike.depth)  # removes, never smooths
    # salt and pepper on the room's ground-truth depth
    _, gt = synth.make_group(synth.default_scene("box"), cam, n_views=2)
    rng = np.random.default_rng(0)
    depth = gt.copy().ravel()
    corrupt = rng.choice(depth.size, size=int(0.05 * depth.size), replace=False)
    depth[corrupt] *= np.where(rng.random(corrupt.size) < 0.5, 0.2, 5.0)
    bad = np.zeros(depth.size, bool)
    bad[corrupt] = True
    bad = bad.reshape(cam.shape)
    out = engine.median_outlier_filter(engine.DepthPanorama(cam, depth.reshape(cam.shape).astype(np.float32),
                                                            np.ones(cam.shape, bool)), window=5, rel_threshold=0.2)
    assert (~out.valid & bad).sum() / bad.sum() >= 0.95 and (~out.valid & ~bad).sum() / (~bad).sum() <= 0.02
    # the output mask is a subset of the input mask
    valid = rng.random(cam.shape) > 0.3
    pano = engine.DepthPanorama(cam, rng.uniform(1.0, 3.0, cam.shape).astype(np.float32), valid)
    assert not (engine.median_outlier_filter(pano, window=3, rel_threshold=0.05).valid & ~valid).any()
    from paper_2211_16266_b200.errors import ConfigError
    for w in (4, 1):
        with pytest.raises(ConfigError):
            engine.median_outlier_filter(flat, window=w, rel_threshold=0.1)
