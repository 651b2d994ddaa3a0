"""Propagation / refinement behaviour tests in the style of the reference's test_engine.py
(TestRedBlack, TestRefinement, TestRunPatchmatch: 332-516), through this package's host API."""
import numpy as np
import pytest

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


def box_normals(scene, rays, depth, center=(0.0, 0.0, 0.0)):
    """Inward wall normal at every ground-truth hit of an axis-aligned box seen from `center`."""
    pts = rays * depth[..., None] + np.asarray(center)
    half = np.asarray(scene.size) / 2.0
    axis = np.argmin(np.abs(np.abs(pts) - half), axis=-1)
    n = np.zeros_like(pts)
    np.put_along_axis(n, axis[..., None], -np.sign(np.take_along_axis(pts, axis[..., None], -1)), -1)
    return n.astype(np.float32)


def poisoned_map(p, engine, cam, normals):
    pm = engine.PlaneMap.empty(cam, DEPTH_RANGE)
    pm.depth[:] = 7.5
    pm.normal[:] = normals
    pm.valid[:] = True
    return pm


def test_costs_never_increase_and_parity_partition(pkg):
    p, engine, synth = pkg
    cam = p.EquirectCamera(64, 32)
    group, _ = synth.make_group(synth.default_scene("box"), cam, n_views=2)
    spec = engine.PatchSpec()
    cur = engine.random_init(engine.PlaneMap.empty(cam, DEPTH_RANGE), DEPTH_RANGE, seed=8)
    xs, ys = np.meshgrid(np.arange(cam.width), np.arange(cam.height))
    for parity in ("red", "black", "red", "black"):
        nxt = engine.red_black_iteration(cur, group, spec, parity)
        finite = np.isfinite(cur.cost)
        assert np.all(nxt.cost[finite] <= cur.cost[finite] + 1e-6)
        still = (xs + ys) % 2 == (1 if parity == "red" else 0)
        assert np.array_equal(nxt.depth[still], cur.depth[still]) and np.array_equal(nxt.normal[still], cur.normal[still])
        cur = nxt


def test_flood_fill_propagation(pkg):
    """Truth planted at one pixel, 7.5 m everywhere else: three full iterations carry it at least
    four pixels along each axis on its own checkerboard sublattice."""
    p, engine, synth = pkg
    cam = p.EquirectCamera(64, 32)
    scene = synth.default_scene("box")
    group, gt = synth.make_group(scene, cam, n_views=2)
    rays = p.camera_rays(cam)
    normals = box_normals(scene, rays, gt)
    pm = poisoned_map(p, engine, cam, (-rays).astype(np.float32))
    x0, y0 = 48, 16
    pm.depth[y0, x0], pm.normal[y0, x0] = gt[y0, x0], normals[y0, x0]
    cur, spec = pm, engine.PatchSpec()
    for _ in range(3):
        cur = engine.red_black_iteration(cur, group, spec, "red")
        cur = engine.red_black_iteration(cur, group, spec, "black")
    for dx, dy in [(4, 0), (-4, 0), (0, 4), (0, -4)]:
        x, y = x0 + dx, y0 + dy
        assert abs(cur.depth[y, x] - gt[y, x]) / gt[y, x] < 0.1, (dx, dy)


def test_seam_propagation(pkg):
    """Truth only in the last column: column 0 can improve only across the wrap-around seam."""
    p, engine, synth = pkg
    cam = p.EquirectCamera(64, 32)
    scene = synth.default_scene("box")
    group, gt = synth.make_group(scene, cam, n_views=2, axis=0)
    rays = p.camera_rays(cam)
    normals = box_normals(scene, rays, gt)
    pm = poisoned_map(p, engine, cam, (-rays).astype(np.float32))
    last = cam.width - 1
    pm.depth[:, last], pm.normal[:, last] = gt[:, last], normals[:, last]
    spec = engine.PatchSpec()
    cur = engine.red_black_iteration(pm, group, spec, "red")
    cur = engine.red_black_iteration(cur, group, spec, "black")
    improved = sum(abs(cur.depth[y, 0] - gt[y, 0]) / gt[y, 0] < 0.1 for y in range(4, cam.height - 4))
    assert improved > (cam.height - 8) * 0.5


def test_ground_truth_planes_beat_wrong_depths_and_more_iterations_never_hurt(pkg):
    p, engine, synth = pkg
    cam = p.EquirectCamera(64, 32)
    scene = synth.default_scene("box")
    rays = p.camera_rays(cam)
    spec = engine.PatchSpec()

    def costs(group, depth, normals):
        prep = engine.prepare_group(group, spec)
        pm = engine.DevicePlaneMap.from_host(engine.PlaneMap(cam, depth.astype(np.float32), normals,
                                                             np.full(cam.shape, np.inf, np.float32),
                                                             np.ones(cam.shape, bool), DEPTH_RANGE))
        engine.evaluate_costs_device(prep, pm)
        return pm.cost.cpu().numpy()

    # tiny baseline, ground-truth planes: near-identical patches (test_engine.py:198-207)
    near, gt_n = synth.make_group(scene, cam, n_views=2, step=0.02)
    c = costs(near, gt_n, box_normals(scene, rays, gt_n))
    assert max(c[y, x] for x, y in [(10, 16), (32, 16), (50, 20), (5, 8)]) < 0.05
    # the true plane beats the same plane at twice the depth (test_engine.py:228-241)
    group, gt = synth.make_group(scene, cam, n_views=2, step=0.15)
    normals = box_normals(scene, rays, gt)
    good, bad = costs(group, gt, normals), costs(group, 2.0 * gt, normals)
    assert (good[4:-4] < bad[4:-4]).mean() >= 0.95
    # more iterations never make the mean cost worse (test_engine.py:490-501)
    init = engine.random_init(engine.PlaneMap.empty(cam, DEPTH_RANGE), DEPTH_RANGE, seed=4)
    few, _ = engine.run_patchmatch(group, init, spec, 2, 4)
    many, _ = engine.run_patchmatch(group, init, spec, 5, 4)
    assert many.cost.mean() <= few.cost.mean()


def test_probe_mode_runs_the_reference_monotonicity_checks_and_changes_nothing(pkg, monkeypatch):
    """E:567-570, E:596-598, E:622-624: eight probe pixels are checked after every pass.  The probed drive
    (pass by pass, no memo) returns what the single-call drive returns, bit for bit."""
    p, engine, synth = pkg
    cam = p.EquirectCamera(128, 64)
    group, _ = synth.make_group(synth.default_scene("box"), cam, n_views=4)
    spec = engine.PatchSpec()
    prep = engine.prepare_group(group, spec)
    init = engine.random_init(engine.PlaneMap.empty(cam, DEPTH_RANGE), DEPTH_RANGE, seed=5)
    outs = []
    for probes in (False, True):
        pm = engine.DevicePlaneMap.from_host(init)
        pm, pano = engine.run_patchmatch_device(prep, pm, 3, 11, probes=probes)
        outs.append((pm.depth.cpu(), pm.normal.cpu(), pm.cost.cpu(), pano.valid.cpu()))
    for a, b in zip(*outs):
        assert torch.equal(a, b)
    # the environment switch selects the same path
    monkeypatch.setenv("D360_PROBES", "1")
    called = []
    real = engine._run_patchmatch_probed
    monkeypatch.setattr(engine, "_run_patchmatch_probed", lambda *a, **k: called.append(1) or real(*a, **k))
    engine.run_patchmatch_device(prep, engine.DevicePlaneMap.from_host(init), 1, 11)
    assert called
