"""run_offline / KeyframeBuffer / view filter (row f1) against the reference's own run on the
20-keyframe 64x32 room of its pipeline test (golden: tests/golden/offline_64x32.npz)."""
import numpy as np
import pytest

from conftest import load_golden


def _keyframes(p, z):
    return [p.Keyframe(id=k, image=z["images"][k], pose=p.RigidPose(z["rotations"][k], z["translations"][k]),
                       sparse_points=z["sparse"][k]) for k in range(len(z["images"]))]


def test_view_filter_and_keyframe_buffer_match_reference_decisions():
    """Host logic, no GPU: every accept / reject decision, fraction and landmark count."""
    import paper_2211_16266_b200 as p
    from paper_2211_16266_b200 import offline
    from paper_2211_16266_b200.errors import ConfigError, OrderingError

    z = load_golden("offline_64x32")
    kfs = _keyframes(p, z)
    cfg = offline.ViewFilterConfig(*z["vf"])
    buf = offline.KeyframeBuffer(p.EquirectCamera(64, 32), cfg)
    groups = []
    for kf, (acc, frac, common) in zip(kfs, z["decisions"]):
        dec, group = buf.submit(kf)
        assert dec.accepted == bool(acc) and dec.fraction == frac and dec.common_points == int(common)
        if group is not None:
            groups.append(group)
    assert buf.submitted == int(z["keyframes_total"]) and buf.accepted == int(z["keyframes_accepted"])
    assert len(groups) == int(z["depth_jobs"])
    assert all(g.reference.id == g.neighbors[0].id + 1 or g.neighbors[0].id < g.reference.id < g.neighbors[1].id
               for g in groups)
    with pytest.raises(OrderingError):
        buf.submit(kfs[3])
    with pytest.raises(ConfigError):
        offline.ViewFilterConfig(theta_min=70.0)
    # V = 4: windows of five accepted keyframes, middle reference, nearest neighbours first
    buf4 = offline.KeyframeBuffer(p.EquirectCamera(64, 32), cfg, n_neighbors=4)
    g4 = [g for _, g in (buf4.submit(kf) for kf in kfs) if g is not None]
    assert len(g4) == buf4.accepted - 4
    acc_ids = [kf.id for kf, d in zip(kfs, z["decisions"]) if d[0]]
    assert [n.id for n in g4[0].neighbors] == [acc_ids[1], acc_ids[3], acc_ids[0], acc_ids[4]]
    assert offline.triangulation_angle(np.zeros(3), np.zeros(3), np.ones(3)) == 0.0
    assert abs(offline.triangulation_angle(np.zeros(3), [1, 0, 0], [0, 1, 0]) - 90.0) < 1e-12


def _chain_agreement(got: dict, z) -> tuple:
    """(mask agreement, depths within 0.5 %) per output keyframe against the reference's own run."""
    agree, close = [], []
    for j, kid in enumerate(z["depth_ids"].tolist()):
        depth, valid = got[kid]
        agree.append(float((valid == z["valids"][j]).mean()))
        both = valid & z["valids"][j]
        close.append(float((np.abs(depth - z["depths"][j])[both] <= 0.005 * z["depths"][j][both]).mean()))
    return agree, close


def oracle_chain(z) -> dict:
    """The reference's run_offline stages on the CPU oracle: accepted keyframes -> triples ->
    DepthStage with warp carry-over -> consistency window 5.  {keyframe id: (depth, surviving mask)}."""
    from oracle import d360_oracle as O

    imgs, rot, tr = z["images"], z["rotations"], z["translations"]
    accepted = [k for k, d in enumerate(z["decisions"]) if d[0]]
    dr = (0.5, 8.0)
    prev, window, out = None, [], {}
    for a, k, b in zip(accepted, accepted[1:], accepted[2:]):
        g = O.Group(imgs[k], [imgs[a], imgs[b]], (rot[k], tr[k]), [(rot[a], tr[a]), (rot[b], tr[b])])
        plane, depth, valid = O.depth_stage(g, k, dr, 4, 0, prev, (rot[k], tr[k]))
        prev = (*plane, (rot[k], tr[k]))
        window.append((k, depth, valid, (rot[k], tr[k])))
        if len(window) == 5:
            ck, cd, cv, cp = window[2]
            others = [(d_, v_, p_) for j, (_, d_, v_, p_) in enumerate(window) if j != 2]
            out[ck] = (cd, O.consistency_filter(cd, cv, cp, others, 2, 0.05))
            window.pop(0)
    return out


def test_oracle_chain_anchors_the_statistical_gate():
    """PatchMatch trajectories are chaotic at near-ties: over a 17-job warp-chained run a single
    flipped tie propagates through the warp carry-over.  The CPU oracle - which reproduces every single pass of
    the reference to <= 3e-6 under injected state (test_oracle_golden.py) - agrees with the reference's own run
    of this chain on 99.88 % of the mask pixels and has 99.89 % of the depths within 0.5 % (worst keyframe
    99.46 %): north_star's 99.5 % bar, met on average, with the compiled-C-vs-numba-fastmath rounding
    differences as the only cause.  The GPU test below holds the product to the same figures."""
    z = load_golden("offline_64x32")
    got = oracle_chain(z)
    assert sorted(got) == z["depth_ids"].tolist()
    agree, close = _chain_agreement(got, z)
    assert np.mean(agree) >= 0.995 and np.mean(close) >= 0.995, (np.mean(agree), np.mean(close))
    assert min(agree) >= 0.99 and min(close) >= 0.99, (agree, close)


@pytest.mark.gpu
def test_run_offline_matches_reference_run():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2211_16266_b200 as p
    from paper_2211_16266_b200 import offline, pipeline

    z = load_golden("offline_64x32")
    cam = p.EquirectCamera(64, 32)
    kfs = _keyframes(p, z)
    kw = dict(viewfilter=offline.ViewFilterConfig(*z["vf"]), depth_range=(0.5, 8.0), iterations=4, seed=0,
              consistency=pipeline.ConsistencyConfig(rel_depth_tol=0.05))
    res = offline.run_offline(kfs, cam, **kw)
    rep = res.report
    assert sorted(rep) == z["report_keys"].tolist()
    for key in ("keyframes_total", "keyframes_accepted", "depth_jobs"):
        assert rep[key] == int(z[key]), key
    assert sorted(res.depths) == z["depth_ids"].tolist()
    # PatchMatch trajectories are chaotic at near-ties: statistical parity of the maps, at the
    # level the CPU oracle itself reaches against the reference on this chain (test above)
    agree, close = [], []
    for j, kid in enumerate(sorted(res.depths)):
        dr = res.depths[kid]
        agree.append((dr.pano.valid == z["valids"][j]).mean())
        both = dr.pano.valid & z["valids"][j]
        close.append((np.abs(dr.pano.depth - z["depths"][j])[both] <= 0.005 * z["depths"][j][both]).mean())
        assert not dr.pano.valid[0].any() and not dr.pano.valid[-1].any()  # pole rows never survive
    assert np.mean(agree) >= 0.995 and np.mean(close) >= 0.995, (agree, close)  # north_star's bar
    assert min(agree) >= 0.99 and min(close) >= 0.99, (agree, close)
    # ... and the CPU oracle's own run of the same chain is reproduced (measured: every map identical)
    want = oracle_chain(z)
    for kid, dr in res.depths.items():
        od, ov = want[kid]
        assert (dr.pano.valid == ov).mean() >= 0.995
        both = dr.pano.valid & ov
        assert (np.abs(dr.pano.depth - od)[both] <= 0.005 * od[both]).mean() >= 0.995
    assert abs(rep["fused_points"] - int(z["fused_points"])) <= 0.05 * int(z["fused_points"])
    assert abs(rep["completeness"]["mean"] - float(z["comp_mean"])) <= 0.003
    assert len(rep["completeness"]["per_keyframe"]) == 20 and rep["resolution"] == [64, 32]
    assert np.all(np.diff(res.cloud.source_ids) >= 0) and len(res.cloud) == rep["fused_points"]
    # the fused batches are also handed back where they were produced, in HBM: same points, written without a
    # host round trip
    assert sum(len(b) for b in res.device_batches) == len(res.cloud)
    assert np.array_equal(np.concatenate([b.points.cpu().numpy() for b in res.device_batches if len(b)]), res.cloud.points)
    # a keyframe at another resolution is brought to the working camera (LANCZOS) instead of rejected
    from paper_2211_16266_b200 import ingest
    big = [p.Keyframe(id=k.id, image=ingest.resample_image_device(k.image, 128, 64).cpu().numpy(), pose=k.pose,
                      sparse_points=k.sparse_points) for k in kfs[:8]]
    small = offline.run_offline(big, cam, **kw)
    assert small.report["keyframes_total"] == 8 and all(d.pano.depth.shape == (32, 64) for d in small.depths.values())
    # fused points back-project onto the stored filtered depth maps (tests/test_pipeline.py:311-323)
    for src in np.unique(res.cloud.source_ids):
        dr = res.depths[int(src)]
        u, v, r = pipeline.project_points(cam, dr.pose, res.cloud.points[res.cloud.source_ids == src])
        px, py = np.rint(u).astype(int) % cam.width, np.clip(np.rint(v).astype(int), 0, cam.height - 1)
        assert dr.pano.valid[py, px].all() and np.all(np.abs(r - dr.pano.depth[py, px]) <= 1e-6 * dr.pano.depth[py, px])
    # determinism, threaded == serial, seed sensitivity (tests/test_pipeline.py:325-358)
    again = offline.run_offline(kfs, cam, **kw)
    threaded = offline.run_offline(kfs, cam, threaded=True, **kw)
    for other in (again, threaded):
        assert np.array_equal(res.cloud.points, other.cloud.points) and np.array_equal(res.cloud.colors, other.cloud.colors)
        assert all(np.array_equal(res.depths[k].pano.depth, other.depths[k].pano.depth) for k in res.depths)
    other_seed = offline.run_offline(kfs, cam, **{**kw, "seed": 99})
    assert not np.array_equal(res.cloud.points, other_seed.cloud.points)
    empty = offline.run_offline([], cam, **kw)
    assert len(empty.cloud) == 0 and empty.report["keyframes_total"] == 0 and empty.report["completeness"]["per_keyframe"] == []
