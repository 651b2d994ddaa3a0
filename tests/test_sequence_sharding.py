"""Keyframe sharding: shard plans and the NCCL/gloo cloud gather.

CPU part: plan algebra + a world_size-2 gloo run of the all-gather-v.  GPU part: two shards
simulated on one GPU reproduce the single-stream cloud bit for bit (warp off)."""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


@pytest.mark.parametrize("n_results", [0, 3, 5, 6, 9, 17, 64])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_plan_shards_partition_and_halos(n_results, world):
    from paper_2211_16266_b200.sequence import plan_shards

    window, buffer = 5, 4
    plans = plan_shards(n_results, world, window, buffer)
    assert [p.rank for p in plans] == list(range(world))
    centres = [c for p in plans for c in p.centres]
    want = list(range(2, n_results - 2)) if n_results >= window else []
    assert centres == want  # contiguous, ordered, nothing lost or duplicated
    sizes = [len(p.centres) for p in plans]
    assert max(sizes) - min(sizes) <= 1
    # every depth result is computed exactly once (no halo recompute) ...
    computed = [i for p in plans for i in p.depth]
    assert computed == (list(range(n_results)) if want else [])
    for p in plans:
        have_raw = set(p.depth) | set(p.raw_halo)
        have_filtered = set(p.centres) | set(p.filtered_halo)
        assert not set(p.depth) & set(p.raw_halo) and not set(p.centres) & set(p.filtered_halo)
        for c in p.centres:  # ... and what a centre reads is either computed here or received
            assert all(j in have_raw for j in range(c - 2, c + 3))
            newer = [j for j in range(c + 1, c + buffer) if j < n_results - 2]
            assert all(j in have_filtered for j in newer)
        # halos come from the neighbouring blocks only: at most `half` before, `half` + buffer - 1 after
        assert len(p.raw_halo) <= 4 and len(p.filtered_halo) <= buffer - 1
        for f in p.raw_halo:
            assert any(f in q.depth for q in plans if q.rank != p.rank)
        for f in p.filtered_halo:
            assert any(f in q.centres for q in plans if q.rank != p.rank)


def test_plan_shards_c5_work_per_rank():
    """BASELINE config C5 (64 keyframes, 4 neighbours -> 60 depth results) on 8 GPUs: 60 / 8 depth maps
    per rank, not the 14 of a halo-recompute plan."""
    from paper_2211_16266_b200.sequence import plan_shards

    plans = plan_shards(60, 8)
    assert sorted(len(p.depth) for p in plans) == [7, 7, 7, 7, 7, 7, 9, 9]
    assert sum(len(p.depth) for p in plans) == 60
    assert max(len(p.raw_halo) + len(p.filtered_halo) for p in plans) <= 7


def _fake_batches(plan):
    """Deterministic stand-in for fused frames: frame c has (c % 5) * 7 + 1 points."""
    from paper_2211_16266_b200.pipeline import DeviceFusedCloud

    out = []
    for c in plan.centres:
        n = (c % 5) * 7 + 1
        rng = np.random.default_rng(c)
        out.append(DeviceFusedCloud(torch.from_numpy(rng.normal(size=(n, 3))),
                                    torch.from_numpy(rng.integers(0, 255, (n, 3), dtype=np.uint8)), 100 + c))
    return out


def _gloo_worker(rank, world, port, n_results, out_path):
    import torch.distributed as dist

    from paper_2211_16266_b200.sequence import gather_cloud, plan_shards

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan = plan_shards(n_results, world)[rank]
        cloud = gather_cloud(_fake_batches(plan), dst=0, device=torch.device("cpu"))
        if rank == 0:
            np.savez(out_path, points=cloud.points, colors=cloud.colors, ids=cloud.source_ids)
        else:
            assert cloud is None
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_results", [19, 6])  # 6: rank 1 owns one frame, rank 0 owns one
def test_gather_cloud_gloo_world2(tmp_path, n_results):
    import torch.multiprocessing as mp

    from paper_2211_16266_b200.sequence import gather_cloud, plan_shards

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = tmp_path / "cloud.npz"
    mp.spawn(_gloo_worker, args=(2, port, n_results, str(out)), nprocs=2, join=True)
    got = np.load(out)
    single = gather_cloud(_fake_batches(plan_shards(n_results, 1)[0]))  # no process group: local concat
    assert np.array_equal(got["points"], single.points)
    assert np.array_equal(got["colors"], single.colors)
    assert np.array_equal(got["ids"], single.source_ids)
    assert list(got["ids"]) == sorted(got["ids"])  # oldest keyframe first


class _FakeStage:
    """Stand-in for DepthStage on a machine without a GPU: frame i is a deterministic pattern."""

    def __init__(self, camera):
        self.camera, self.device = camera, torch.device("cpu")


def _fake_frame(shape, index, salt):
    g = torch.Generator().manual_seed(1000 * salt + index)
    return (torch.rand(shape, generator=g, dtype=torch.float32),
            (torch.rand(shape, generator=g) > 0.5).to(torch.uint8))


def _fake_run(plan, n_results, camera):
    import paper_2211_16266_b200 as p
    from paper_2211_16266_b200 import pipeline
    from paper_2211_16266_b200.sequence import ShardRun

    refs = [(100 + i, p.RigidPose(np.eye(3), np.array([0.0, 0.0, 0.1 * i]))) for i in range(n_results)]
    run = ShardRun([None] * n_results, plan, _FakeStage(camera), pipeline.ConsistencyConfig(), pipeline.FusionConfig(),
                   refs=refs)
    for i in plan.depth:
        run.accept_frame("raw", i, *_fake_frame(camera.shape, i, 1))
    for c in plan.centres:
        run.accept_frame("filtered", c, *_fake_frame(camera.shape, c, 2))
    return run


def _halo_worker(rank, world, port, n_results, out_dir):
    import torch.distributed as dist

    import paper_2211_16266_b200 as p
    from paper_2211_16266_b200.sequence import exchange_frames, plan_shards

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cam = p.EquirectCamera(16, 8)
        plans = plan_shards(n_results, world)
        run = _fake_run(plans[rank], n_results, cam)
        got = exchange_frames(run, plans, "raw", comm_device="cpu")
        got += exchange_frames(run, plans, "filtered", comm_device="cpu")
        frame_bytes = 16 * 8 * 5
        assert got == frame_bytes * (len(plans[rank].raw_halo) + len(plans[rank].filtered_halo))
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"),
                 **{f"raw{i}_{k}": t.numpy() for i in plans[rank].raw_halo for k, t in
                    zip("dv", run.frame_tensors("raw", i))},
                 **{f"fil{i}_{k}": t.numpy() for i in plans[rank].filtered_halo for k, t in
                    zip("dv", run.frame_tensors("filtered", i))})
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n_results", [(2, 19), (2, 7), (3, 30)])
def test_halo_exchange_gloo(tmp_path, world, n_results):
    """The two point-to-point halo exchanges over a real process group (gloo, CPU tensors): every rank
    ends up with exactly the frames its plan lists, bit for bit what their owners hold."""
    import torch.multiprocessing as mp

    import paper_2211_16266_b200 as p
    from paper_2211_16266_b200.sequence import plan_shards

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(_halo_worker, args=(world, port, n_results, str(tmp_path)), nprocs=world, join=True)
    cam = p.EquirectCamera(16, 8)
    plans = plan_shards(n_results, world)
    assert any(pl.raw_halo for pl in plans) and any(pl.filtered_halo for pl in plans)
    for pl in plans:
        z = np.load(tmp_path / f"rank{pl.rank}.npz")
        for i in pl.raw_halo:
            d, v = _fake_frame(cam.shape, i, 1)
            assert np.array_equal(z[f"raw{i}_d"], d.numpy()) and np.array_equal(z[f"raw{i}_v"], v.numpy())
        for i in pl.filtered_halo:
            d, v = _fake_frame(cam.shape, i, 2)
            assert np.array_equal(z[f"fil{i}_d"], d.numpy()) and np.array_equal(z[f"fil{i}_v"], v.numpy())


@pytest.mark.gpu
def test_two_shards_reproduce_single_stream():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2211_16266_b200 as p
    from paper_2211_16266_b200 import engine, pipeline, synth
    from paper_2211_16266_b200.sequence import gather_cloud, simulate_shards

    cam = p.EquirectCamera(64, 32)
    scene = synth.default_scene("box")
    kfs = []
    for k in range(13):
        pose = p.RigidPose(np.eye(3), np.array([0.1, 0.0, -0.6 + 0.1 * k]))
        img, _ = synth.render_scene(scene, cam, pose)
        kfs.append(p.Keyframe(id=k, image=img, pose=pose))
    groups = [p.StereoGroup(reference=kfs[i], neighbors=(kfs[i - 1], kfs[i + 1]), camera=cam) for i in range(1, 12)]
    ccfg, fcfg = pipeline.ConsistencyConfig(), pipeline.FusionConfig()

    def stage():
        return pipeline.DepthStage(cam, engine.PatchSpec(), (0.5, 8.0), 2, 0, warp=False)

    def run(world):
        cloud, runs = simulate_shards(groups, world, stage, ccfg, fcfg)
        assert sum(r.computed for r in runs) == len(groups)  # every depth map computed once
        return cloud

    one, two, three = run(1), run(2), run(3)
    assert len(one) > 0
    for other in (two, three):
        assert np.array_equal(one.points, other.points)
        assert np.array_equal(one.colors, other.colors)
        assert np.array_equal(one.source_ids, other.source_ids)
    # and it is the reference's stage C: stream the same depth results through the FIFO classes
    st = stage()
    fb = pipeline.FusionBuffer(cam, fcfg)
    window, ref_batches = [], []
    for g in groups:
        window.append(st.process_device(g))
        if len(window) == ccfg.window:
            c = window[2]
            pano = pipeline.consistency_filter_device(c.pano, c.pose, [(w.pano, w.pose) for j, w in enumerate(window) if j != 2], ccfg)
            got = fb.push_device(pipeline.DeviceDepthResult(c.id, pano, c.pose, c.image))
            if got is not None:
                ref_batches.append(got)
            window.pop(0)
    ref_batches += fb.flush_device()
    ref = gather_cloud(ref_batches)
    assert np.array_equal(one.points, ref.points) and np.array_equal(one.source_ids, ref.source_ids)


@pytest.mark.gpu
def test_c5_sequence_sharding_full_size():
    """BASELINE config C5: 64 keyframes at 1920x960 with 4 neighbour views and the C3 settings
    (6 iterations), sharded 1 / 8 ways (the 8 shards run one after the other on the one GPU, halos
    handed across): every depth map is computed once and the gathered cloud is the single-stream
    cloud bit for bit, oldest keyframe first."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2211_16266_b200 as p
    from paper_2211_16266_b200 import engine, pipeline, synth
    from paper_2211_16266_b200.sequence import simulate_shards

    cam = p.EquirectCamera(1920, 960)
    scene = synth.default_scene("corridor")
    kfs = []
    for k in range(64):
        pose = p.RigidPose(np.eye(3), np.array([0.2, -0.1, -4.7 + 0.15 * k]))
        img, _ = synth.render_scene(scene, cam, pose)
        kfs.append(p.Keyframe(id=k, image=img, pose=pose))
    groups = [p.StereoGroup(reference=kfs[i], neighbors=(kfs[i - 1], kfs[i + 1], kfs[i - 2], kfs[i + 2]), camera=cam)
              for i in range(2, 62)]
    ccfg, fcfg = pipeline.ConsistencyConfig(), pipeline.FusionConfig()

    def run(world):
        ws = {}

        def stage():  # the simulated ranks share one GPU: one workspace for all of them
            st = pipeline.DepthStage(cam, engine.PatchSpec(), (0.5, 16.0), 6, 0, warp=False, init_rng="philox")
            if "ws" in ws:
                st._ws = ws["ws"]
            ws["ws"] = st._ws
            return st

        cloud, runs = simulate_shards(groups, world, stage, ccfg, fcfg)
        assert [r.computed for r in runs] == [len(r.plan.depth) for r in runs]
        assert sum(r.computed for r in runs) == len(groups) and max(r.computed for r in runs) <= -(-len(groups) // world) + 2
        return cloud

    one, eight = run(1), run(8)
    assert len(one) > 100000
    assert np.array_equal(one.points, eight.points) and np.array_equal(one.colors, eight.colors)
    assert np.array_equal(one.source_ids, eight.source_ids)
    assert np.all(np.diff(one.source_ids) >= 0)


def _nccl_worker(rank, world, port, out_path):
    import torch.distributed as dist

    import paper_2211_16266_b200 as p
    from paper_2211_16266_b200 import engine, pipeline, synth
    from paper_2211_16266_b200.sequence import densify_sequence

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        cam, groups = _small_sequence(p, synth)
        stats = {}
        cloud, plan = densify_sequence(
            groups, lambda: pipeline.DepthStage(cam, engine.PatchSpec(), (0.5, 8.0), 2, 0, warp=False, device=dev),
            pipeline.ConsistencyConfig(), pipeline.FusionConfig(), rank=rank, world=world, stats=stats)
        assert stats["depth_maps_computed"] == len(plan.depth)
        if rank == 0:
            np.savez(out_path, points=cloud.points, colors=cloud.colors, ids=cloud.source_ids)
        dist.barrier()
    finally:
        dist.destroy_process_group()


def _small_sequence(p, synth):
    cam = p.EquirectCamera(64, 32)
    scene = synth.default_scene("box")
    kfs = []
    for k in range(13):
        pose = p.RigidPose(np.eye(3), np.array([0.1, 0.0, -0.6 + 0.1 * k]))
        img, _ = synth.render_scene(scene, cam, pose)
        kfs.append(p.Keyframe(id=k, image=img, pose=pose))
    return cam, [p.StereoGroup(reference=kfs[i], neighbors=(kfs[i - 1], kfs[i + 1]), camera=cam) for i in range(1, 12)]


@pytest.mark.gpu
def test_densify_sequence_nccl_world2(tmp_path):
    """Two ranks on two GPUs over NCCL: halo send / recv and the all-gather-v of the cloud; the result is
    the single-process cloud bit for bit.  Needs two visible GPUs (skipped on the 1-GPU boxes)."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs two CUDA devices")
    import torch.multiprocessing as mp

    import paper_2211_16266_b200 as p
    from paper_2211_16266_b200 import engine, pipeline, synth
    from paper_2211_16266_b200.sequence import simulate_shards

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = tmp_path / "cloud.npz"
    mp.spawn(_nccl_worker, args=(2, port, str(out)), nprocs=2, join=True)
    got = np.load(out)
    cam, groups = _small_sequence(p, synth)
    one, _ = simulate_shards(groups, 1, lambda: pipeline.DepthStage(cam, engine.PatchSpec(), (0.5, 8.0), 2, 0, warp=False),
                             pipeline.ConsistencyConfig(), pipeline.FusionConfig())
    assert np.array_equal(got["points"], one.points) and np.array_equal(got["colors"], one.colors)
    assert np.array_equal(got["ids"], one.source_ids)
