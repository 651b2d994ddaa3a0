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
    for p in plans:
        for c in p.centres:
            newer = [j for j in range(c + 1, c + buffer) if j < n_results - 2]
            assert all(j in p.filtered for j in [c, *newer])
        for f in p.filtered:
            assert all(j in p.depth for j in range(f - 2, f + 3))
        assert all(0 <= j < n_results for j in p.depth)


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


@pytest.mark.gpu
def test_two_shards_reproduce_single_stream():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2211_16266_b200 as p
    from paper_2211_16266_b200 import engine, pipeline, synth
    from paper_2211_16266_b200.sequence import densify_shard, gather_cloud, plan_shards

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
        batches = []
        for plan in plan_shards(len(groups), world):
            batches += densify_shard(groups, plan, stage(), ccfg, fcfg)
        return gather_cloud(batches)

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
    """BASELINE config C5: 64 keyframes at 1920x960 with 4 neighbour views, sharded 1 / 8 ways
    (the 8 shards run one after the other on the one GPU): the gathered cloud is the
    single-stream cloud bit for bit, oldest keyframe first."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2211_16266_b200 as p
    from paper_2211_16266_b200 import engine, pipeline, synth
    from paper_2211_16266_b200.sequence import densify_shard, gather_cloud, plan_shards

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
        clouds = []
        for plan in plan_shards(len(groups), world):
            stage = pipeline.DepthStage(cam, engine.PatchSpec(), (0.5, 16.0), 1, 0, warp=False, init_rng="philox")
            clouds.append(gather_cloud(densify_shard(groups, plan, stage, ccfg, fcfg)))
        return pipeline.FusedCloud.concat(clouds)

    one, eight = run(1), run(8)
    assert len(one) > 100000
    assert np.array_equal(one.points, eight.points) and np.array_equal(one.colors, eight.colors)
    assert np.array_equal(one.source_ids, eight.source_ids)
    assert np.all(np.diff(one.source_ids) >= 0)
