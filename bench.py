#!/usr/bin/env python
"""Headline benchmark: depth maps per second at 1920x960 with 4 neighbour views.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--workload c3]

One "step" = one reference keyframe densified end to end on its GPU: luma planes of the
keyframe that enters the sliding window (each keyframe is converted once and reused by the 5
groups it takes part in), plane-map warp from the previous keyframe + random fill,
eval + I x (red, black, refine) PatchMatch passes, median outlier filter, pole mask, and the
geometric-consistency filter of the centre frame of the last 5 depth maps (BASELINE.json
configs[2], "C3").  N > 1: one process per GPU (torchrun), every rank densifies its own
keyframe sequence, no data-path collective -> weak scaling.

Prints ONE JSON line (rank 0).  `value` = keyframes of all ranks / max-over-ranks device
time with the uint8 frames already resident in HBM; `e2e` = the same through the host-array
streaming API (numpy frames in pinned memory -> StreamingDensifier.push -> numpy depth + mask)
with the copies inside the timed region.

`--impl reference` times the CPU restatement of the reference path (oracle/, C + pthreads,
all host cores) on a bounded sample of the same workload; the product arm never touches it
except for the `cpu_baseline` leg at N=1.
"""
from __future__ import annotations

import argparse
import gc
import json
import math
import os
import subprocess
import sys
import threading
import time
from collections import deque
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

METRIC = "depth maps/sec at 1920x960, 4 views"
UNIT = "maps/s"

WORKLOADS = {
    # name: (width, height, n_views, half_window, stride, iterations)
    "c1": (256, 128, 2, 5, 2, 3),
    "c2": (960, 480, 4, 3, 1, 6),
    "c3": (1920, 960, 4, 5, 2, 6),
    "c4": (3840, 1920, 6, 5, 2, 6),
}
DEPTH_RANGE = (0.5, 16.0)
SEED = 0
STEP_M = 0.15  # keyframe spacing along z
SEQ_LEN = 24  # distinct keyframes per rank; the sequence is walked back and forth


def flops_per_eval(n_samples: int, n_views: int) -> int:
    """Algorithmic FLOPs of one plane-hypothesis cost evaluation:
    F = S*(7 + 83 V) + 12 V + 6, FMA = 2, div/sqrt/rsqrt = 1."""
    return n_samples * (7 + 83 * n_views) + 12 * n_views + 6


def n_samples_of(half_window: int, stride: int) -> int:
    reach = (half_window // stride) * stride
    return (2 * reach // stride + 1) ** 2


def sequence_positions(rank: int):
    """SEQ_LEN keyframe centres on a straight line inside the 4 x 3 x 5 m box, one lane per rank."""
    z0 = -0.5 * STEP_M * (SEQ_LEN - 1)
    x = 0.35 * ((rank % 5) - 2)
    y = 0.25 * ((rank // 5) % 3 - 1)
    return [np.array([x, y, z0 + k * STEP_M]) for k in range(SEQ_LEN)]


def loop_positions(rank: int):
    """The line of sequence_positions followed by a second lane, one step to the side, walked back:
    a closed loop of 2 SEQ_LEN distinct keyframes with STEP_M between any two consecutive ones, so a
    stream of any length never meets the same position twice inside one stereo window."""
    lane_a = sequence_positions(rank)
    lane_b = [t + np.array([STEP_M, 0.0, 0.0]) for t in reversed(lane_a)]
    return lane_a + lane_b


def walk(n: int):
    """Indices 2..SEQ_LEN-3 walked back and forth, so every group has its 4 neighbours."""
    lo, hi = 2, SEQ_LEN - 3
    fwd = list(range(lo, hi + 1))
    cyc = fwd + fwd[-2:0:-1]
    return [cyc[i % len(cyc)] for i in range(n)]


# ---------------------------------------------------------------------------------------
# clock sampling (B200_PROFILING.md "clocks DURING the timed region")
# ---------------------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._thread = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                parts = [p.strip() for p in out.stdout.strip().split(",")]
                if len(parts) >= 6:
                    self.samples.append(parts)
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._thread = threading.Thread(target=self._run, daemon=True)
        self._thread.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._thread.join(timeout=10)

    def summary(self) -> dict:
        sm = sorted(int(float(s[0])) for s in self.samples if s[0].replace(".", "").isdigit())
        mx = [int(float(s[1])) for s in self.samples if s[1].replace(".", "").isdigit()]
        reasons = set()
        for s in self.samples:
            for name, val in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"), s[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------------------
# product arm
# ---------------------------------------------------------------------------------------

def run_product(args) -> dict | None:
    import torch
    import torch.distributed as dist

    import paper_2211_16266_b200 as p
    from paper_2211_16266_b200 import _lib, engine, pipeline, synth

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit(f"--gpus {args.gpus} needs torchrun (one process per GPU); WORLD_SIZE is 1")
        raise SystemExit(f"--gpus {args.gpus} does not match WORLD_SIZE={world}")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)
    _lib.load()

    W, H, V, hw, stride, iters = WORKLOADS[args.workload]
    S = n_samples_of(hw, stride)
    cam = p.EquirectCamera(W, H)
    spec = engine.PatchSpec(hw, stride, 1.2)
    scene = synth.default_scene("box")
    ccfg = pipeline.ConsistencyConfig()

    # ---- synthetic input: SEQ_LEN rendered keyframes, on the device and in pinned host memory
    poses = [p.RigidPose(np.eye(3), t) for t in sequence_positions(rank)]
    dev_imgs, host_imgs = [], []
    for pose in poses:
        img, _ = synth.render_scene_device(scene, cam, pose, dev)
        dev_imgs.append(img)
        pinned = torch.empty(img.shape, dtype=torch.uint8).pin_memory()
        pinned.copy_(img)
        host_imgs.append(pinned.numpy())
    torch.cuda.synchronize()
    kfs = [p.Keyframe(id=k, image=host_imgs[k], pose=poses[k]) for k in range(SEQ_LEN)]
    nb_order = []
    for k in range(1, V // 2 + 1):
        nb_order += [-k, k]
    if V % 2:
        nb_order.append(V // 2 + 1)

    def group_of(i):
        return p.StereoGroup(reference=kfs[i], neighbors=tuple(kfs[i + o] for o in nb_order), camera=cam)

    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    order = walk(args.warmup + args.steps)

    def make_stage():
        return pipeline.DepthStage(cam, spec, DEPTH_RANGE, iters, SEED, warp=True, precision=args.precision,
                                   init_rng="philox", device=dev, count_evals=True)

    # ---- (A) device-resident steps
    stage = make_stage()
    window = deque(maxlen=ccfg.window)

    dk_cache = {}  # keyframe index -> DeviceKeyframe (planes computed once, on first use)
    group_buffers = {}  # the group's planes live in the same memory from step to step

    def device_keyframe(idx):
        dk = dk_cache.get(idx)
        if dk is None:
            dk = dk_cache[idx] = engine.DeviceKeyframe(dev_imgs[idx], cam, dev)
            for old in [k for k in dk_cache if abs(k - idx) > V]:
                del dk_cache[old]
        return dk

    def step_device(i):
        flush_buf.zero_()  # L2 flush (256 MiB > 126 MB L2), inside the timed region
        g = group_of(i)
        prep = engine.PreparedGroup(g, spec, precision=args.precision, device=dev, buffers=group_buffers,
                                    device_keyframes=[device_keyframe(i)] + [device_keyframe(i + o) for o in nb_order])
        res = stage.process_device(prep)
        window.append(res)
        if len(window) == ccfg.window:
            c = ccfg.window // 2
            others = [(window[j].pano, window[j].pose) for j in range(ccfg.window) if j != c]
            return pipeline.consistency_filter_device(window[c].pano, window[c].pose, others, ccfg)
        return res.pano

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    for i in order[:args.warmup]:
        step_device(i)
    barrier()
    stage.workspace.n_evals.zero_()
    _lib.trace_enable(True)
    launches0 = _lib.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    gc.collect()
    gc.disable()
    with ClockSampler(local_rank) as clocks:
        barrier()
        e0.record()
        marks = []
        for i in order[args.warmup:]:
            step_device(i)
            if os.environ.get("D360_BENCH_DEBUG"):
                marks.append(torch.cuda.Event(enable_timing=True))
                marks[-1].record()
        e1.record()
        barrier()
    gc.enable()
    dev_ms = e0.elapsed_time(e1)
    if marks:
        print("device per-step gpu ms:", [round(a.elapsed_time(b), 1) for a, b in zip([e0] + marks[:-1], marks)],
              file=sys.stderr)
    launches = _lib.launch_count() - launches0
    trace = _lib.trace_summary()
    _lib.trace_enable(False)
    n_evals_counted, n_cut = (int(x) for x in stage.workspace.n_evals.tolist())

    # ---- (B) end to end through the host-array streaming API: one pinned uint8 keyframe in per
    # step (each keyframe is uploaded once and reused by the 5 groups it takes part in), one
    # consistency-filtered depth map + mask out per step
    stream = pipeline.StreamingDensifier(cam, spec, DEPTH_RANGE, iters, SEED, n_neighbors=V, warp=True,
                                         consistency=ccfg, fusion=None, precision=args.precision,
                                         init_rng="philox", device=dev)
    fill = V + ccfg.window - 1  # pushes before the first output
    n_push = fill + args.warmup + args.steps
    if n_push > SEQ_LEN:  # longer than the line: continue around the two-lane loop (second lane rendered here)
        for t in loop_positions(rank)[SEQ_LEN:]:
            pose = p.RigidPose(np.eye(3), t)
            img, _ = synth.render_scene_device(scene, cam, pose, dev)
            pinned = torch.empty(img.shape, dtype=torch.uint8).pin_memory()
            pinned.copy_(img)
            poses.append(pose)
            host_imgs.append(pinned.numpy())
        torch.cuda.synchronize()
    positions = [k % len(poses) for k in range(n_push)]
    bytes_in = bytes_out = 0
    produced = 0

    def step_host(k):
        nonlocal bytes_in, bytes_out, produced
        flush_buf.zero_()
        kf = p.Keyframe(id=k, image=host_imgs[positions[k]], pose=poses[positions[k]])
        outs = stream.push(kf)  # numpy frame in, numpy depth + mask out
        bytes_in += kf.image.nbytes
        for o in outs:
            bytes_out += o.pano.depth.nbytes + o.pano.valid.nbytes
            produced += 1

    for k in range(fill + args.warmup):
        step_host(k)
    bytes_in = bytes_out = produced = 0
    per_step, evs = [], []
    debug = bool(os.environ.get("D360_BENCH_DEBUG"))
    gc.collect()
    gc.disable()  # keep the cyclic collector out of the 0.5 s timed region
    barrier()
    t0 = time.perf_counter()
    for k in range(fill + args.warmup, n_push):
        ts = time.perf_counter()
        if debug:
            ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ea.record()
        step_host(k)
        if debug:
            eb.record()
            evs.append((ea, eb))
        per_step.append(time.perf_counter() - ts)
    barrier()
    e2e_s = time.perf_counter() - t0
    gc.enable()
    if debug:
        print("e2e per-step wall ms:", [round(x * 1e3, 1) for x in per_step], file=sys.stderr)
        print("e2e per-step gpu  ms:", [round(a.elapsed_time(b), 1) for a, b in evs], file=sys.stderr)
    if produced != args.steps:
        raise SystemExit(f"streaming leg produced {produced} depth maps in {args.steps} steps")

    # ---- reduce over ranks
    times = torch.tensor([dev_ms, e2e_s * 1e3], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(times, op=dist.ReduceOp.MAX)
    dev_ms, e2e_ms = (float(x) for x in times.tolist())

    result = None
    if rank == 0:
        P = W * H
        F = flops_per_eval(S, V)
        evals = {"eval_costs": P * args.steps, "refine": 6 * P * iters * args.steps}
        evals["red_black"] = n_evals_counted - evals["refine"]
        kinds = {}
        total_traced = sum(ms for _, ms in trace.values())
        for kind, (cnt, ms) in sorted(trace.items(), key=lambda kv: -kv[1][1]):
            kinds[kind] = {"launches": cnt, "ms_per_launch": round(ms / cnt, 4), "share": round(ms / total_traced, 4)}
        dominant = max(("red_black", "refine", "eval_costs"), key=lambda k: trace.get(k, (0, 0.0))[1])
        d_cnt, d_ms = trace[dominant]
        # The reference computes everything after lam = num / dn in float64 (numba type inference,
        # DESIGN.md "Precision"), and the 1e-4 cost parity needs (u, v) to ~1e-10 px, so the
        # binding resource is the FP64 pipe: the denominator is the DFMA peak measured in this run.
        fp64_peak = float(_lib.load().d360_measure_fma_peak(1, 20000))
        fp32_peak = float(_lib.load().d360_measure_fma_peak(0, 20000))
        # refinement evaluations decided after V - 1 views did not do the last view's share of F
        flops = {k: n * F for k, n in evals.items()}
        flops["refine"] -= n_cut * (S * 83 + 12)
        achieved = flops[dominant] / (d_ms * 1e-3) / 1e12
        traffic = None
        tf = ROOT / "profiles" / "traffic.json"
        if tf.exists():
            traffic = json.loads(tf.read_text()).get(args.workload, {}).get(dominant)
        peaks = {}
        pk = ROOT / "MEASURED_PEAKS.json"
        if pk.exists():
            peaks = json.loads(pk.read_text())
        hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
        # algorithmic HBM bytes per step: per pass 20 B/px state read + 20 B/px written, images 4 B/px
        # per frame per pass -> (1 + 3 I) passes
        passes = 1 + 3 * iters
        alg_bytes = P * (passes * (40 + 4 * (1 + V)) + 12)
        result = {
            "metric": METRIC, "value": round(world * args.steps / (dev_ms * 1e-3), 4), "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(dev_ms / args.steps, 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64/f32 mixed" if args.precision == "mixed" else "f64",
            "data": "synthetic (GPU-rendered textured box room, value-noise texture)",
            "config": {"workload": f"{args.workload}: {W}x{H} keyframe, {V} neighbour views, {S}-sample "
                                   f"{2 * hw + 1}x{2 * hw + 1} patch, {iters} iterations, warp init + median + pole "
                                   f"mask + consistency(window 5)",
                       "precision": args.precision, "top_k": engine.default_top_k(V), "init": "warp + philox fill",
                       "l2": "256 MiB memset between steps (inside the timed region); working set > L2",
                       "keyframes_per_rank": args.steps, "parallelism": f"keyframe-sharded x{world}"},
            "clocks": clocks.summary(),
            "e2e": {"value": round(world * args.steps / (e2e_ms * 1e-3), 4), "unit": UNIT,
                    "h2d_bytes_per_step": bytes_in // args.steps, "d2h_bytes_per_step": bytes_out // args.steps,
                    "ms_per_step": round(e2e_ms / args.steps, 3)},
            "gpu_launches": int(launches),
            "roofline": {"bound": "fp64", "kernel": dominant, "achieved": round(achieved, 3),
                         "peak": round(fp64_peak, 2), "unit": "TFLOP/s", "frac": round(achieved / fp64_peak, 4),
                         "traffic": traffic,
                         "peak_source": "in-run DFMA microbenchmark (MEASURED_PEAKS.json has no FP64/FP32 figure); "
                                        "not HBM- or tensor-bound, see roofline.hbm",
                         "fp32_fma_peak": round(fp32_peak, 2),
                         "flops_per_eval": F, "evals_per_launch": evals[dominant] // max(d_cnt, 1),
                         "flops_per_launch": flops[dominant] // max(d_cnt, 1),
                         "ms_per_launch": round(d_ms / d_cnt, 4),
                         "hbm": {"algorithmic_bytes_per_step": alg_bytes,
                                 "achieved_gbs": round(alg_bytes * args.steps / (dev_ms * 1e-3) / 1e9, 2),
                                 "peak_gbs": hbm_peak,
                                 "frac": round(alg_bytes * args.steps / (dev_ms * 1e-3) / 1e9 / hbm_peak, 5)}},
            "kernels": kinds,
            "evals_per_step": {k: v // args.steps for k, v in evals.items()},
            "refine_evals_cut_after_v_minus_1_views_per_step": n_cut // args.steps,
        }
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return result


# ---------------------------------------------------------------------------------------
# CPU arm: the oracle (C restatement of the reference) on a bounded sample
# ---------------------------------------------------------------------------------------

CPU_SAMPLE = {"c1": (256, 128), "c2": (320, 160), "c3": (384, 192), "c4": (384, 192)}


def render_cpu_inputs(w: int, h: int, n: int):
    """Frames for the CPU arm.  Rendered with the product's GPU renderer when a GPU is
    visible (input generation, outside every timed region), else a numpy sinusoid-textured
    box so the arm also runs on a GPU-less machine."""
    poses = [(np.eye(3), t) for t in sequence_positions(0)[:n]]
    try:
        import torch

        if torch.cuda.is_available():
            import paper_2211_16266_b200 as p
            from paper_2211_16266_b200 import synth

            cam = p.EquirectCamera(w, h)
            scene = synth.default_scene("box")
            return [synth.render_scene(scene, cam, p.RigidPose(r, t))[0] for r, t in poses], poses
    except Exception:
        pass
    ys, xs = np.mgrid[0:h, 0:w]
    lam = 2 * np.pi * (xs + 0.5) / w - np.pi
    phi = np.pi / 2 - np.pi * (ys + 0.5) / h
    d = np.stack([np.cos(phi) * np.sin(lam), -np.sin(phi), np.cos(phi) * np.cos(lam)], -1)
    half = np.array([2.0, 1.5, 2.5])
    imgs = []
    for _, t in poses:
        with np.errstate(divide="ignore", invalid="ignore"):
            tt = np.where(d > 0, (half - t) / d, (-half - t) / d)
        hit = t + d * tt.min(-1, keepdims=True)
        tex = sum(np.sin(hit @ k + ph) for k, ph in (((7.1, 3.3, 5.9), 0.3), ((13.7, 17.9, 11.3), 1.1),
                                                      ((29.0, 23.0, 31.0), 2.0)))
        g = np.clip(127.5 + 40.0 * tex, 0, 255).astype(np.uint8)
        imgs.append(np.repeat(g[..., None], 3, axis=2))
    return imgs, poses


def run_cpu(workload: str, steps: int, warmup: int, max_seconds: float = 240.0) -> dict:
    """maps/s of the CPU path, measured on a reduced-resolution sample and scaled by pixel count."""
    from oracle import d360_oracle as O

    O.build()
    cores = os.cpu_count() or 1
    O.set_threads(cores)
    W, H, V, hw, stride, iters = WORKLOADS[workload]
    w, h = CPU_SAMPLE[workload]
    imgs, poses = render_cpu_inputs(w, h, SEQ_LEN)
    nb_order = []
    for k in range(1, V // 2 + 1):
        nb_order += [-k, k]
    order = walk(warmup + steps)
    prev = None
    window = deque(maxlen=5)
    spent = []
    t_start = time.perf_counter()
    done = 0
    for n, i in enumerate(order):
        t0 = time.perf_counter()
        g = O.Group(imgs[i], [imgs[i + o] for o in nb_order], poses[i], [poses[i + o] for o in nb_order],
                    hw, stride, 1.2)
        plane, depth, valid = O.depth_stage(g, i, DEPTH_RANGE, iters, SEED, prev=prev, ref_pose=poses[i])
        prev = (*plane, poses[i])
        window.append((depth, valid, poses[i]))
        if len(window) == 5:
            c = window[2]
            O.consistency_filter(c[0], c[1], c[2], [window[j] for j in (0, 1, 3, 4)])
        dt = time.perf_counter() - t0
        if n >= warmup:
            spent.append(dt)
            done += 1
        if time.perf_counter() - t_start > max_seconds and done >= 1:
            break
    per_map_sample = float(np.mean(spent))
    scale = (W * H) / (w * h)
    value = 1.0 / (per_map_sample * scale)
    return {"value": round(value, 5), "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{done} keyframes of the same scene/config at {w}x{h} ({1 / scale:.4f} of the {W}x{H} pixels), "
                      f"{per_map_sample:.2f} s each on {cores} threads, scaled by pixel count",
            "seconds_per_sample_step": round(per_map_sample, 3), "steps_done": done}


def run_reference(args) -> dict | None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    W, H, V, hw, stride, iters = WORKLOADS[args.workload]
    S = n_samples_of(hw, stride)
    cpu = run_cpu(args.workload, args.steps, args.warmup)
    return {
        "impl": "reference", "metric": METRIC, "value": cpu["value"], "unit": UNIT, "n_gpus": args.gpus,
        "steps": cpu["steps_done"], "warmup": args.warmup, "ms_per_step": round(1e3 / cpu["value"], 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64/f32 mixed (CPU)",
        "data": "synthetic (textured box room)",
        "config": {"workload": f"{args.workload}: {W}x{H} keyframe, {V} neighbour views, {S}-sample "
                               f"{2 * hw + 1}x{2 * hw + 1} patch, {iters} iterations, warp init + median + pole "
                               f"mask + consistency(window 5)", "top_k": 2 if V > 2 else V},
        "cpu_baseline": {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": cpu["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }


def main() -> None:
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c3")
    ap.add_argument("--precision", choices=("mixed", "exact"), default="mixed")
    ap.add_argument("--no-cpu-baseline", action="store_true", help="skip the cpu_baseline leg (N=1 only)")
    args = ap.parse_args()
    if args.steps < 1 or args.warmup < 0:
        raise SystemExit("--steps must be >= 1 and --warmup >= 0")
    if args.impl == "reference":
        out = run_reference(args)
    else:
        out = run_product(args)
        if out is not None and args.gpus == 1 and not args.no_cpu_baseline:
            cpu = run_cpu(args.workload, steps=3, warmup=1, max_seconds=60.0)
            out["cpu_baseline"] = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
