#!/usr/bin/env python
"""Headline benchmark: depth maps per second at 1920x960 with 4 neighbour views.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--workload c3]

One "step" = one reference keyframe densified end to end on its GPU: luma planes of the
keyframe that enters the sliding window (each keyframe is converted once and reused by the 5
groups it takes part in), plane-map warp from the previous keyframe + random fill,
eval + I x (red, black, refine) PatchMatch passes, median outlier filter, pole mask, and the
geometric-consistency filter of the centre frame of the last 5 depth maps (BASELINE.json
configs[2], "C3").  N > 1: one process per GPU (torchrun); the ranks share one sequence of N x K
depth results (BASELINE.json configs[4], "C5", at K keyframes per rank -> weak scaling) through
paper_2211_16266_b200.sequence.densify_sequence: every rank computes its block of depth maps once,
exchanges the consistency / fusion halos with its neighbours point to point over NCCL, fuses its
centres, and the cloud is gathered to rank 0 - all inside the timed region.

SM clock and throttle reasons are sampled every 0.1 s during the timed region (NVML, the library behind
nvidia-smi, in-process; the command-line tool as fallback) and reported under `clocks`.

Prints ONE JSON line (rank 0).  `value` = keyframes of all ranks / max-over-ranks device
time with the uint8 frames already resident in HBM; `e2e` = the same through the host-array
streaming API (numpy frames in pinned memory -> StreamingDensifier.push -> numpy depth + mask)
with the copies inside the timed region.

`--impl reference` times the CPU path on the box's host cores at the workload's own size: the C
port of the reference (oracle/, pthreads, all host threads) on full-resolution keyframes with the
metric's 4 neighbour views, and beside it the unmodified reference itself (baseline/_ref, numba) on
one keyframe with the 2 neighbours it supports.  Neither leg imports the product package; the
product arm touches oracle/ only for its `cpu_baseline` leg at N=1 (one full-size keyframe).
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

METRIC = "depth maps/sec at 1920x960, 4 views"  # BASELINE.json's metric (workload c3)
UNIT = "maps/s"

WORKLOADS = {
    # name: (width, height, n_views, half_window, stride, iterations)
    "c1": (256, 128, 2, 5, 2, 3),
    "c2": (960, 480, 4, 3, 1, 6),
    "c3": (1920, 960, 4, 5, 2, 6),
    "c4": (3840, 1920, 6, 5, 2, 6),
}


def metric_of(workload: str) -> str:
    """BASELINE.json's metric for c3; the other workloads name their own size and view count."""
    w, h, v = WORKLOADS[workload][:3]
    return METRIC if workload == "c3" else f"depth maps/sec at {w}x{h}, {v} views"


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
    """SM clock and throttle reasons sampled every 0.1 s during the timed region.  Through NVML in this process
    (nvidia_ml_py): spawning `nvidia-smi` ten times a second initialises the driver's management layer each time and
    can hold up kernel launches for milliseconds; the command-line tool is the fallback when NVML cannot be loaded."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._thread = None
        self._nvml = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nvml = pynvml
            self._handle = pynvml.nvmlDeviceGetHandleByIndex(index)
            self._max = pynvml.nvmlDeviceGetMaxClockInfo(self._handle, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        n = self._nvml
        sm = n.nvmlDeviceGetClockInfo(self._handle, n.NVML_CLOCK_SM)
        try:
            reasons = n.nvmlDeviceGetCurrentClocksEventReasons(self._handle)
        except Exception:
            reasons = n.nvmlDeviceGetCurrentClocksThrottleReasons(self._handle)
        flag = lambda bit: "Active" if reasons & bit else "Not Active"
        try:
            power = n.nvmlDeviceGetPowerUsage(self._handle) / 1e3
        except Exception:
            power = 0.0
        return [str(sm), str(self._max), flag(n.nvmlClocksThrottleReasonHwSlowdown),
                flag(n.nvmlClocksThrottleReasonHwThermalSlowdown), flag(n.nvmlClocksThrottleReasonSwThermalSlowdown),
                flag(n.nvmlClocksThrottleReasonSwPowerCap), f"{power:.1f}"]

    def _run(self):
        while not self._stop.is_set():
            try:
                if self._nvml is not None:
                    self.samples.append(self._sample_nvml())
                else:
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
                "reasons": sorted(reasons), "samples": len(self.samples),
                "source": "nvml" if self._nvml is not None else "nvidia-smi"}


# ---------------------------------------------------------------------------------------
# product arm
# ---------------------------------------------------------------------------------------

def roofline_block(trace, evals, n_cut, S, V, workload, P, iters, maps, dev_ms) -> dict:
    """`roofline` object of the JSON line for the dominant cost kernel of this rank.

    The reference computes everything after lam = num / dn in float64 (numba type inference,
    DESIGN.md "Precision"), and the 1e-4 cost parity needs (u, v) to ~1e-10 px, so the binding
    resource is the FP64 pipe: the denominator is the DFMA peak measured in this run (`frac`);
    `frac_fp32` is the same work against the FP32-FMA peak SURVEY.md section 8d named."""
    from paper_2211_16266_b200 import _lib

    F = flops_per_eval(S, V)
    dominant = max(("red_black", "refine", "eval_costs"), key=lambda k: trace.get(k, (0, 0.0))[1])
    d_cnt, d_ms = trace[dominant]
    fp64_peak = float(_lib.load().d360_measure_fma_peak(1, 20000))
    fp32_peak = float(_lib.load().d360_measure_fma_peak(0, 20000))
    # refinement evaluations decided after V - 1 views did not do the last view's share of F
    flops = {k: n * F for k, n in evals.items()}
    flops["refine"] -= n_cut * (S * 83 + 12)
    achieved = flops[dominant] / (d_ms * 1e-3) / 1e12
    traffic = None
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists():
        traffic = json.loads(tf.read_text()).get(workload, {}).get(dominant)
    peaks = {}
    pk = ROOT / "MEASURED_PEAKS.json"
    if pk.exists():
        peaks = json.loads(pk.read_text())
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    # algorithmic HBM bytes per map: per pass 20 B/px state read + 20 B/px written, images 4 B/px
    # per frame per pass -> (1 + 3 I) passes
    passes = 1 + 3 * iters
    alg_bytes = P * (passes * (40 + 4 * (1 + V)) + 12)
    return {"bound": "fp64", "kernel": dominant, "achieved": round(achieved, 3), "peak": round(fp64_peak, 2),
            "unit": "TFLOP/s", "frac": round(achieved / fp64_peak, 4), "traffic": traffic,
            "peak_source": "in-run DFMA microbenchmark (MEASURED_PEAKS.json has no FP64/FP32 figure; "
                           "profiles/fp_peaks.json keeps the last recorded pair); not HBM- or tensor-bound, see roofline.hbm",
            "fp32_fma_peak": round(fp32_peak, 2), "frac_fp32": round(achieved / fp32_peak, 4),
            "flops_per_eval": F, "evals_per_launch": evals[dominant] // max(d_cnt, 1),
            "flops_per_launch": flops[dominant] // max(d_cnt, 1), "ms_per_launch": round(d_ms / d_cnt, 4),
            "hbm": {"algorithmic_bytes_per_step": alg_bytes,
                    "achieved_gbs": round(alg_bytes * maps / (dev_ms * 1e-3) / 1e9, 2), "peak_gbs": hbm_peak,
                    "frac": round(alg_bytes * maps / (dev_ms * 1e-3) / 1e9 / hbm_peak, 5)}}


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
    # D360_BENCH_BACKEND=gloo: rehearsal of the N > 1 path on a box with fewer GPUs than ranks (ranks
    # share GPUs, halos and cloud staged through host memory); the measured configuration is NCCL
    backend = os.environ.get("D360_BENCH_BACKEND", "nccl")
    dev_index = local_rank if backend == "nccl" else local_rank % torch.cuda.device_count()
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "WARN")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    _lib.load()
    if world == 1 and args.sequence:
        # the N = 1 point of the C5 curve: the same sharded-sequence code on one rank (one-rank process group,
        # so the exchange / gather calls are the ones N > 1 runs; no halo exists, the gather is local)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(29500 + os.getpid() % 2000))
        dist.init_process_group(backend, rank=0, world_size=1, **({"device_id": dev} if backend == "nccl" else {}))
    if world > 1 or args.sequence:
        out = run_product_sharded(args, world, rank, dev, backend)
        dist.barrier()
        dist.destroy_process_group()
        return out

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

    # warm-up; its first keyframe has no previous map to warp from, so it is the stream's cold start (every
    # hypothesis drawn by Philox): timed on its own and reported beside the steady state
    cold = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    if args.warmup:  # one keyframe through a scratch stage first: one-time set-up (ray tables, kernel attributes, allocator)
        scratch_stage, stage = stage, make_stage()
        g0 = group_of(order[0])
        scratch_stage.process_device(engine.PreparedGroup(g0, spec, precision=args.precision, device=dev))
        del scratch_stage, g0
    for n_w, i in enumerate(order[:args.warmup]):
        if n_w == 0:
            torch.cuda.synchronize()
            cold[0].record()
        step_device(i)
        if n_w == 0:
            cold[1].record()
    barrier()
    cold_ms = cold[0].elapsed_time(cold[1]) if args.warmup else None
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
                                         init_rng="philox", device=dev, overlap=True)
    # overlap=True: pinned staging + copy stream for the frame in and the depth map out, events between the
    # stages; push() hands out the previous keyframe's output while this one's kernels are queued
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
        take(outs)

    def take(outs):
        nonlocal bytes_out, produced
        for o in outs:
            bytes_out += o.pano.depth.nbytes + o.pano.valid.nbytes
            produced += 1

    for k in range(fill + args.warmup):
        step_host(k)
    stream.drain()  # nothing in flight when the clock starts: the timed steps deliver exactly their own outputs
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
    take(stream.drain())  # the last step's depth map + mask, read back inside the timed region
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
        roofline = roofline_block(trace, evals, n_cut, S, V, args.workload, P, iters, args.steps, dev_ms)
        result = {
            "metric": metric_of(args.workload), "value": round(world * args.steps / (dev_ms * 1e-3), 4), "unit": UNIT,
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
            "generic_fallbacks": int(_lib.generic_fallbacks()),
            "cold_start": {"ms_first_keyframe": None if cold_ms is None else round(cold_ms, 3),
                           "maps_per_s": None if not cold_ms else round(1e3 / cold_ms, 3),
                           "what": "first keyframe of the stream: no previous map to warp from, every hypothesis drawn "
                                   "by Philox; `value` is the "
                                   "warp-initialised steady state the reference's stream also runs in (P:213-232)"},
            "roofline": roofline,
            "kernels": kinds,
            "evals_per_step": {k: v // args.steps for k, v in evals.items()},
            "refine_evals_cut_after_v_minus_1_views_per_step": n_cut // args.steps,
        }
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return result



def run_product_sharded(args, world: int, rank: int, dev, backend: str) -> dict | None:
    """N > 1: one sequence of world x steps depth results, sharded by keyframe (sequence.py)."""
    import torch
    import torch.distributed as dist

    import paper_2211_16266_b200 as p
    from paper_2211_16266_b200 import _lib, engine, pipeline, sequence, synth

    W, H, V, hw, stride, iters = WORKLOADS[args.workload]
    S = n_samples_of(hw, stride)
    cam = p.EquirectCamera(W, H)
    spec = engine.PatchSpec(hw, stride, 1.2)
    scene = synth.default_scene("box")
    ccfg, fcfg = pipeline.ConsistencyConfig(), pipeline.FusionConfig()
    nb_order = []
    for k in range(1, V // 2 + 1):
        nb_order += [-k, k]
    half_v = V // 2
    n_results = world * args.steps
    loop = loop_positions(0)
    n_kf = n_results + 2 * half_v

    def pose_of(j):
        return p.RigidPose(np.eye(3), loop[j % len(loop)])

    refs = [(i + half_v, pose_of(i + half_v)) for i in range(n_results)]
    plan = sequence.plan_shards(n_results, world, ccfg.window, fcfg.buffer)[rank]
    mine = range(max(0, plan.depth.start), min(n_kf, plan.depth.stop + 2 * half_v)) if len(plan.depth) else range(0)
    dev_imgs, host_imgs, pinned_imgs = {}, {}, {}
    for j in mine:  # the keyframes this rank's groups read: resident on the device and in pinned host memory
        img, _ = synth.render_scene_device(scene, cam, pose_of(j), dev)
        dev_imgs[j] = img
        pinned = torch.empty(img.shape, dtype=torch.uint8).pin_memory()
        pinned.copy_(img)
        host_imgs[j] = pinned.numpy()
        pinned_imgs[j] = pinned  # the same memory as a tensor: DeviceKeyframe copies it up asynchronously
    torch.cuda.synchronize()
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    comm_device = None if backend == "nccl" else "cpu"

    def barrier():
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()

    def run(images, stats):
        """One pass over the whole sequence from `images` (device tensors or pinned host arrays)."""
        dk_cache, buffers = {}, {}

        def device_keyframe(j):
            dk = dk_cache.get(j)
            if dk is None:
                dk = dk_cache[j] = engine.DeviceKeyframe(images[j], cam, dev)
                for old in [k for k in dk_cache if k < j - 2 * V]:
                    del dk_cache[old]
            return dk

        def group(i):
            def make():
                flush_buf.zero_()  # L2 flush between keyframes, inside the timed region
                c = i + half_v
                kfs = [p.Keyframe(id=c, image=host_imgs[c], pose=pose_of(c))] + \
                      [p.Keyframe(id=c + o, image=host_imgs[c + o], pose=pose_of(c + o)) for o in nb_order]
                g = p.StereoGroup(reference=kfs[0], neighbors=tuple(kfs[1:]), camera=cam)
                return engine.PreparedGroup(g, spec, precision=args.precision, device=dev, buffers=buffers,
                                            device_keyframes=[device_keyframe(c)] + [device_keyframe(c + o) for o in nb_order])
            return make

        groups = [group(i) for i in range(n_results)]

        def stage_factory():
            st = pipeline.DepthStage(cam, spec, DEPTH_RANGE, iters, SEED, warp=True, precision=args.precision,
                                     init_rng="philox", device=dev, count_evals=True)
            stats["stage"] = st
            return st

        return sequence.densify_sequence(groups, stage_factory, ccfg, fcfg, rank=rank, world=world, refs=refs,
                                         comm_device=comm_device, stats=stats)

    # warm-up: one untimed pass over the same sequence through the same path - kernels, the caching allocator (the pass
    # keeps ~1 GB of depth results alive; a cold allocator answers with synchronising cudaMallocs), NCCL channels
    if args.warmup:
        run(dev_imgs, {})
    tok = torch.zeros(1, device=dev if backend == "nccl" else "cpu")
    dist.all_reduce(tok)
    barrier()

    _lib.trace_enable(True)
    launches0 = _lib.launch_count()
    stats = {}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    gc.collect()
    gc.disable()
    with ClockSampler(dev.index) as clocks:
        barrier()
        e0.record()
        cloud, _ = run(dev_imgs, stats)
        e1.record()
        barrier()
    gc.enable()
    dev_ms = e0.elapsed_time(e1)
    launches = _lib.launch_count() - launches0
    trace = _lib.trace_summary()
    _lib.trace_enable(False)
    n_points = len(cloud) if cloud is not None else 0
    n_evals_counted, n_cut = (int(x) for x in stats.pop("stage").workspace.n_evals.tolist())

    stats_h = {}
    gc.collect()
    gc.disable()
    barrier()
    t0 = time.perf_counter()
    cloud_h, _ = run(pinned_imgs, stats_h)  # frames from pinned host memory, cloud to host on rank 0
    stats_h.pop("stage", None)
    barrier()
    e2e_s = time.perf_counter() - t0
    gc.enable()
    bytes_in = sum(host_imgs[j].nbytes for j in mine)
    bytes_out = (cloud_h.points.nbytes + cloud_h.colors.nbytes + cloud_h.source_ids.nbytes) if cloud_h is not None else 0

    cdev = dev if backend == "nccl" else torch.device("cpu")
    times = torch.tensor([dev_ms, e2e_s * 1e3], dtype=torch.float64, device=cdev)
    dist.all_reduce(times, op=dist.ReduceOp.MAX)
    sums = torch.tensor([stats["depth_maps_computed"], stats["halo_bytes_received"], bytes_in, bytes_out, launches],
                        dtype=torch.float64, device=cdev)
    dist.all_reduce(sums, op=dist.ReduceOp.SUM)
    dev_ms, e2e_ms = (float(x) for x in times.tolist())
    computed, halo_bytes, bytes_in, bytes_out, launches = (int(x) for x in sums.tolist())
    if rank != 0:
        return None
    kinds = {}
    total_traced = sum(ms for _, ms in trace.values()) or 1.0
    for kind, (cnt, ms) in sorted(trace.items(), key=lambda kv: -kv[1][1]):
        kinds[kind] = {"launches": cnt, "ms_per_launch": round(ms / cnt, 4), "share": round(ms / total_traced, 4)}
    mine_n = stats["depth_maps_computed"]  # rank 0's own block
    P = W * H
    evals = {"eval_costs": P * mine_n, "refine": 6 * P * iters * mine_n}
    evals["red_black"] = n_evals_counted - evals["refine"]
    roofline = roofline_block(trace, evals, n_cut, S, V, args.workload, P, iters, mine_n, dev_ms)
    return {
        "metric": metric_of(args.workload), "value": round(n_results / (dev_ms * 1e-3), 4), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dev_ms / args.steps, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64/f32 mixed" if args.precision == "mixed" else "f64",
        "data": "synthetic (GPU-rendered textured box room, value-noise texture)",
        "config": {"workload": f"c5 at {args.steps} keyframes per GPU: one sequence of {n_results} depth results at {W}x{H}, "
                               f"{V} neighbour views, {S}-sample {2 * hw + 1}x{2 * hw + 1} patch, {iters} iterations, warp init "
                               f"(restarted per shard) + median + pole mask + consistency(window 5) + fusion(buffer 4), "
                               f"keyframe-sharded with halo exchange and cloud gather inside the timed region",
                   "precision": args.precision, "top_k": engine.default_top_k(V), "init": "warp + philox fill",
                   "l2": "256 MiB memset between keyframes (inside the timed region); working set > L2",
                   "keyframes_per_rank": args.steps, "parallelism": f"keyframe-sharded x{world}", "backend": backend,
                   "depth_maps_computed_all_ranks": computed, "halo_bytes_received_all_ranks": halo_bytes,
                   "cloud_points": n_points},
        "clocks": clocks.summary(),
        "e2e": {"value": round(n_results / (e2e_ms * 1e-3), 4), "unit": UNIT,
                "h2d_bytes_per_step": bytes_in // max(n_results, 1), "d2h_bytes_per_step": bytes_out // max(n_results, 1),
                "ms_per_step": round(e2e_ms / args.steps, 3)},
        "gpu_launches": launches,
        "roofline": roofline,
        "kernels_rank0": kinds,
    }


# ---------------------------------------------------------------------------------------
# CPU arm: the oracle (C restatement of the reference) on a bounded sample
# ---------------------------------------------------------------------------------------

REF_ROOT = ROOT / "baseline" / "_ref"  # the unmodified reference, pip-installed (--target) from /root/reference/pkg


def _reference_on_path() -> bool:
    """Make the installed reference importable (it is not product code and never imported by it)."""
    if not (REF_ROOT / "densify360").is_dir():
        return False
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/d360_numba_cache")
    if str(REF_ROOT) not in sys.path:
        sys.path.insert(0, str(REF_ROOT))
    return True


def _render_one(job):
    """One frame of the benchmark scene by the reference's own renderer (synth.py:154-169), or, when the
    reference is not installed, a numpy sinusoid-textured box (same geometry)."""
    w, h, t, use_ref = job
    if use_ref:
        _reference_on_path()
        from densify360 import geometry as G, synth as SY

        img, _ = SY.render_scene(SY.default_scene("box"), G.EquirectCamera(w, h), G.RigidPose(np.eye(3), np.asarray(t)))
        return np.ascontiguousarray(img)
    ys, xs = np.mgrid[0:h, 0:w]
    lam = 2 * np.pi * (xs + 0.5) / w - np.pi
    phi = np.pi / 2 - np.pi * (ys + 0.5) / h
    d = np.stack([np.cos(phi) * np.sin(lam), -np.sin(phi), np.cos(phi) * np.cos(lam)], -1)
    half = np.array([2.0, 1.5, 2.5])
    with np.errstate(divide="ignore", invalid="ignore"):
        tt = np.where(d > 0, (half - t) / d, (-half - t) / d)
    hit = t + d * tt.min(-1, keepdims=True)
    tex = sum(np.sin(hit @ k + ph) for k, ph in (((7.1, 3.3, 5.9), 0.3), ((13.7, 17.9, 11.3), 1.1),
                                                  ((29.0, 23.0, 31.0), 2.0)))
    g = np.clip(127.5 + 40.0 * tex, 0, 255).astype(np.uint8)
    return np.repeat(g[..., None], 3, axis=2)


def render_cpu_inputs(w: int, h: int, indices):
    """Frames of the product arm's scene for the CPU arm, rendered on the host cores (one process per
    frame; ~11 s per 1920x960 frame with the reference's renderer) outside every timed region.  The
    product's GPU renderer reproduces these bytes for identity rotations (tests/test_gpu_parity.py), so
    both arms see the same images; the product package is not imported here."""
    import multiprocessing as mp

    use_ref = _reference_on_path()
    pos = sequence_positions(0)
    jobs = [(w, h, pos[i], use_ref) for i in indices]
    with mp.get_context("spawn").Pool(min(len(jobs), os.cpu_count() or 1)) as pool:
        imgs = pool.map(_render_one, jobs)
    return dict(zip(indices, imgs)), ("reference synth.render_scene" if use_ref else "numpy sinusoid box")


def time_reference_v2(imgs, order, w, h, hw, stride, iters) -> dict | None:
    """The reference's own numba path (engine.run_patchmatch, E:529-631) on one full-resolution keyframe
    with its 2 neighbours (the only neighbourhood it accepts, keyframes.py:47-49), all host cores,
    after a JIT warm-up on a small image."""
    if not _reference_on_path():
        return None
    try:
        import numba
        from densify360 import engine as E, geometry as G, keyframes as KF
    except Exception as exc:  # numba / Pillow missing on this host
        return {"unavailable": f"{type(exc).__name__}: {exc}"}
    cores = os.cpu_count() or 1
    pos = sequence_positions(0)

    def group(cam, i, crop=None):
        def kf(j):
            im = imgs[j] if crop is None else np.ascontiguousarray(imgs[j][::crop, ::crop])
            return KF.Keyframe(id=j, image=im, pose=G.RigidPose(np.eye(3), pos[j]))
        return KF.StereoGroup(reference=kf(i), neighbors=(kf(i - 1), kf(i + 1)), camera=cam)

    spec = E.PatchSpec(hw, stride, 1.2)
    small = G.EquirectCamera(w // 8, h // 8)
    i = order[0]
    init = E.random_init(E.PlaneMap.empty(small, DEPTH_RANGE), DEPTH_RANGE, SEED + i)
    E.run_patchmatch(group(small, i, 8), init, spec, 1, SEED + i, workers=cores)  # JIT
    cam = G.EquirectCamera(w, h)
    g = group(cam, i)
    init = E.random_init(E.PlaneMap.empty(cam, DEPTH_RANGE), DEPTH_RANGE, SEED + i)
    t0 = time.perf_counter()
    E.run_patchmatch(g, init, spec, iters, SEED + i, workers=cores)
    dt = time.perf_counter() - t0
    return {"seconds_per_map": round(dt, 2), "maps_per_s": round(1.0 / dt, 5), "views": 2,
            "threads": int(numba.get_num_threads()), "what": f"densify360.engine.run_patchmatch {w}x{h}, 2 neighbours, "
            f"{iters} iterations, random init, numba {numba.__version__}"}


def run_cpu(workload: str, steps: int, warmup: int, max_seconds: float = 200.0, with_reference: bool = True) -> dict:
    """maps/s of the CPU path at the workload's own size and view count: the C port of the reference
    (oracle/, pthreads over rows, all host threads, -O3 -march=native timing build) runs the same chain
    as the product arm (warp init + PatchMatch + median + pole mask + consistency) on full-resolution
    keyframes for as many steps as `max_seconds` allows (at least one timed keyframe, never a scaled
    crop).  The reference's own numba path is timed beside it on one keyframe with 2 neighbours."""
    from oracle import d360_oracle as O

    O.use_timing_build()
    cores = os.cpu_count() or 1
    O.set_threads(cores)
    W, H, V, hw, stride, iters = WORKLOADS[workload]
    nb_order = []
    for k in range(1, V // 2 + 1):
        nb_order += [-k, k]
    order = walk(max(1, warmup) + steps)
    # the chain visits consecutive keyframes: render only what the affordable steps can reach
    reach = min(len(order), 2 + int(max_seconds // 8))
    need = sorted({i + o for i in order[:reach] for o in [0] + nb_order})
    t_r = time.perf_counter()
    imgs, renderer = render_cpu_inputs(W, H, need)
    render_s = time.perf_counter() - t_r
    poses = {i: (np.eye(3), sequence_positions(0)[i]) for i in need}
    prev = None
    window = deque(maxlen=5)
    spent = []
    t_start = time.perf_counter()
    n_warm = 1 if warmup >= 1 else 0  # one untimed keyframe: page-in, thread pool, first warp source
    for n, i in enumerate(order[:reach]):
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
        if n >= n_warm:
            spent.append(dt)
        if spent and time.perf_counter() - t_start + dt > max_seconds:
            break
        if len(spent) >= steps:
            break
    per_map = float(np.mean(spent))
    out = {"value": round(1.0 / per_map, 5), "unit": UNIT, "cores": cores, "kind": "port",
           "sample": f"{len(spent)} full-size keyframe(s) of the same scene and config ({W}x{H}, {V} neighbour views, "
                     f"{iters} iterations, warp init + median + pole mask + consistency), {per_map:.1f} s each on {cores} "
                     f"threads after {n_warm} untimed one; frames by {renderer} ({render_s:.0f} s, untimed)",
           "seconds_per_sample_step": round(per_map, 3), "steps_done": len(spent), "warmup_done": n_warm}
    if with_reference:
        ref = time_reference_v2(imgs, order, W, H, hw, stride, iters)
        if ref is not None:
            out["reference_numba_v2"] = ref
    return out


def run_reference(args) -> dict | None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    W, H, V, hw, stride, iters = WORKLOADS[args.workload]
    S = n_samples_of(hw, stride)
    cpu = run_cpu(args.workload, args.steps, args.warmup)
    base = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
    if "reference_numba_v2" in cpu:
        base["reference_numba_v2"] = cpu["reference_numba_v2"]
    return {
        "impl": "reference", "metric": metric_of(args.workload), "value": cpu["value"], "unit": UNIT, "n_gpus": args.gpus,
        "steps": cpu["steps_done"], "warmup": cpu["warmup_done"], "ms_per_step": round(1e3 / cpu["value"], 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64/f32 mixed (CPU)",
        "data": "synthetic (textured box room, value-noise texture)",
        "config": {"workload": f"{args.workload}: {W}x{H} keyframe, {V} neighbour views, {S}-sample "
                               f"{2 * hw + 1}x{2 * hw + 1} patch, {iters} iterations, warp init + median + pole "
                               f"mask + consistency(window 5)", "top_k": 2 if V > 2 else V,
                   "steps_requested": args.steps, "note": "full-size keyframes until the time budget; `steps` = done"},
        "cpu_baseline": base,
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
    ap.add_argument("--sequence", action="store_true",
                    help="N = 1 only: run the sharded-sequence path of N > 1 (BASELINE config C5: depth maps + consistency + "
                         "fusion + cloud gather over one sequence of --steps results) on the single GPU")
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
            cpu = run_cpu(args.workload, steps=1, warmup=0, max_seconds=30.0, with_reference=False)
            out["cpu_baseline"] = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
