#!/usr/bin/env python
"""Benchmark of the stereo Whitted hot path (BASELINE.json metric on configs[3] = C4).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C4]
                    [--inflight F] [--gather peer|nccl] [--no-e2e] [--no-cpu-baseline]

One "step" = one stereo frame of the whole hot path: primary rays,
LBVH traversal + intersection, shading with shadow rays, reflection/refraction to max_depth,
pack to RGBA8, and for N>1 the assembly of every rank's tiles in rank 0's framebuffers inside
the library (rt_dist_init: fused peer stores over NVLink by default, or NCCL gather + root
unpack with --gather nccl).
The scene (upload + LBVH build, a1-a2) is resident before the timed region; its cost is
reported separately as scene_upload_ms.  Two timed regions: one frame at a time (latency and
the kernel's own duration, L2 flushed before each frame outside the events) and the throughput
loop behind `value` (F = 4 frames in flight on 4 streams, L2 flush per frame inside the timed
region).  Multi-GPU: launched by torchrun, one process per GPU, image tiles sharded across ranks
(strong scaling: the frame is fixed), device-timed, max over ranks.

Rank 0 prints ONE JSON line.  `--impl reference` times the CPU oracle (oracle/, brute force,
double precision) on bounded pixel samples of the same workload instead.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1702_01530_b200 import scenes  # noqa: E402

METRIC = "Mrays/s and stereo frames/s at 1/2/4/8 B200; % FP32 roofline"
UNIT = "Mrays/s"
# Algorithmic FP32 flops per counted unit (frozen; FMA = 2).
# The slab test is counted per REAL child box tested (box_tests, instrumented build), not as 4 per
# BVH4 node visit: empty child slots hold inverted boxes that the layout tests for free.
FLOPS_PER = {"primary": 20, "ray_setup": 3, "box_tests": 12, "tri_tests": 44, "sphere_tests": 18,
             "plane_tests": 12, "shade_hits": 20, "light_evals": 67, "reflection": 16, "refraction": 24,
             "misses": 6, "pixels": 9}
FP32_LANES_PER_SM = 128      # B200 SM: 4 SMSPs x 32 FP32 lanes
L2_FLUSH_MIN = 160 << 20     # > the 126.5 MiB L2 of a B200


def l2_flush_bytes(dev):
    """A write of 1.25x the device's L2 (at least 160 MiB) evicts every line of the scene."""
    import torch
    l2 = int(getattr(torch.cuda.get_device_properties(dev), "L2_cache_size", 0) or 0)
    return max(L2_FLUSH_MIN, ((l2 * 5 // 4) + (1 << 20) - 1) >> 20 << 20)


def algorithmic_flops(c):
    rays = c["primary"] + c["reflection"] + c["refraction"] + c["shadow"]
    f = FLOPS_PER["ray_setup"] * rays
    for k, v in FLOPS_PER.items():
        if k != "ray_setup":
            f += v * c[k]
    return float(f)


def workload_desc(s):
    return (f"{s.name}: {s.width}x{s.height} per eye stereo pair, {s.n_tris} triangles + {s.n_spheres} spheres + "
            f"{s.n_planes} planes via LBVH, {len(s.lights)} point lights, depth {s.max_depth}")


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock + throttle reasons sampled every 10 ms (NVML) during the timed region."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown"}

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = 0
        self.stop_ev = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            self.ok = True
        except Exception as e:  # noqa: BLE001
            self.err = str(e)

    def _run(self):
        nv = self.nv
        while not self.stop_ev.is_set():
            try:
                self.samples.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
                self.reasons |= int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.01)

    def start(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()

    def stop(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [f"nvml unavailable: {self.err}"]}
        self.stop_ev.set()
        self.t.join(timeout=2)
        names = sorted(n for bit, n in self.REASONS.items() if self.reasons & bit)
        return {"sm_mhz": float(np.median(self.samples)) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": names, "samples": len(self.samples), "source": "nvml, 10 ms"}


# ------------------------------------------------------------------------------ CPU oracle legs
def oracle_sample(scene, n_per_eye, seed, threads, keep=None):
    from oracle.oracle import Oracle
    pix = scenes.sample_pixels(scene.width, scene.height, n_per_eye, seed)
    o = Oracle(scene)
    t0 = time.perf_counter()
    out = o.render(pixels=pix, flags=False, threads=threads)
    dt = time.perf_counter() - t0
    if keep is not None:
        keep.update(out=out, pix=pix)
    return int(out["counts"].sum()), dt, len(pix)


def sample_agreement(gpu, keep):
    """Raw agreement of the GPU frame with the oracle on the timed sample (no fragile-pixel
    exclusion: the north-star criteria with exclusions are the GPU tests' job)."""
    out, pix = keep["out"], keep["pix"]
    e, x, y = pix[:, 0], pix[:, 1], pix[:, 2]
    gid = gpu["id"][e, y, x]
    d8 = np.abs(gpu["fb"][e, y, x][:, :3].astype(int) - out["rgba8"].reshape(-1, 4)[:, :3].astype(int)).max(1)
    err = np.abs(np.clip(gpu["radiance"][e, y, x][:, :3].astype(np.float64), 0, 1)
                 - np.clip(out["radiance"].reshape(-1, 3), 0, 1)).max(1)
    return {"pixels": int(len(pix)), "id_equal_frac": float((gid == out["id"].reshape(-1)).mean()),
            "rgb_within_2_frac": float((d8 <= 2).mean()), "max_abs_radiance_err": float(err.max()),
            "p999_abs_radiance_err": float(np.quantile(err, 0.999)),
            "note": "raw, on the cpu_baseline sample, fragile pixels included"}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(scene, target_s=15.0, seed=99, gpu=None):
    """The oracle as it stands, timed on this host's cores on a bounded pixel sample (and, given
    the GPU's full frame, the raw agreement of the two on that sample)."""
    threads = os.cpu_count() or 1
    rays, dt, n = oracle_sample(scene, max(8, threads), seed, threads)   # calibration (every thread busy)
    per_px = dt / n
    n_eye = int(max(8, min(4096, target_s / max(per_px, 1e-9) / 2)))
    keep = {}
    rays, dt, n = oracle_sample(scene, n_eye, seed + 1, threads, keep)
    if dt < 0.5 * target_s and n_eye < 4096:                    # the calibration overestimated a pixel
        n_eye = int(min(4096, n_eye * target_s / max(dt, 1e-3)))
        keep = {}
        rays, dt, n = oracle_sample(scene, n_eye, seed + 1, threads, keep)
    # single-core rate on a smaller sample (SURVEY §8(d) "also report 1-core numbers")
    per_px = dt / n
    n1 = int(max(2, min(n_eye, target_s / 3 / max(per_px * threads, 1e-9) / 2)))
    r1, d1, _ = oracle_sample(scene, n1, seed + 2, 1)
    return {"value": rays / dt / 1e6, "unit": UNIT, "cores": threads, "kind": "oracle",
            "cpu_model": cpu_model(), "one_core_value": r1 / d1 / 1e6,
            "one_core_sample": f"{2 * n1} seeded pixels, 1 thread, {d1:.1f} s",
            "sample": f"{n} seeded pixels ({n // 2} per eye) of {scene.name} {scene.width}x{scene.height} stereo, "
                      f"depth {scene.max_depth}: {rays} rays in {dt:.1f} s (double precision, brute force, "
                      f"OpenMP {threads} threads)",
            "frame_s_extrapolated": dt / n * 2 * scene.width * scene.height,
            **({"gpu_agreement": sample_agreement(gpu, keep)} if gpu is not None else {})}


def run_reference(args, scene):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0                      # under torchrun only rank 0 runs the CPU reference
    threads = os.cpu_count() or 1
    budget = 150.0 / max(1, args.steps + args.warmup)              # seconds per step
    _, dt, n = oracle_sample(scene, 4, 7, threads)
    n_eye = int(max(2, min(4096, budget / max(dt / n, 1e-9) / 2)))
    for w in range(args.warmup):
        oracle_sample(scene, max(1, n_eye // 4), 100 + w, threads)
    rays_tot, t_tot = 0, 0.0
    for k in range(args.steps):
        r, dt, _ = oracle_sample(scene, n_eye, 1000 + k, threads)
        rays_tot += r
        t_tot += dt
    val = rays_tot / t_tot / 1e6
    ms = t_tot / max(1, args.steps) * 1e3
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded scene generator)",
            "config": {"workload": workload_desc(scene), "width": scene.width, "height": scene.height,
                       "max_depth": scene.max_depth, "step": f"{2 * n_eye} seeded pixels (bounded sample)"},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": f"{2 * n_eye} seeded pixels per step of {scene.name}, {args.steps} steps"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------ GPU leg
def run_ours(args, scene):
    import torch
    import torch.distributed as dist

    from paper_1702_01530_b200 import multigpu, rt

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    # RT_BENCH_SHARE_DEVICE=1 (tests only): every rank on cuda:0 with a gloo process group, so the
    # multi-rank path (peer-store frames, barriers, max over ranks, e2e) runs on a one-GPU box
    share = os.environ.get("RT_BENCH_SHARE_DEVICE") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    W, H, D = scene.width, scene.height, scene.max_depth
    R = rt.StereoRenderer(local)
    t0 = time.perf_counter()
    info = R.upload(scene)
    upload_ms = (time.perf_counter() - t0) * 1e3
    R.set_camera(scene.rig)
    shard = (rank, world)

    # ---- instrumented (untimed) pass: ray and work counts of this rank's shard
    out = R.render(W, H, D, fb=False, count=True, shard=shard)
    torch.cuda.synchronize()
    cnt = R.counters_dict(out["counters"])
    cvec = torch.tensor([cnt[k] for k in rt.COUNTER_NAMES], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(cvec)
    tot = dict(zip(rt.COUNTER_NAMES, cvec.cpu().numpy().astype(np.int64).tolist()))
    rays_total = tot["primary"] + tot["reflection"] + tot["refraction"] + tot["shadow"]
    my_flops = algorithmic_flops(cnt)

    # ---- frame assembly (a7) inside the library for N>1: every rank joins the world (Python only
    # broadcasts the job id); a frame render then traces this rank's tiles and rank 0's
    # framebuffers receive the whole frame (peer stores over NVLink, or NCCL gather + unpack)
    dist_info = multigpu.join_world(R, rank, world, dist, args.gather) if world > 1 else \
        {"rank": 0, "world": 1, "transport": "none"}
    flush_bytes = l2_flush_bytes(dev)
    flush = torch.empty(flush_bytes // 4, dtype=torch.float32, device=dev)
    # frames in flight: F framebuffer slots on rank 0 and F streams per rank
    F = max(1, args.inflight)
    fbs = [R.alloc_fb(W, H) if rank == 0 else None for _ in range(F)]
    frames = [multigpu.Frame(R, fbs[i], W, H) for i in range(F)]
    frame = frames[0]
    streams = [torch.cuda.Stream(device=dev) for _ in range(F)]

    for _ in range(max(3, args.warmup)):
        frame.render(D)
    torch.cuda.synchronize()
    barrier()

    # ---- (1) frame latency: one frame at a time, L2 flushed before each (untimed); the trace
    # kernel's own duration per launch (roofline) and the frame time a single frame sees
    ev_s = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev_k = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]   # after the trace kernel
    ev_e = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    clk = ClockSampler(local)
    clk.start()
    barrier()
    torch.cuda.synchronize()
    for k in range(args.steps):
        flush.zero_()                                          # L2 flush between timed steps (untimed)
        ev_s[k].record()
        frame.render(D)                                        # N>1, rank 0: + the wait for every rank
        ev_k[k].record()
        ev_e[k].record()
    torch.cuda.synchronize()
    barrier()
    step_ms = np.array([ev_s[k].elapsed_time(ev_e[k]) for k in range(args.steps)])
    kern_ms = np.array([ev_s[k].elapsed_time(ev_k[k]) for k in range(args.steps)])
    t = torch.tensor([step_ms.sum(), kern_ms.mean(), np.median(step_ms), step_ms.min()], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    lat_total_ms = float(t[0])
    med_ms, best_ms = float(t[2]), float(t[3])

    # ---- (2) throughput: K frames with F in flight on F streams (rt_render_stereo_async), the
    # L2 flush (1.25x L2 write) enqueued before every frame on its own stream and timed with it
    # (it overlaps the other frames, so it cannot be left out).  A frame's pixel trees end in a
    # latency-bound tail (the deepest trees: ~0.7 ms for C4 even on an idle GPU);
    # frames in flight fill the SMs that tail would leave idle.  For N>1 the library orders the
    # frames across ranks on the device (rank 0 posts "slot free" before a frame, the other ranks
    # wait for it and post their completion; rank 0's stream waits for every post), so the host
    # just enqueues.
    if F > 1:
        def pipe_step(k):
            slot = k % F
            with torch.cuda.stream(streams[slot]):
                flush.zero_()
            frames[slot].render(D, streams[slot])

        for k in range(max(3, args.warmup)):
            pipe_step(k)
        torch.cuda.synchronize()
        barrier()
        t_start = torch.cuda.Event(enable_timing=True)
        t_start.record()
        for x in streams:
            x.wait_event(t_start)
        for k in range(args.steps):
            pipe_step(k)
        t_end = []
        for x in streams:
            e = torch.cuda.Event(enable_timing=True)
            e.record(x)
            t_end.append(e)
        torch.cuda.synchronize()
        barrier()
        total_ms = max(t_start.elapsed_time(e) for e in t_end)
        tt = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt[0])
    else:
        total_ms = lat_total_ms
    clocks = clk.stop()
    ms_per_step = total_ms / args.steps

    # ---- end-to-end through the public C ABI with host buffers (camera in, frame out)
    e2e = run_e2e(args, R, scene, rank, world, frames, fbs, streams, dev, rays_total) if not args.no_e2e else None

    # ---- machine ceilings measured live (B0): FFMA / FFMA2 / FMNMX rates and the
    # L1 / shared-memory bandwidth per SM per clock (rt_bench_ceilings), and the FFMA peak
    ffma_tflops, _ = rt.rt_bench_ffma(R.ctx, 2048)
    ceil = rt.rt_bench_ceilings(R.ctx)

    if rank == 0:
        value = rays_total / (ms_per_step * 1e-3) / 1e6
        sm_max = clocks.get("sm_max_mhz") or 1965.0
        peak = 148 * FP32_LANES_PER_SM * 2 * sm_max * 1e6 / 1e12
        # the dominant kernel's own duration: the event-timed trace launch of the one-frame-at-a-time
        # loop (L2 flushed before it); the in-flight loop overlaps 4 launches, so its per-frame time
        # is a throughput, not a launch duration, and is reported separately
        kernel_ms = float(t[1])
        achieved = my_flops / (kernel_ms * 1e-3) / 1e12
        achieved_inflight = my_flops / (ms_per_step * 1e-3) / 1e12
        traffic = load_traffic(scene.name, world)
        prof = load_profile(scene.name, world)
        par = f"tile-sharded x{world}" + {"none": "", "peer": " + fused peer-store assembly on rank 0 inside the library "
                                                              "(rt_dist_init: CUDA IPC over NVLink, device-side flags)",
                                          "nccl": " + NCCL gather to rank 0 + unpack inside the library (rt_dist_init)"}[
            dist_info["transport"]]
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": f"synthetic (seeded generator, scene sha256 {scene.sha256()[:16]})",
            "config": {"workload": workload_desc(scene), "width": W, "height": H, "max_depth": D,
                       "triangles": scene.n_tris, "rays_per_step": rays_total,
                       "rays_by_type": {k: tot[k] for k in ("primary", "reflection", "refraction", "shadow")},
                       "parallelism": par, "gather": dist_info["transport"] if world > 1 else "single",
                       "frames_in_flight": F,
                       "l2": (f"flushed ({flush_bytes >> 20} MiB write, 1.25x L2) before every timed frame, on the "
                              "frame's stream and inside the timed region" if F > 1
                              else f"flushed ({flush_bytes >> 20} MiB write) between timed steps")
                             + f"; scene+BVH {info['device_bytes'] / 1e6:.0f} MB"},
            "stereo_fps": 1e3 / ms_per_step,
            "value_definitions": {
                "value": "whole-job throughput: rays of K frames / device time of the K frames with 4 frames in "
                         "flight (L2 flushed before each, inside the timed region)",
                "frame_latency.mrays_s_median": "SURVEY §8(d) Mrays/s: rays per frame / median time of one frame "
                                                "rendered alone (L2 flushed before it, untimed)"},
            "frame_latency": {"ms_mean": lat_total_ms / args.steps, "ms_median": med_ms, "ms_best": best_ms,
                              "mrays_s": rays_total / (lat_total_ms / args.steps * 1e-3) / 1e6,
                              "mrays_s_median": rays_total / (med_ms * 1e-3) / 1e6,
                              "stereo_fps_median": 1e3 / med_ms,
                              "note": "one frame at a time, L2 flushed before each (untimed)"},
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "k_trace_stereo", "kernel_ms": kernel_ms,
                         "kernel_ms_basis": "mean event-timed duration of the trace launch, one frame at a time",
                         "kernel_share_of_step": kernel_ms / (lat_total_ms / args.steps),
                         "algorithmic_flops_per_launch": my_flops,
                         "flops_basis": "SURVEY §8(d) frozen per-unit flops x this launch's instrumented counts "
                                        "(box_tests = real child boxes tested)",
                         "inflight": {"ms_per_frame": ms_per_step, "achieved": achieved_inflight,
                                      "frac": achieved_inflight / peak,
                                      "note": "4 launches overlap: per-frame throughput time, not a launch duration"},
                         "peak_basis": f"148 SM x 128 FP32 lanes x 2 x {sm_max:.0f} MHz (sm_max; B200_PROFILING "
                                       f"unit counts); live FFMA microbenchmark {ffma_tflops:.1f} TFLOP/s",
                         "ceilings_b0": ceil,
                         **l1_roofline(prof, ceil, kernel_ms, sm_max)},
            "clocks": clocks,
            # our kernels per frame in the throughput region: the trace kernel; N>1 on rank 0 also
            # the slot post and the completion wait (peer transport) or the unpack (NCCL)
            "gpu_launches": args.steps * (1 if world == 1 else (3 if dist_info["transport"] == "peer" else 2)),
            "paper_context": {"hardware": "'a video graphics card NVIDIA', model unstated (PAPER.md:66)",
                              "timings": "no Mrays/s or frames/s published; 'few milliseconds' per frame for scenes of "
                                         "1-6 small polyhedra and one light (PAPER.md:104); ~60 % compute / up to 40 % "
                                         "CPU<->GPU transfer (PAPER.md:15, :106-107); (4:1) network 2.5x faster than "
                                         "(1:1) (PAPER.md:109)", "note": "context, not the target (BASELINE.md)"},
            "scene_upload_ms": upload_ms, "bvh": info,
            "work_counts": tot,
        }
        if e2e is not None:
            line["e2e"] = e2e
        if not args.no_cpu_baseline and world == 1:
            # the GPU's full frame (untimed, ids + radiance), compared with the oracle on the
            # baseline's own sample
            g = R.render(W, H, D, want_id=True, want_radiance=True)
            torch.cuda.synchronize()
            gpu = {k: v.cpu().numpy() for k, v in g.items()}
            line["cpu_baseline"] = cpu_baseline(scene, target_s=args.cpu_seconds, gpu=gpu)
        print(json.dumps(line), flush=True)
    if world > 1:
        rt.rt_dist_finalize(R.ctx)
        dist.barrier()
        dist.destroy_process_group()
    R.close()
    return 0


def run_e2e(args, R, scene, rank, world, frames, fbs, streams, dev, rays_total):
    """Same metric through the public C ABI: every step sets the camera from host values
    (rt_set_stereo_camera), renders (for N>1 the library assembles the frame on rank 0) and rank 0
    downloads the finished stereo frame into pinned host memory (rt_download_after on the copy
    stream, ordered after the frame's stream -- after the completion wait for every rank --
    and overlapped with the frames still rendering).  With F frames in flight each frame renders
    on its slot's stream into its slot's framebuffers; rank 0 re-renders a slot only after the
    slot's previous download completed (host wait), which the other ranks follow on the device."""
    import ctypes

    import torch

    from paper_1702_01530_b200 import rt

    W, H, D = scene.width, scene.height, scene.max_depth
    F = len(frames)
    nbytes = 2 * H * W * 4
    hosts = [rt.rt_host_alloc(nbytes) for _ in range(F)] if rank == 0 else []
    # C5: sustained camera orbit, frame k uses orbit camera k mod 60; the rays of
    # every orbit frame are counted up front (instrumented pass, untimed)
    orbit = scene.name.startswith("C5")
    n_rig = 60 if orbit else 1
    rigs = [scenes.c5_rig(k) for k in range(n_rig)] if orbit else [scene.rig]
    rays_of = [rays_total] * n_rig
    if orbit:
        for k, rg in enumerate(rigs):
            R.set_camera(rg)
            out = R.render(W, H, D, fb=False, count=True, shard=(rank, world))
            torch.cuda.synchronize()
            c = R.counters_dict(out["counters"])
            v = torch.tensor([c["primary"] + c["reflection"] + c["refraction"] + c["shadow"]], dtype=torch.float64,
                             device=dev)
            if world > 1:
                import torch.distributed as dist
                dist.all_reduce(v)
            rays_of[k] = int(v.item())
    if world > 1:
        import torch.distributed as dist
    pending = [None] * F

    def frame_step(k):
        slot = k % F
        if rank == 0 and pending[slot] is not None:
            rt.rt_wait(pending[slot])                          # the slot's previous frame is on the host
            pending[slot] = None
        rig = rigs[k % n_rig]
        rt.rt_set_stereo_camera(R.ctx, rig.eye, rig.look_at, rig.up, rig.vfov_deg, rig.interocular,
                                rig.convergence)
        st = streams[slot] if F > 1 else None
        frames[slot].render(D, st)
        if rank == 0:
            pending[slot] = rt.rt_download_after(R.ctx, fbs[slot].data_ptr(), hosts[slot], nbytes,
                                                 st.cuda_stream if st is not None else None)

    def drain():
        for i in range(F):
            if pending[i] is not None:
                rt.rt_wait(pending[i])
                pending[i] = None

    for k in range(max(3, args.warmup)):
        frame_step(k)
    drain()
    rt.rt_synchronize(R.ctx)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for k in range(args.steps):
        frame_step(k)
    drain()
    rt.rt_synchronize(R.ctx)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    tt = torch.tensor([dt], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    dt = float(tt[0])
    # paper-structure stage split (PAPER.md:15, :106-107 -- ~60 % compute / up to 40 % transfer on
    # the paper's GPU): serialised render vs download times of one frame on this box
    stages = None
    fb = fbs[0]
    if rank == 0 and world == 1:
        rt.rt_synchronize(R.ctx)
        t0 = time.perf_counter()
        for _ in range(5):
            rt.rt_wait(rt.rt_download(R.ctx, fb.data_ptr(), hosts[0], nbytes))
        d_ms = (time.perf_counter() - t0) / 5 * 1e3
        t0 = time.perf_counter()
        for _ in range(5):
            rt.rt_render_stereo(R.ctx, W, H, D, rt.rt_fb(fb[0].data_ptr(), 0, W * 4), rt.rt_fb(fb[1].data_ptr(), 0, W * 4))
            rt.rt_synchronize(R.ctx)
        r_ms = (time.perf_counter() - t0) / 5 * 1e3
        stages = {"render_ms": r_ms, "download_ms": d_ms, "compute_fraction_serialised": r_ms / (r_ms + d_ms),
                  "transfer_fraction_serialised": d_ms / (r_ms + d_ms),
                  "transfer_hidden_by_overlap": True,
                  "paper": "~60 % compute / up to 40 % CPU<->GPU transfer (PAPER.md:15, :106-107), unnamed NVIDIA GPU"}
        # the stage split re-rendered slot 0: download it again so the check below sees a pair
        rt.rt_wait(rt.rt_download(R.ctx, fb.data_ptr(), hosts[0], nbytes))
    ok = True
    if rank == 0:
        slot = (args.steps - 1) % F
        src = fbs[slot]
        host = np.frombuffer((ctypes.c_uint8 * nbytes).from_address(hosts[slot]), np.uint8)
        ok = bool(np.array_equal(host, src.reshape(-1).cpu().numpy()))
        for h in hosts:
            rt.rt_host_free(h)
    rays_timed = sum(rays_of[k % n_rig] for k in range(args.steps))
    return {"value": rays_timed / dt / 1e6, "unit": UNIT,
            "camera": "C5 orbit: frame k uses orbit camera k mod 60 (rays counted per orbit frame)" if orbit
            else "fixed (the config's rig)",
            "h2d_bytes_per_step": 76, "d2h_bytes_per_step": nbytes if rank == 0 else 0,
            "ms_per_step": dt / args.steps * 1e3, "stereo_fps": args.steps / dt, "download_verified": ok,
            "frames_in_flight": F, "stages": stages,
            "note": "per step: camera set from host values (the 76-byte camera block travels in the kernel "
                    "launch parameters), render, pinned async D2H (rt_download_after, copy stream) of the RGBA8 "
                    "stereo frame overlapped with the frames still rendering; host wall clock around K steps incl. "
                    "the last download"}


def load_profile(name, world):
    """ncu counters of one trace launch (profiles/trace_profile.json, written by scripts/ncu_summary.py
    from the committed --set full capture): dram / L1 bytes, pipe utilisation, launch duration."""
    p = os.path.join(ROOT, "profiles", "trace_profile.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(f"{name}/x{world}", d.get(name))
    except (OSError, ValueError):
        return None


def l1_roofline(prof, ceil, kernel_ms, sm_mhz):
    """Second ceiling: the trace kernel's L1 bytes per launch (ncu l1tex__t_bytes of
    the committed capture) over its live-timed duration, against 148 SMs x the B0-measured L1 bytes
    per clock x the SM clock."""
    if not prof or not prof.get("l1tex_t_bytes") or not ceil.get("l1_bytes_clk_sm"):
        return {"l1": None}
    peak = 148 * ceil["l1_bytes_clk_sm"] * sm_mhz * 1e6 / 1e9
    ach = prof["l1tex_t_bytes"] / (kernel_ms * 1e-3) / 1e9
    return {"l1": {"achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                   "bytes_per_launch": prof["l1tex_t_bytes"],
                   "data_pipe_wavefronts_pct_of_peak": prof.get("l1tex_data_pipe_lsu_wavefronts_pct_peak"),
                   "note": "bytes = L1 tag lookups x 32 B; the L1 data pipe is the tighter L1 limit: incoherent "
                           "128-bit loads cost one wavefront per distinct line", "source": prof.get("source")}}


def load_traffic(name, world):
    p = os.path.join(ROOT, "profiles", "trace_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(f"{name}/x{world}", d.get(name))
    except (OSError, ValueError):
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C4")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--gather", choices=["peer", "nccl"], default="peer",
                    help="N>1 frame assembly: fused peer stores into rank 0's FB (default) or NCCL gather")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--width", type=int, default=0, help="override the config's per-eye width")
    ap.add_argument("--height", type=int, default=0, help="override the config's per-eye height")
    ap.add_argument("--depth", type=int, default=-1, help="override the config's max_depth")
    ap.add_argument("--inflight", type=int, default=4,
                    help="frames in flight on separate streams in the throughput loop (1 = one at a time)")
    args = ap.parse_args()
    scene = scenes.make_scene(args.config)
    if args.width > 0 or args.height > 0 or args.depth >= 0:
        scene = scene.with_view(width=args.width or scene.width, height=args.height or scene.height,
                                max_depth=args.depth if args.depth >= 0 else scene.max_depth)
    if args.impl == "reference":
        return run_reference(args, scene)
    return run_ours(args, scene)


if __name__ == "__main__":
    sys.exit(main())
