#!/usr/bin/env python
"""Benchmark of the B200 gather + F-test hot path (BASELINE.json metric).

A step is one FPPM iteration of the workload (default: BASELINE configs[1],
"c2"): the max-live-radius reduction, the photon hash-grid build (cell keys,
radix sort, cell table, record permute), the warp-per-hit-point gather with
fp64 sector moments, and the fused end-of-iteration F-test/radius update.

Arms
  default            this repo's CUDA path (libfppm_gpu.so) on N GPUs
  --impl reference   the reference's own CPU code (oracle/_ref, compiled
                     unmodified from proj/core) on the host cores, bounded
                     samples of the same workload

Output: one JSON line on rank 0 (contract in the task statement).
"""
from __future__ import annotations

import argparse
import functools
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("hit-point×photon kernel queries/sec (gather+F-test), photons traced/sec, "
          "% HBM roofline")
UNIT = "queries/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--workload", default="c2", choices=["c1", "c2", "c5"],
                   help="c5: BASELINE configs[4] at full size (bench_c5.py)")
    p.add_argument("--kernel", default="auto", choices=["auto", "fine", "warp", "3d"],
                   help="gather kernel variant (A/B)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-trace", action="store_true", help="skip the light-phase (photons traced/s) leg")
    p.add_argument("--dist-mode", default="auto", choices=["auto", "a", "b"],
                   help="multi-GPU decomposition (distributed.py); auto = measure both in warm-up")
    p.add_argument("--cpu-trace-paths", type=int, default=1 << 20)
    p.add_argument("--no-render", action="store_true", help="skip the C3 full-iteration leg")
    return p.parse_args()


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi samples every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self._t = threading.Thread(target=self._read, daemon=True)
        self._t.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


KERNEL_NAMES = {"auto": "k_gather_ring (lean fine gather, double-buffered windows; F-test fused in k_tile_finalize)",
                "fine": "k_gather_ring (lean fine gather, double-buffered windows; F-test fused in k_tile_finalize)",
                "warp": "k_gather_test", "3d": "k_gather_3d (gather + accumulate; F-test in k_apply_deltas)"}


# ---------------------------------------------------------------- helpers
def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy, burst)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def ncu_traffic():
    """dram bytes per gather launch from the committed ncu --set full capture."""
    path = os.path.join(ROOT, "profiles", "gather_ncu.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch"), d.get("workload")
    except (OSError, ValueError):
        return None, None


def raster_rows(W, rank, world):
    r0 = W * rank // world
    r1 = W * (rank + 1) // world
    return r0, r1


def hitpoints_for_rows(W, r0, r1):
    import numpy as np
    j, i = np.meshgrid(np.arange(r0, r1), np.arange(W), indexing="ij")
    pos = np.zeros(((r1 - r0) * W, 3))
    pos[:, 0] = ((i.ravel() + 0.5) / W).astype(np.float32)
    pos[:, 1] = ((j.ravel() + 0.5) / W).astype(np.float32)
    nrm = np.tile([0.0, 0.0, 1.0], (len(pos), 1))
    return pos, nrm


def emit(line):
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- CPU reference
def cpu_sample(wl, n=None, seed=0xC0FFEE):
    """Seeded random hit-point sample (sorted): no raster aliasing.  1/64 of
    the frame for C2, 1/16 for C1."""
    import numpy as np
    n = n or wl.hitpoints // (64 if wl.hitpoints >= 1 << 18 else 16)
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(wl.hitpoints, n, replace=False)).astype(np.uint32)


def cpu_reference_run(wl, first, last, threads, sample=None):
    """The reference's own CPU path (oracle/_ref: PhotonGrid + GatherRegion,
    compiled unmodified) on a hit-point sample, iterations 1..last; per
    iteration the FULL photon grid is built (serial std::sort,
    photon_map.cpp:26-51) and every sampled hit point is gathered and tested
    on `threads` threads (integrator.cpp:52-70).  Iterations < first are the
    untimed warm-up (they only bring the sampled regions' radii to the state
    of the timed iterations).  Returns (records of the timed iterations,
    sample): each record holds the measured grid / gather seconds, the
    sample's accepted pairs, and the frame estimate (queries and seconds
    scaled by H / n)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Oracle
    ref, port = Oracle("reference"), Oracle("port")
    sub = cpu_sample(wl) if sample is None else sample
    hp = port.gen_raster_hitpoints(wl.raster)
    sess = ref.session(dict(n_annuli=wl.n_annuli, n_sectors=wl.n_sectors, alpha_f=wl.alpha_f,
                            initial_radius=wl.initial_radius, r_min_base=0.001 * wl.initial_radius,
                            samples_per_iteration=wl.photons, k=wl.k, alpha=wl.alpha,
                            threads=threads), {k: v[sub] for k, v in hp.items()})
    scale = wl.hitpoints / len(sub)
    out = []
    for it in range(1, last + 1):
        ph = port.gen_photons(wl.generator, wl.seed, it, 0, wl.photons)
        t0 = time.perf_counter()
        r = sess.iterate(it, ph)
        wall = time.perf_counter() - t0
        grid_s, gather_s = r["times"]
        if it >= first:
            q = float(r["accepted"].sum())
            out.append({"iteration": it, "grid_s": grid_s, "gather_s": gather_s, "wall_s": wall,
                        "q_sample": q, "accepted": r["accepted"].copy(),
                        "q_frame_est": q * scale, "s_frame_est": grid_s + gather_s * scale})
    return out, sub


def cpu_sample_text(wl, sub, threads, first, last):
    return (f"{wl.name} iterations {first}..{last} (after untimed iterations 1..{first - 1} of the same "
            f"sample): per iteration the full {wl.photons}-photon grid build (reference PhotonGrid, "
            f"serial std::sort) + gather/F-test of {len(sub)} of {wl.hitpoints} hit points (seeded random "
            f"sample) on {threads} threads; value = the frame rate estimated from it (queries and gather "
            f"time x{wl.hitpoints / len(sub):g}, grid build once), ms_per_step = the measured time")


def run_reference_arm(args, wl, rank):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    first, last = max(args.warmup, 0) + 1, max(args.warmup, 0) + max(args.steps, 1)
    try:
        run, sub = cpu_reference_run(wl, first, last, threads)
    except Exception as e:  # the reference arm must still print a line
        emit({"impl": "reference", "unavailable": f"reference CPU run failed: {e}"})
        return
    q = sum(x["q_frame_est"] for x in run)
    t = sum(x["s_frame_est"] for x in run)
    v = q / t
    measured = sum(x["grid_s"] + x["gather_s"] for x in run)
    sample = cpu_sample_text(wl, sub, threads, first, last)
    emit({"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
          "steps": len(run), "warmup": args.warmup, "ms_per_step": 1e3 * measured / len(run),
          "frame_ms_per_step_estimate": 1e3 * t / len(run),
          "sample_queries_per_step": sum(x["q_sample"] for x in run) / len(run),
          "frame_queries_per_step_estimate": q / len(run),
          "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
          "data": "synthetic (canonical PCG32 inputs, DESIGN.md §3)",
          "config": workload_config(wl),
          "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
                           "sample": sample},
          "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
          "trace": reference_trace(threads, args),
          "render": None if args.no_render else reference_render(threads),
          "vcm": None if args.no_render else reference_vcm(threads)})


def gpu_sample_check(wl, last, sub, local_rank, kernel):
    """The device's per-hit-point accepted counts and frame Q for iterations
    1..last (a fresh context on the same inputs), for the inline CPU
    baseline's parity and sample-bias check."""
    from paper_2504_04411_b200 import FppmContext
    ctx = FppmContext(**wl.context_kwargs(device=local_rank, gather_kernel=kernel))
    wl.set_hitpoints(ctx)
    acc, qf = {}, {}
    for it in range(1, last + 1):
        ctx.generate_photons(wl.generator, wl.seed, it, wl.photons)
        o, sm = ctx.iterate(it)
        acc[it] = o["accepted"][sub].astype("uint64")
        qf[it] = sm["accepted"]
    ctx.close()
    return acc, qf


def reference_trace(threads, args):
    if args.no_trace:
        return None
    try:
        paths = args.cpu_trace_paths
        dep, secs = cpu_trace_run(paths, threads)
        return {"photons_traced_per_s": dep / secs, "light_paths_per_s": paths / secs, "cores": threads,
                "kind": "reference", "sample": f"{paths} light paths of iteration 1 (of {TRACE_PATHS})",
                "config": trace_config()}
    except Exception as e:
        return {"unavailable": f"reference tracer failed: {e}"}


# ---------------------------------------------------------------- light phase
TRACE_PATHS = 1 << 23      # BASELINE configs[2]: 8M photons (light paths) per iteration
TRACE_MAX_DEPTH = 8        # maximum path length 8


def trace_config():
    return {"workload": "c3 light phase (BASELINE configs[2]): caustic box (scene.caustic_box), "
                        f"{TRACE_PATHS} light paths per iteration, max_depth {TRACE_MAX_DEPTH}",
            "roulette": "from depth 5 (reference kRouletteDepth, path.hpp:156)"}


def cpu_trace_run(paths, threads, iteration=1):
    """Reference light phase (oracle/_ref: Scene + BVH + trace_light_subpath)
    on `paths` light paths with `threads` host threads.  (deposits, seconds)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Oracle
    from paper_2504_04411_b200.scene import caustic_box
    sc = Oracle("reference").scene(caustic_box().arrays())
    t0 = time.perf_counter()
    out = sc.trace(0x5EED, iteration, paths, TRACE_MAX_DEPTH, threads=threads)
    return len(out["depth"]), time.perf_counter() - t0


def run_trace_bench(args, local_rank, steps, warmup):
    """photons traced/s: fppm_gpu_trace_photons (emission + tracing + path-order
    compaction into the staging buffers of the next grid build), timed with
    CUDA events on the context stream."""
    import torch
    from paper_2504_04411_b200 import FppmContext
    from paper_2504_04411_b200.scene import caustic_box
    ctx = FppmContext(initial_radius=0.01, samples_per_iteration=TRACE_PATHS, max_hitpoints=1,
                      max_photons=4 * TRACE_PATHS, device=local_rank)
    ctx.set_scene(caustic_box())
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    for it in range(1, warmup + 1):
        ctx.trace_photons(0x5EED, it, TRACE_PATHS, TRACE_MAX_DEPTH)
    torch.cuda.synchronize()
    l0 = FppmContext.kernel_launches()
    ms, dep = [], 0
    for it in range(warmup + 1, warmup + steps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        dep += ctx.trace_photons(0x5EED, it, TRACE_PATHS, TRACE_MAX_DEPTH)
        e1.record(stream)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    launches = FppmContext.kernel_launches() - l0
    ctx.close()
    secs = sum(ms) / 1e3
    return {"photons_traced_per_s": dep / secs, "light_paths_per_s": TRACE_PATHS * steps / secs,
            "ms_per_iteration": 1e3 * secs / steps, "deposits_per_iteration": dep / steps,
            "gpu_launches": launches, "steps": steps,
            "timing": "CUDA events around fppm_gpu_trace_photons on the context stream",
            "config": trace_config()}


RENDER_RES = 1024          # BASELINE configs[2]: 1024 x 1024 camera


def render_config():
    return {"workload": f"c3 full improved-PPM iteration (BASELINE configs[2]): caustic box, {RENDER_RES}^2 "
                        f"pinhole, {TRACE_PATHS} light paths, max_depth {TRACE_MAX_DEPTH}",
            "test": "reference defaults (C3 leaves them open): 2x6 groups, alpha_F 0.01, "
                    "r1 = 0.002 * bounding radius, luminance channel",
            "stages": "light phase + eye pass + grid + gather/F-test + film (Renderer::step)"}


def run_render_bench(local_rank, steps, warmup):
    """C3: Renderer::step on the device, timed with CUDA events per iteration."""
    import torch
    from paper_2504_04411_b200 import FppmContext
    from paper_2504_04411_b200.scene import bounding_radius, caustic_box, caustic_box_camera
    sc, cam = caustic_box(), caustic_box_camera(RENDER_RES)
    r1 = 0.002 * bounding_radius(sc)
    ctx = FppmContext(initial_radius=r1, samples_per_iteration=TRACE_PATHS, n_annuli=2, n_sectors=6,
                      alpha_f=0.01, r_min_base=0.001 * r1, max_depth=TRACE_MAX_DEPTH,
                      max_hitpoints=RENDER_RES * RENDER_RES, max_photons=4 * TRACE_PATHS, device=local_rank)
    ctx.set_scene(sc)
    ctx.set_camera(cam)
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    for it in range(1, warmup + 1):
        ctx.render_iteration(0x5EED, it, TRACE_PATHS)
    torch.cuda.synchronize()
    c0 = ctx.counters()["accepted"]
    ms = []
    for it in range(warmup + 1, warmup + steps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ctx.render_iteration(0x5EED, it, TRACE_PATHS)
        e1.record(stream)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    q = ctx.counters()["accepted"] - c0
    ctx.close()
    return {"ms_per_iteration": statistics.mean(ms), "queries_per_s": q / (sum(ms) / 1e3),
            "steps": steps, "timing": "CUDA events around FppmContext.render_iteration on the context stream",
            "config": render_config()}


def reference_render(threads):
    """The reference's own render() (oracle/_ref), one C3 iteration."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Oracle
    from paper_2504_04411_b200.scene import caustic_box, caustic_box_camera
    try:
        rs = Oracle("reference").scene(caustic_box().arrays())
        _, _, secs = rs.render_fppm(caustic_box_camera(RENDER_RES), 0x5EED, 1, TRACE_MAX_DEPTH, TRACE_PATHS,
                                    r0_frac=0.002, n_annuli=2, n_sectors=6, alpha_f=0.01, threads=threads)
        return {"ms_per_iteration": 1e3 * secs, "cores": threads, "kind": "reference",
                "sample": "iteration 1 of the full C3 config through the reference's render() "
                          "(IterationReport wall time of the whole call)"}
    except Exception as e:
        return {"unavailable": f"reference render failed: {e}"}


VCM_PATHS = 1 << 20       # BASELINE configs[3]: 1M light sub-paths per iteration


def vcm_config():
    return {"workload": f"c4 full VCM+ iteration (BASELINE configs[3]): caustic box, {RENDER_RES}^2 pinhole, "
                        f"{VCM_PATHS} light sub-paths, max_depth {TRACE_MAX_DEPTH}",
            "test": "4 sectors (1x4), alpha_F 0.05, r1 = 0.002 * bounding radius, luminance channel",
            "stages": "light sub-paths + camera splats + eye sub-paths (emitter hits, NEE, connections) + grid + "
                      "merges at every rough eye vertex (primary F-tested) + film (Renderer::step, vcm_plus)"}


def run_vcm_bench(local_rank, steps, warmup):
    """C4: Renderer::step with vcm_plus on the device (fppm_gpu_render_vcm),
    timed with CUDA events per iteration."""
    import torch
    from paper_2504_04411_b200 import FppmContext
    from paper_2504_04411_b200.scene import bounding_radius, caustic_box, caustic_box_camera
    sc, cam = caustic_box(), caustic_box_camera(RENDER_RES)
    r1 = 0.002 * bounding_radius(sc)
    ctx = FppmContext(initial_radius=r1, samples_per_iteration=VCM_PATHS, n_annuli=1, n_sectors=4,
                      alpha_f=0.05, r_min_base=0.001 * r1, max_depth=TRACE_MAX_DEPTH,
                      max_hitpoints=RENDER_RES * RENDER_RES, max_photons=8 * VCM_PATHS, device=local_rank,
                      vcm_plus=True, mis_n_vm=VCM_PATHS)
    ctx.set_scene(sc)
    ctx.set_camera(cam)
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    for it in range(1, warmup + 1):
        ctx.render_vcm_iteration(0x5EED, it, VCM_PATHS)
    torch.cuda.synchronize()
    c0 = ctx.counters()["accepted"]
    l0 = FppmContext.kernel_launches()
    ms = []
    for it in range(warmup + 1, warmup + steps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ctx.render_vcm_iteration(0x5EED, it, VCM_PATHS)
        e1.record(stream)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    q = ctx.counters()["accepted"] - c0
    launches = FppmContext.kernel_launches() - l0
    ctx.close()
    return {"ms_per_iteration": statistics.mean(ms), "merge_queries_per_s": q / (sum(ms) / 1e3),
            "gpu_launches": launches, "steps": steps,
            "timing": "CUDA events around FppmContext.render_vcm_iteration on the context stream",
            "config": vcm_config()}


def reference_vcm(threads):
    """The reference's own render() with vcm_plus (oracle/_ref), one C4 iteration."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Oracle
    from paper_2504_04411_b200.scene import caustic_box, caustic_box_camera
    try:
        rs = Oracle("reference").scene(caustic_box().arrays())
        _, _, secs = rs.render_vcm_plus(caustic_box_camera(RENDER_RES), 0x5EED, 1, TRACE_MAX_DEPTH, VCM_PATHS,
                                        r0_frac=0.002, n_annuli=1, n_sectors=4, alpha_f=0.05, threads=threads)
        return {"ms_per_iteration": 1e3 * secs, "cores": threads, "kind": "reference",
                "sample": "iteration 1 of the full C4 config through the reference's render() with vcm_plus "
                          "(IterationReport wall time of the whole call)"}
    except Exception as e:
        return {"unavailable": f"reference render failed: {e}"}


def workload_config(wl, **extra):
    cfg = {"workload": f"{wl.name} (BASELINE configs[{0 if wl.name.startswith('c1') else 1}])",
           "hitpoints": wl.hitpoints, "photons_per_iteration": wl.photons,
           "groups": f"{wl.n_annuli}x{wl.n_sectors}", "alpha_f": wl.alpha_f,
           "initial_radius": wl.initial_radius}
    cfg.update(extra)
    return cfg


# ---------------------------------------------------------------- GPU arm
class Arm:
    """One decomposition of the iteration over `world` ranks (distributed.py).

    mode "a": this rank's raster-row band of hit points; photon shares
              all-gathered (NCCL) so every rank builds the full grid.
    mode "b": every hit point on every rank; the local photon share only,
              gathered into partial-sum rows, reduce-scattered to the owners,
              owners test, radii all-gathered.
    With world == 1 both are the plain single-GPU iteration (b through the
    deltas API)."""

    def __init__(self, mode, wl, args, rank, world, local_rank, dev):
        import torch
        from paper_2504_04411_b200 import FppmContext
        self.mode, self.wl, self.rank, self.world, self.dev = mode, wl, rank, world, dev
        W = wl.raster
        if mode == "a":
            r0, r1 = raster_rows(W, rank, world)
        else:
            r0, r1 = 0, W
        self.H = (r1 - r0) * W
        self.ctx = FppmContext(**wl.context_kwargs(max_hitpoints=self.H, max_photons=wl.photons,
                                                   device=local_rank, gather_kernel=args.kernel))
        pos, nrm = hitpoints_for_rows(W, r0, r1)
        self.ctx.set_hitpoints(pos, nrm)
        self.stream = torch.cuda.ExternalStream(self.ctx.stream, device=dev)
        self.n_local = wl.photons * (rank + 1) // world - wl.photons * rank // world
        self.begin = wl.photons * rank // world
        if mode == "a" and world > 1:
            from paper_2504_04411_b200.distributed import share_stride
            self.stride = share_stride(wl.photons, world)
            self.part_n = [wl.photons * (r + 1) // world - wl.photons * r // world for r in range(world)]
            self.cell = torch.zeros(1, dtype=torch.float64, device=dev)
        if mode == "b":
            from paper_2504_04411_b200.distributed import owner_slice
            self.h0, self.n_own = owner_slice(self.H, rank, world)
            self.rows = torch.zeros((self.H, self.ctx.delta_stride), dtype=torch.float64, device=dev)
            self.radius = self.ctx.radius_tensor()

    def photons(self, src, n):
        from paper_2504_04411_b200 import _native as N
        return N.Photons(*[src[k].data_ptr() for k, _, _ in photon_layout()])

    def step(self, it, b, host_out=None):
        """One iteration on photon share `b` (device tensors, this rank's
        share); `host_out`: optional IterOut pointer for this rank's results."""
        import torch
        import torch.distributed as dist
        from paper_2504_04411_b200 import _native as N
        ctx, world = self.ctx, self.world
        if self.mode == "a":
            if world > 1:
                # one packed all-gather of the shares; r_max all-reduced on the
                # device; each rank stages only the photons within r_max of its
                # band's hit points and builds its grid from the device cell
                from paper_2504_04411_b200.distributed import allgather_packed, device_cell_size, pack_photons
                with torch.cuda.stream(self.stream):
                    packed = pack_photons(b["photon_pos"], b["photon_normal"], b["photon_wi"], b["photon_power"],
                                          b["photon_depth"], self.stride)
                    full = allgather_packed(packed)
                device_cell_size(ctx, self.cell)
                ctx.set_photons_packed(full, self.part_n, margin=self.cell)
                ctx.build_grid_device(self.cell)
            else:
                N.check(ctx._lib.fppm_gpu_set_photons_device(ctx._h, self.photons(b, 0),
                                                             self.wl.photons), ctx._h)
                ctx.build_grid(0.0)  # device-side max live radius
            N.check(ctx._lib.fppm_gpu_gather_test(ctx._h, it, host_out, None), ctx._h)
            return
        self._step_b(it, b, host_out)

    def _step_b(self, it, b, host_out):
        import torch
        from paper_2504_04411_b200 import _native as N
        from paper_2504_04411_b200.distributed import allgather_owner_values, reduce_scatter_rows
        ctx, world = self.ctx, self.world
        N.check(ctx._lib.fppm_gpu_set_photons_device(ctx._h, self.photons(b, 0), self.n_local), ctx._h)
        ctx.build_grid(0.0)  # radii are replicated: the local max is the global r_max
        with torch.cuda.stream(self.stream):
            ctx.gather_deltas(it, self.rows)
            mine = reduce_scatter_rows(self.rows, world)
            N.check(ctx._lib.fppm_gpu_apply_deltas(ctx._h, it, self.h0, self.n_own, mine.data_ptr(),
                                                   host_out, None), ctx._h)
            if world > 1:
                self.radius.copy_(allgather_owner_values(self.radius[self.h0:self.h0 + self.n_own],
                                                         self.H, world))

    def close(self):
        self.ctx.close()


@functools.lru_cache(maxsize=None)
def photon_layout():
    """(name, dtype, per-photon shape) of the fppm_photons SoA fields."""
    import torch
    return (("photon_pos", torch.float32, (3,)), ("photon_normal", torch.float32, (3,)),
            ("photon_wi", torch.float32, (3,)), ("photon_power", torch.float32, (3,)),
            ("photon_depth", torch.int32, ()))


def run_gpu_arm(args, wl, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2504_04411_b200 import FppmContext
    from paper_2504_04411_b200 import _native as N
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    total_steps = args.warmup + args.steps
    n_local = wl.photons * (rank + 1) // world - wl.photons * rank // world
    begin = wl.photons * rank // world

    # ---- per-iteration photon shares, resident in HBM before timing
    gen_ctx = FppmContext(initial_radius=wl.initial_radius, samples_per_iteration=wl.photons,
                          max_hitpoints=1, max_photons=1, device=local_rank)

    def gen_batch(it):
        out = {k: torch.empty((n_local,) + shape, dtype=dt, device=dev) for k, dt, shape in photon_layout()}
        ph = N.Photons(*[out[k].data_ptr() for k, _, _ in photon_layout()])
        torch.cuda.synchronize()
        N.check(gen_ctx._lib.fppm_gpu_generate_photons_to(gen_ctx._h, wl.generator, wl.seed, it, begin,
                                                          n_local, ph), gen_ctx._h)
        gen_ctx.synchronize()
        return out

    batches = [gen_batch(it) for it in range(1, total_steps + 1)]
    gen_ctx.close()
    torch.cuda.synchronize()

    # ---- decomposition: fixed by --dist-mode, or chosen by measurement over
    # the warm-up iterations (BASELINE: all-gather vs reduce-scatter)
    modes = [args.dist_mode] if args.dist_mode != "auto" else (["a", "b"] if world > 1 else ["a"])
    choice = {}
    arm = None
    for mode in modes:
        cand = Arm(mode, wl, args, rank, world, local_rank, dev)
        for s in range(args.warmup):
            cand.step(s + 1, batches[s])
        torch.cuda.synchronize()
        if len(modes) > 1:
            # time one more warm-up-style iteration (max over ranks), then rewind
            cand.ctx.reset_regions()
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            if world > 1:
                dist.barrier()
            t0.record(cand.stream)
            for s in range(args.warmup):
                cand.step(s + 1, batches[s])
            t1.record(cand.stream)
            torch.cuda.synchronize()
            ms = torch.tensor([t0.elapsed_time(t1) / max(args.warmup, 1)], dtype=torch.float64, device=dev)
            if world > 1:
                dist.all_reduce(ms, op=dist.ReduceOp.MAX)
            choice[mode] = float(ms.item())
        if arm is None or (len(modes) > 1 and choice[mode] < choice[arm.mode]):
            if arm is not None:
                arm.close()
            arm = cand
        else:
            cand.close()
    ctx, H, stream = arm.ctx, arm.H, arm.stream
    if len(modes) > 1:
        # replay the warm-up on the chosen arm so the timed iterations continue it
        ctx.reset_regions()
        for s in range(args.warmup):
            arm.step(s + 1, batches[s])
        torch.cuda.synchronize()

    ctx.gather_kernel_ms()  # drop the warm-up launches
    if world > 1:
        dist.barrier()
    c0 = ctx.counters()
    l0 = FppmContext.kernel_launches()
    clocks = ClockSampler(local_rank)
    clocks.start()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for s in range(args.warmup, total_steps):
        arm.step(s + 1, batches[s])
    t_end.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    launches = FppmContext.kernel_launches() - l0
    c1 = ctx.counters()
    elapsed_ms = t_start.elapsed_time(t_end)
    g_ms = ctx.gather_kernel_ms()  # the dominant kernel alone (events in the library)
    q_local = c1["accepted"] - c0["accepted"]
    stats = torch.tensor([elapsed_ms, float(q_local), float(launches)], dtype=torch.float64, device=dev)
    if world > 1:
        t_max = stats[:1].clone()
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
        q_sum = stats[1:2].clone()
        dist.all_reduce(q_sum, op=dist.ReduceOp.SUM)
        elapsed_ms, q_total = float(t_max.item()), float(q_sum.item())
    else:
        q_total = float(q_local)
    value = q_total / (elapsed_ms / 1e3)

    # ---- roofline of the dominant kernel (the gather), rank 0
    G, C = wl.groups, 1
    gather_avg_s = statistics.mean(g_ms) / 1e3
    alg_bytes = 16.0 * q_local / args.steps + (64 + 48 * G * C) * H
    peak, peak_src = peaks()
    achieved = alg_bytes / gather_avg_s / 1e9
    traffic, traffic_wl = ncu_traffic()

    # ---- end to end through the C ABI with pinned host buffers
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(arm, batches, args, dev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # the reference on the first two timed iterations (same sample, same
        # state: iterations 1..warmup replayed untimed first)
        try:
            import numpy as np
            threads = os.cpu_count() or 1
            first = args.warmup + 1
            last = first + min(args.steps, 2) - 1
            run, sub = cpu_reference_run(wl, first, last, threads)
            acc, qf = gpu_sample_check(wl, last, sub, local_rank, args.kernel)
            q = sum(x["q_frame_est"] for x in run)
            t = sum(x["s_frame_est"] for x in run)
            cpu = {"value": q / t, "unit": UNIT, "cores": threads, "kind": "reference",
                   "sample": cpu_sample_text(wl, sub, threads, first, last),
                   "measured_ms_per_iteration": 1e3 * sum(x["grid_s"] + x["gather_s"] for x in run) / len(run),
                   "grid_build_s": [round(x["grid_s"], 4) for x in run],
                   "sample_gather_s": [round(x["gather_s"], 4) for x in run],
                   "sample_accepted_equal_to_gpu": all(np.array_equal(x["accepted"], acc[x["iteration"]])
                                                       for x in run),
                   "sample_queries": [x["q_sample"] for x in run],
                   "frame_queries_estimate": [x["q_frame_est"] for x in run],
                   "frame_queries_gpu": [qf[x["iteration"]] for x in run],
                   "frame_estimate_over_gpu": [x["q_frame_est"] / qf[x["iteration"]] for x in run]}
        except Exception as e:
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    trace = None
    if not args.no_trace:
        trace = run_trace_bench(args, local_rank, max(args.steps, 1), max(args.warmup, 1))
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            trace["cpu_baseline"] = reference_trace(os.cpu_count() or 1, args)
    render = vcm = None
    if not args.no_render:
        render = run_render_bench(local_rank, max(min(args.steps, 5), 1), max(min(args.warmup, 3), 1))
        vcm = run_vcm_bench(local_rank, max(min(args.steps, 5), 1), max(min(args.warmup, 3), 1))
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            render["cpu_baseline"] = reference_render(os.cpu_count() or 1)
            vcm["cpu_baseline"] = reference_vcm(os.cpu_count() or 1)

    if rank == 0:
        if world == 1:
            par = "1 GPU"
        elif arm.mode == "a":
            par = (f"option A over {world} GPUs: hit points sharded by raster rows; photon shares "
                   "all-gathered (NCCL) each step; every rank builds the full grid")
        else:
            par = (f"option B over {world} GPUs: every rank gathers its own photon share for all "
                   "hit points; partial-sum rows reduce-scattered (NCCL) to the owners, radii "
                   "all-gathered")
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps,
            "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (canonical PCG32 inputs generated on device, DESIGN.md §3)",
            "config": workload_config(
                wl, parallelism=par,
                decomposition={"mode": arm.mode, "measured_ms_per_iteration": choice or None},
                l2=f"inputs larger than L2: fresh {wl.photons * 52 / 1e6:.0f} MB photon batch "
                   "per step (+256 MB sorted records)" if wl.photons * 52 > 126e6 else
                   "photon batch smaller than L2 (not flushed)",
                iterations_timed=f"{args.warmup + 1}..{args.warmup + args.steps}"),
            "photons_per_s": wl.photons * args.steps / (elapsed_ms / 1e3),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": KERNEL_NAMES.get(args.kernel, args.kernel),
                         "algorithmic_bytes_per_launch": alg_bytes,
                         "bytes_formula": "16*Q + (64 + 48*G*C)*H (SURVEY.md 8d)",
                         "avg_launch_ms": gather_avg_s * 1e3, "launch_ms": [round(x, 3) for x in g_ms],
                         "timing": "CUDA events around the kernel launch on the context stream "
                                   "(fppm_gpu_gather_kernel_ms)",
                         "share_of_step": gather_avg_s * 1e3 / (elapsed_ms / args.steps),
                         "peak_source": peak_src, "traffic_source": traffic_wl},
            "gpu_launches": launches,
            "clocks": clk,
            "counters": {"accepted": q_total, "candidates": c1["candidates"] - c0["candidates"],
                         "exact_path_pairs": c1["exact"] - c0["exact"],
                         "ambiguous_pairs": c1["ambiguous"] - c0["ambiguous"]},
        }
        if e2e:
            line["e2e"] = e2e
        if cpu:
            line["cpu_baseline"] = cpu
        if trace:
            line["trace"] = trace
        if render:
            line["render"] = render
        if vcm:
            line["vcm"] = vcm
        emit(line)
    arm.close()


def run_e2e(arm, batches, args, dev):
    """Same metric through the C-ABI host path: per step the photon share is
    copied from pinned host memory (fppm_gpu_set_photons) and the per-hit-point
    radius, radiance and decision of this rank's hit points are read back."""
    import ctypes as C
    import torch
    import torch.distributed as dist
    from paper_2504_04411_b200 import _native as N
    ctx, wl, world, H = arm.ctx, arm.wl, arm.world, arm.H
    pinned = []
    for b in batches:
        hb = {k: torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for k, t in b.items()}
        for k in b:
            hb[k].copy_(b[k])
        pinned.append(hb)
    n_out = H if arm.mode == "a" else arm.n_own
    out_r = torch.empty(max(n_out, 1), dtype=torch.float64, pin_memory=True)
    out_rad = torch.empty((max(n_out, 1), 3), dtype=torch.float32, pin_memory=True)
    out_rej = torch.empty(max(n_out, 1), dtype=torch.uint8, pin_memory=True)
    io = N.IterOut()
    io.radius = out_r.data_ptr()
    io.radiance = out_rad.data_ptr()
    io.rejected = out_rej.data_ptr()
    local = {k: torch.empty_like(t) for k, t in batches[0].items()}
    torch.cuda.synchronize()
    ctx.reset_regions()
    n_local = next(iter(pinned[0].values())).shape[0]
    h2d = sum(t.numel() * t.element_size() for t in pinned[0].values())
    d2h = n_out * (8 + 12 + 1)

    token = C.c_uint64(0)

    def one(it, hb, nxt=None):
        if world == 1 and arm.mode == "a":
            if token.value:  # this step's batch was prefetched during the previous step
                N.check(ctx._lib.fppm_gpu_adopt_photons(ctx._h, token.value), ctx._h)
                token.value = 0
            else:
                ph = N.Photons(*[hb[k].data_ptr() for k, _, _ in photon_layout()])
                N.check(ctx._lib.fppm_gpu_set_photons(ctx._h, ph, n_local), ctx._h)
            if nxt is not None:  # the next step's upload overlaps this iteration
                pn = N.Photons(*[nxt[k].data_ptr() for k, _, _ in photon_layout()])
                N.check(ctx._lib.fppm_gpu_prefetch_photons(ctx._h, pn, n_local, C.byref(token)), ctx._h)
            N.check(ctx._lib.fppm_gpu_iterate(ctx._h, it, C.byref(io), None), ctx._h)
            return
        with torch.cuda.stream(arm.stream):
            for k in local:
                local[k].copy_(hb[k], non_blocking=True)
        arm.step(it, local, C.byref(io))

    for s in range(args.warmup):
        one(s + 1, pinned[s])
    c0 = ctx.counters()["accepted"]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    end = args.warmup + args.steps
    for s in range(args.warmup, end):  # every step's upload is inside the timed region
        one(s + 1, pinned[s], pinned[s + 1] if s + 1 < end else None)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    q = float(ctx.counters()["accepted"] - c0)
    el = torch.tensor([t1 - t0, q], dtype=torch.float64, device=dev)
    if world > 1:
        tm = el[:1].clone()
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        qs = el[1:].clone()
        dist.all_reduce(qs, op=dist.ReduceOp.SUM)
        secs, q = float(tm.item()), float(qs.item())
    else:
        secs = t1 - t0
    path = ("pinned host photons -> device through the ABI: step i+1's upload issued by fppm_gpu_prefetch_photons "
            "before step i's fppm_gpu_iterate (it overlaps that iteration) and adopted by fppm_gpu_adopt_photons; "
            "the first timed step uploads with fppm_gpu_set_photons; fppm_gpu_iterate with host outputs"
            if world == 1 and
            arm.mode == "a" else f"pinned host share -> device, option {arm.mode.upper()} step with host outputs")
    return {"value": q / secs, "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": 1e3 * secs / args.steps, "path": path}


def main():
    # no Python garbage-collection pauses inside timed regions (a gen-2 pass
    # between two launches would be charged to the device timeline)
    gc.collect()
    gc.disable()
    args = parse()
    from paper_2504_04411_b200.workloads import WORKLOADS
    wl = WORKLOADS[args.workload]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if args.workload == "c5":
            import bench_c5
            bench_c5.run_reference(args, wl, rank, emit, METRIC)
        else:
            run_reference_arm(args, wl, rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        if args.workload == "c5":
            import bench_c5
            bench_c5.run_gpu(args, wl, rank, world, local_rank, emit, METRIC, ClockSampler, peaks)
        else:
            run_gpu_arm(args, wl, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
