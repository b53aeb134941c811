"""C5 leg of bench.py (BASELINE configs[4], the 1/2/4/8-GPU scaling stress):
16M hit points uniform in the unit cube with random normals, 2^27 photons
per iteration from 64 Gaussian clusters + 20 % background restricted to the
nearest hit point's tangent slab, r0 = 0.005, 2 x 4 groups, alpha_F 0.05.

A step is one FPPM iteration over the whole frame: r_max, grid build
(3D fine cells), the 3D warp-per-hit-point gather + F-test.  On N GPUs hit
points are sharded by index range and every rank generates its photon share
[r N / G, (r + 1) N / G); an NCCL all-gather assembles the full, identically
ordered photon set; r_max is an all-reduce(max) on the device (no host round
trip) -- SURVEY.md 8(e) option A.

The reference arm and the inline cpu_baseline time the reference's own code
(oracle/_ref) on a bounded sample (cpu_c5_sample): 1/1024 of the hit points
against the full-density photons of their neighbourhoods -- from the C
restatement of the generator on every host thread (reference arm) or from
the device generator (inline baseline); both are the same canonical photons."""
from __future__ import annotations

import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
UNIT = "queries/s"
CPU_HP_FRACTION = 1024


def c5_config(wl, world, extra=None):
    cfg = {"workload": f"{wl.name} (BASELINE configs[4])", "hitpoints": wl.hitpoints,
           "photons_per_iteration": wl.photons, "groups": f"{wl.n_annuli}x{wl.n_sectors}", "alpha_f": wl.alpha_f,
           "initial_radius": wl.initial_radius,
           "parallelism": "1 GPU" if world == 1 else
           f"option A over {world} GPUs: hit points sharded by index range, photon shares all-gathered (NCCL), "
           "r_max all-reduced on the device"}
    if extra:
        cfg.update(extra)
    return cfg


def _near_mask(ph_pos, hit_pos, cell, chunk=1 << 24):
    """Photons whose reference cell lies within +-2 cells of a sampled hit
    point's cell: an order-preserving superset of every sampled hit point's
    27-cell neighbourhood (photon_map.cpp:53-78), so the sample's queries are
    exactly the full frame's."""
    import numpy as np
    inv = 1.0 / cell

    def cells(p):
        return np.floor(np.asarray(p, np.float64) * inv).astype(np.int64)

    def pack(c):
        b = 1 << 20
        return ((c[:, 0] + b) << 42) | ((c[:, 1] + b) << 21) | (c[:, 2] + b)

    off = np.stack(np.meshgrid(*[np.arange(-2, 3)] * 3, indexing="ij"), -1).reshape(-1, 3)
    want = np.unique(pack((cells(hit_pos)[:, None, :] + off[None]).reshape(-1, 3)))
    m = np.zeros(len(ph_pos), bool)
    for a in range(0, len(ph_pos), chunk):
        m[a:a + chunk] = np.isin(pack(cells(ph_pos[a:a + chunk])), want)
    return m


def cpu_photons(c5, wl, it, threads):
    """The iteration's full photon set from the C restatement of the
    generator, in chunks on `threads` host threads (ctypes drops the GIL)."""
    import numpy as np
    from concurrent.futures import ThreadPoolExecutor
    n = wl.photons
    step = max(1 << 16, (n + 8 * threads - 1) // (8 * threads))
    parts = list(range(0, n, step))
    with ThreadPoolExecutor(max_workers=threads) as ex:
        chunks = list(ex.map(lambda b: c5.photons(it, b, min(step, n - b)), parts))
    return {k: np.concatenate([c[k] for c in chunks]) for k in chunks[0]}


def cpu_c5_sample(wl, iterations, threads, photons_fn=None, hit_pos=None):
    """Reference code (oracle/_ref) on the C5 sample: 1/1024 of the hit points
    (seeded random), each against the full-density photons of its own
    neighbourhood (_near_mask of the iteration's whole photon set), grid
    built over those photons with cell = r_1 (= r_max of iterations 1-2).
    Frame estimates: gather time x H / n, grid time x N / n_photons (the
    reference sorts all N; n log n makes this an underestimate of its cost),
    queries x H / n.  photons_fn(it) -> photon dict (full set)."""
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Oracle
    ref, port = Oracle("reference"), Oracle("port")
    c5 = port.c5(wl.seed, wl.hitpoints)
    rng = np.random.default_rng(0xC5)
    n_hp = wl.hitpoints // CPU_HP_FRACTION
    sub = np.sort(rng.choice(wl.hitpoints, n_hp, replace=False))
    hp = c5.hitpoints()
    hs = {k: v[sub] for k, v in hp.items()}
    sess = ref.session(dict(n_annuli=wl.n_annuli, n_sectors=wl.n_sectors, alpha_f=wl.alpha_f,
                            initial_radius=wl.initial_radius, r_min_base=0.001 * wl.initial_radius,
                            samples_per_iteration=wl.photons, k=wl.k, alpha=wl.alpha, threads=threads), hs)
    out = []
    for it in iterations:
        ph = photons_fn(it) if photons_fn else cpu_photons(c5, wl, it, threads)
        m = _near_mask(ph["pos"], hs["pos"], wl.initial_radius)
        ph = {k: v[m] for k, v in ph.items()}
        n_ph = int(m.sum())
        r = sess.iterate(it, ph, cell=wl.initial_radius)
        grid_s, gather_s = r["times"]
        q = float(r["accepted"].sum())
        sh = wl.hitpoints / n_hp
        out.append({"iteration": it, "grid_s": grid_s, "gather_s": gather_s, "q_sample": q, "photons": n_ph,
                    "q_frame_est": q * sh, "s_frame_est": grid_s * wl.photons / max(n_ph, 1) + gather_s * sh})
    return out, n_hp


def sample_text(wl, n_hp, threads, iters, run=None):
    nph = f" ({', '.join(str(x['photons']) for x in run)} photons)" if run else ""
    return (f"{wl.name} iterations {iters[0]}..{iters[-1]}: {n_hp} random hit points (of {wl.hitpoints}) against "
            f"the full-density photons of their +-2-cell neighbourhoods{nph}, reference PhotonGrid over those "
            f"photons + GatherRegion gather/F-test on {threads} threads; queries and gather time "
            f"x{wl.hitpoints / n_hp:g}, grid time x N / photons")


def run_reference(args, wl, rank, emit, metric):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    its = list(range(1, min(max(args.steps, 1), 2) + 1))  # bounded: <= 2 iterations of the full generator
    try:
        run, n_hp = cpu_c5_sample(wl, its, threads)
    except Exception as e:  # the reference arm must still print a line
        emit({"impl": "reference", "unavailable": f"reference C5 run failed: {e}"})
        return
    q = sum(x["q_frame_est"] for x in run)
    t = sum(x["s_frame_est"] for x in run)
    v = q / t
    emit({"impl": "reference", "metric": metric, "value": v, "unit": UNIT, "n_gpus": args.gpus,
          "steps": len(run), "warmup": 0, "ms_per_step": 1e3 * sum(x["grid_s"] + x["gather_s"] for x in run) / len(run),
          "frame_ms_per_step_estimate": 1e3 * t / len(run), "higher_is_better": True, "scaling": "weak",
          "vs_baseline": None, "dtype": "f64", "data": "synthetic (C5 generator, DESIGN.md §3)",
          "config": c5_config(wl, 1),
          "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
                           "sample": sample_text(wl, n_hp, threads, its, run)},
          "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})


def run_gpu(args, wl, rank, world, local_rank, emit, metric, clock_sampler, peaks):
    import torch
    import torch.distributed as dist
    from paper_2504_04411_b200 import FppmContext
    from paper_2504_04411_b200 import _native as N
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    H, NP = wl.hitpoints, wl.photons
    h0, nh = H * rank // world, H * (rank + 1) // world - H * rank // world
    p0, npn = NP * rank // world, NP * (rank + 1) // world - NP * rank // world
    ctx = FppmContext(**wl.context_kwargs(max_hitpoints=nh, max_photons=NP, device=local_rank))
    ctx.c5_setup(wl.seed, H)
    ctx.c5_hitpoints(h0, nh)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    fields = (("pos", torch.float32, (3,)), ("normal", torch.float32, (3,)), ("wi", torch.float32, (3,)),
              ("power", torch.float32, (3,)), ("depth", torch.int32, ()))
    total = args.warmup + args.steps
    # photon shares of every iteration, resident in HBM before timing
    shares = []
    for it in range(1, total + 1):
        b = {k: torch.empty((npn,) + sh, dtype=dt, device=dev) for k, dt, sh in fields}
        ph = N.Photons(*[b[k].data_ptr() for k, _, _ in fields])
        torch.cuda.synchronize()
        N.check(ctx._lib.fppm_gpu_generate_photons_to(ctx._h, 5, wl.seed, it, p0, npn, ph), ctx._h)
        ctx.synchronize()
        shares.append(b)
    full = {k: torch.empty((NP,) + sh, dtype=dt, device=dev) for k, dt, sh in fields} if world > 1 else None
    rmax = torch.zeros(1, dtype=torch.float64, device=dev)

    def step(it, b):
        with torch.cuda.stream(stream):
            src = b
            if world > 1:
                for k in full:
                    dist.all_gather_into_tensor(full[k], b[k])
                src = full
            N.check(ctx._lib.fppm_gpu_set_photons_device(
                ctx._h, N.Photons(*[src[k].data_ptr() for k, _, _ in fields]), NP), ctx._h)
            if world > 1:
                ctx.max_radius_device(rmax)
                dist.all_reduce(rmax, op=dist.ReduceOp.MAX)  # integrator.cpp:159-161 over all ranks
                ctx.build_grid_device(rmax)
            else:
                ctx.build_grid(0.0)
            N.check(ctx._lib.fppm_gpu_gather_test(ctx._h, it, None, None), ctx._h)

    for s in range(args.warmup):
        step(s + 1, shares[s])
    torch.cuda.synchronize()
    ctx.gather_kernel_ms()
    c0 = ctx.counters()
    l0 = FppmContext.kernel_launches()
    clocks = clock_sampler(local_rank)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for s in range(args.warmup, total):
        step(s + 1, shares[s])
    t1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    launches = FppmContext.kernel_launches() - l0
    c1 = ctx.counters()
    g_ms = ctx.gather_kernel_ms()
    ms = t0.elapsed_time(t1)
    q_local = float(c1["accepted"] - c0["accepted"])
    st = torch.tensor([ms, q_local], dtype=torch.float64, device=dev)
    if world > 1:
        tm = st[:1].clone()
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        qs = st[1:].clone()
        dist.all_reduce(qs, op=dist.ReduceOp.SUM)
        ms, q_total = float(tm.item()), float(qs.item())
    else:
        q_total = q_local
    value = q_total / (ms / 1e3)
    G = wl.groups
    gather_s = statistics.mean(g_ms) / 1e3
    alg = 16.0 * q_local / args.steps + (64 + 48 * G) * nh
    peak, peak_src = peaks()
    achieved = alg / gather_s / 1e9
    del shares
    # ---- e2e through the C ABI: the step's photon share from pinned host
    # memory (fppm_gpu_set_photons; all-gathered on device for N > 1) and the
    # radius / radiance / decision of this rank's hit points read back
    e2e = None
    if not args.no_e2e:
        import ctypes as C
        host = {k: torch.empty((npn,) + sh, dtype=dt, pin_memory=True) for k, dt, sh in fields}
        dshare = {k: torch.empty((npn,) + sh, dtype=dt, device=dev) for k, dt, sh in fields}
        out_r = torch.empty(nh, dtype=torch.float64, pin_memory=True)
        out_rad = torch.empty((nh, 3), dtype=torch.float32, pin_memory=True)
        out_rej = torch.empty(nh, dtype=torch.uint8, pin_memory=True)
        io = N.IterOut()
        io.radius, io.radiance, io.rejected = out_r.data_ptr(), out_rad.data_ptr(), out_rej.data_ptr()
        e_ms, e_q = 0.0, 0.0
        for s in range(args.steps):
            it = total + 1 + s
            # untimed: this step's share generated into pinned host memory
            ph = N.Photons(*[dshare[k].data_ptr() for k, _, _ in fields])
            N.check(ctx._lib.fppm_gpu_generate_photons_to(ctx._h, 5, wl.seed, it, p0, npn, ph), ctx._h)
            ctx.synchronize()
            for k in host:
                host[k].copy_(dshare[k])
            torch.cuda.synchronize()
            qa = ctx.counters()["accepted"]
            if world > 1:
                dist.barrier()
            ta = time.perf_counter()
            with torch.cuda.stream(stream):
                if world > 1:
                    for k in dshare:
                        dshare[k].copy_(host[k], non_blocking=True)
                        dist.all_gather_into_tensor(full[k], dshare[k])
                    N.check(ctx._lib.fppm_gpu_set_photons_device(
                        ctx._h, N.Photons(*[full[k].data_ptr() for k, _, _ in fields]), NP), ctx._h)
                    ctx.max_radius_device(rmax)
                    dist.all_reduce(rmax, op=dist.ReduceOp.MAX)
                    ctx.build_grid_device(rmax)
                    N.check(ctx._lib.fppm_gpu_gather_test(ctx._h, it, C.byref(io), None), ctx._h)
                else:
                    N.check(ctx._lib.fppm_gpu_set_photons(
                        ctx._h, N.Photons(*[host[k].data_ptr() for k, _, _ in fields]), NP), ctx._h)
                    N.check(ctx._lib.fppm_gpu_iterate(ctx._h, it, C.byref(io), None), ctx._h)
            torch.cuda.synchronize()
            el = time.perf_counter() - ta
            qq = float(ctx.counters()["accepted"] - qa)
            v2 = torch.tensor([el, qq], dtype=torch.float64, device=dev)
            if world > 1:
                a_ = v2[:1].clone()
                dist.all_reduce(a_, op=dist.ReduceOp.MAX)
                b_ = v2[1:].clone()
                dist.all_reduce(b_, op=dist.ReduceOp.SUM)
                el, qq = float(a_.item()), float(b_.item())
            e_ms += 1e3 * el
            e_q += qq
        h2d = sum(t.numel() * t.element_size() for t in host.values())
        e2e = {"value": e_q / (e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": nh * (8 + 12 + 1), "ms_per_step": e_ms / args.steps,
               "path": "fppm_gpu_set_photons from pinned host + fppm_gpu_iterate with host outputs"
                       if world == 1 else "pinned host share -> device, all-gather, device r_max, gather_test "
                                          "with host outputs",
               "timing": "host wall clock per step around the upload + iteration + output copy (sync), max over ranks"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            import numpy as np
            threads = os.cpu_count() or 1
            its = [1, 2]

            def gpu_photons(it):  # the same canonical photons, from the device generator
                ctx.generate_photons(5, wl.seed, it, NP)
                return ctx.get_photons()

            run, n_hp = cpu_c5_sample(wl, its, threads, photons_fn=gpu_photons)
            cpu = {"value": sum(x["q_frame_est"] for x in run) / sum(x["s_frame_est"] for x in run), "unit": UNIT,
                   "cores": threads, "kind": "reference", "sample": sample_text(wl, n_hp, threads, its, run),
                   "grid_build_s": [round(x["grid_s"], 3) for x in run],
                   "sample_gather_s": [round(x["gather_s"], 3) for x in run]}
        except Exception as e:
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}
    ctx.close()
    if rank == 0:
        line = {"metric": metric, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (C5 generator on device, DESIGN.md §3)",
                "config": c5_config(wl, world, {
                    "iterations_timed": f"{args.warmup + 1}..{total}",
                    "l2": f"inputs larger than L2: fresh {NP * 52 / 1e9:.1f} GB photon set per step"}),
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                             "frac": achieved / peak, "traffic": None,
                             "kernel": "k_prep_3d + k_gather_3d (3D warp-per-hit-point gather; F-test in "
                                       "k_apply_deltas)",
                             "algorithmic_bytes_per_launch": alg, "bytes_formula": "16*Q + (64 + 48*G*C)*H (SURVEY.md 8d)",
                             "avg_launch_ms": gather_s * 1e3, "launch_ms": [round(x, 3) for x in g_ms],
                             "share_of_step": gather_s * 1e3 / (ms / args.steps), "peak_source": peak_src},
                "gpu_launches": launches, "clocks": clk,
                "counters": {"accepted": q_total, "candidates": c1["candidates"] - c0["candidates"]}}
        if e2e:
            line["e2e"] = e2e
        if cpu:
            line["cpu_baseline"] = cpu
        emit(line)
    return value
