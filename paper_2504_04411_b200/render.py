"""render() on the device for the kernel-estimation algorithms of the
reference (integrator.hpp:21-66, integrator.cpp:669-683): the per-iteration
Renderer::step runs on the B200 (light phase, eye pass, grid, gather +
end-of-iteration policy, film), this module only sequences iterations and
assembles the RenderResult the reference returns.

    fppm      tested per-pixel radius, ANOVA F-test (policy ftest)
    cppm      tested per-pixel radius, chi-squared test (policy chi2)
    sppm      one global radius schedule (policy schedule: every pixel,
              gathered or not, takes schedule_radius(r_1, alpha, i + 1))
    vcm_plus  bidirectional + merges, tested per-pixel radius (F-test)
    vcm       bidirectional + merges, the global schedule

Path tracing and BDPT (no kernel estimation) are outside this repository's
hot path (SURVEY.md 8 / DESIGN.md §9).
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from .api import FppmContext, RadiusSchedule, TestConfig, resolve_channels
from .scene import Camera, Scene, bounding_radius

ALGORITHMS = ("fppm", "cppm", "sppm", "vcm_plus", "vcm")


@dataclass
class IterationReport:
    """integrator.hpp:38-50."""
    iteration: int = 0
    seconds: float = 0.0
    radius: Optional[np.ndarray] = None
    rejected: Optional[np.ndarray] = None
    vc_luminance: float = 0.0
    vm_luminance: float = 0.0


@dataclass
class RenderResult:
    """integrator.hpp:56-59: the film (mean image [h, w, 3] fp64 plus the
    per-pixel vc / vm luminance totals) and the iteration reports."""
    image: np.ndarray = None
    vc_total: np.ndarray = None
    vm_total: np.ndarray = None
    iterations: int = 0
    reports: List[IterationReport] = field(default_factory=list)


def render(scene: Scene, camera: Camera, algorithm: str = "fppm", iterations: int = 1, seed: int = 0,
           max_depth: int = 10, light_paths: int = 0, r0_frac: float = 0.002,
           test: Optional[TestConfig] = None, schedule: Optional[RadiusSchedule] = None, mis_beta: float = 1.0,
           keep_reports: bool = True, device: int = 0) -> RenderResult:
    """The reference's render(scene, config) for the merging algorithms."""
    if algorithm not in ALGORITHMS:
        raise ValueError(f"render: algorithm '{algorithm}' is not a kernel-estimation algorithm on the device")
    if iterations < 1:
        raise ValueError("render: iterations must be >= 1")
    if max_depth < 1:
        raise ValueError("render: max_depth must be >= 1")
    test = test or TestConfig()
    schedule = schedule or RadiusSchedule()
    npix = camera.width * camera.height
    J = light_paths or npix                                   # integrator.cpp:109
    r1 = r0_frac * bounding_radius(scene)                     # integrator.cpp:121
    r_min = schedule.r_min_base if schedule.r_min_base > 0 else 0.001 * r1  # :125-126
    vcm = algorithm in ("vcm_plus", "vcm")
    policy = {"fppm": "ftest", "vcm_plus": "ftest", "cppm": "chi2", "sppm": "schedule", "vcm": "schedule"}[algorithm]
    ctx = FppmContext(initial_radius=r1, samples_per_iteration=J, n_annuli=test.n_annuli, n_sectors=test.n_sectors,
                      alpha_f=test.alpha_f, alpha_chi2=test.alpha_chi2,
                      channels=resolve_channels(test.channels, scene), override_decision=test.override_decision,
                      policy=policy, k=schedule.k, alpha=schedule.alpha, r_min_base=r_min, max_depth=max_depth,
                      max_hitpoints=npix, max_photons=J * max(max_depth - 1, 1), device=device,
                      vcm_plus=vcm, mis_n_vm=J if vcm else 0, mis_beta=mis_beta)
    try:
        ctx.set_scene(scene)
        ctx.set_camera(camera)
        res = RenderResult()
        vc0 = vm0 = 0.0
        for i in range(1, iterations + 1):
            t0 = time.perf_counter()
            if vcm:
                ctx.render_vcm_iteration(seed, i, J, max_depth)
                out = ctx.regions()
                rej = None
            else:
                o, _ = ctx.render_iteration(seed, i, J, max_depth, outputs=True)
                out, rej = o, o["rejected"].copy()
            ctx.synchronize()
            secs = time.perf_counter() - t0
            if keep_reports:
                vc, vm = ctx.film_splits()
                vcs, vms = float(vc.sum()), float(vm.sum())
                res.reports.append(IterationReport(i, secs, np.asarray(out["radius"]).copy(), rej, vcs - vc0,
                                                   vms - vm0))
                vc0, vm0 = vcs, vms
        res.image, res.iterations = ctx.film_mean()
        res.vc_total, res.vm_total = ctx.film_splits()
        return res
    finally:
        ctx.close()
