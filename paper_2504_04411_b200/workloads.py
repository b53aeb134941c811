"""BASELINE.json synthetic configurations.

Each workload fixes the canonical input generator, the hit-point raster and
the TestConfig/RadiusSchedule of one BASELINE config.  Where BASELINE leaves
a reference parameter open, the choice is recorded here and in DESIGN.md:

* hit points: Lambertian albedo 1, throughput 1, wo = n = +z, eye depth 1;
* photons: depth 1 (J = N light paths of one vertex), deposit normal +z,
  wi cosine-distributed about +z;
* r_min_base = 0.001 r_1 (integrator.cpp:125-126), k = 0.7, alpha = 0.75,
  max_depth 10, normal guard cos 30 deg (integrator.cpp:47).
* C5: hit points uniform in the unit cube with uniform random normals (raster
  = 4096 only fixes H = 4096^2); photons from the generator in generate.cu
  (clusters + background, nearest-hit-point tangent-plane restriction).
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Workload:
    name: str
    generator: int          # FPPM_WORKLOAD_* id of the canonical photon generator
    raster: int             # hit points = raster x raster on z = 0
    photons: int            # N = J per iteration
    initial_radius: float
    n_annuli: int
    n_sectors: int
    alpha_f: float
    iterations: int
    seed: int = 0x5EED
    k: float = 0.7
    alpha: float = 0.75

    @property
    def hitpoints(self) -> int:
        return self.raster * self.raster

    @property
    def groups(self) -> int:
        return self.n_annuli * self.n_sectors

    def context_kwargs(self, **over):
        kw = dict(initial_radius=self.initial_radius, samples_per_iteration=self.photons,
                  n_annuli=self.n_annuli, n_sectors=self.n_sectors, alpha_f=self.alpha_f,
                  k=self.k, alpha=self.alpha, r_min_base=0.001 * self.initial_radius,
                  max_hitpoints=self.hitpoints, max_photons=self.photons)
        kw.update(over)
        return kw

    def set_hitpoints(self, ctx, h0: int = 0, n: int | None = None):
        """The workload's hit points [h0, h0 + n) on a context (C1/C2: the
        raster, all of it; C5: a share of the generated set)."""
        if self.generator == 5:
            ctx.c5_setup(self.seed, self.hitpoints)
            ctx.c5_hitpoints(h0, self.hitpoints - h0 if n is None else n)
        else:
            ctx.generate_raster_hitpoints(self.raster)

    def scaled(self, raster: int, photons: int, name: str | None = None) -> "Workload":
        """Same density law at a smaller size (parity tests)."""
        from dataclasses import replace
        return replace(self, name=name or f"{self.name}-r{raster}-n{photons}", raster=raster,
                       photons=photons)


# BASELINE configs[0]: gather-only synthetic PPM step on z = 0
C1 = Workload("c1_uniform_plane", generator=1, raster=256, photons=1 << 20,
              initial_radius=0.02, n_annuli=1, n_sectors=4, alpha_f=0.05, iterations=16)
# BASELINE configs[1]: non-uniform density (step 10:1 + Gaussian blob)
C2 = Workload("c2_step_blob", generator=2, raster=512, photons=1 << 22,
              initial_radius=0.01, n_annuli=2, n_sectors=4, alpha_f=0.01, iterations=64)

# BASELINE configs[4]: scaling stress gather, 3D (hit points in the unit cube)
C5 = Workload("c5_clusters_3d", generator=5, raster=4096, photons=1 << 27,
              initial_radius=0.005, n_annuli=2, n_sectors=4, alpha_f=0.05, iterations=32)

WORKLOADS = {"c1": C1, "c2": C2, "c5": C5}
