"""Kernel timing on a fixed state: reset regions, iteration `it` photons,
build grid, gather; repeated (diagnostic for A/B experiments)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gc
gc.disable()
from paper_2504_04411_b200 import FppmContext, WORKLOADS
wl = WORKLOADS[os.environ.get("WL", "c2")]
ctx = FppmContext(**wl.context_kwargs())
ctx.generate_raster_hitpoints(wl.raster)
ctx.generate_photons(wl.generator, wl.seed, 1, wl.photons)
ts = []
for rep in range(6):
    ctx.reset_regions()
    ctx.build_grid(0.0)
    ctx.gather_test(1, outputs=False, summary=False)
    ctx.synchronize()
ms = ctx.gather_kernel_ms()[1:]
print(os.environ.get("FPPM_GPU_LIB", "default"), "iteration-1 kernel ms", [round(x, 3) for x in ms],
      "min", round(min(ms), 3))
