"""Host-side timing of gather_test phases (diagnostic)."""
import time, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gc
if os.environ.get("NOGC"): gc.disable()
from paper_2504_04411_b200 import FppmContext, WORKLOADS
wl = WORKLOADS["c2"]
kern = sys.argv[1] if len(sys.argv) > 1 else "auto"
ctx = FppmContext(**wl.context_kwargs(gather_kernel=kern))
ctx.generate_raster_hitpoints(wl.raster)
for it in range(1, 9):
    ctx.generate_photons(wl.generator, wl.seed, it, wl.photons)
    ctx.synchronize()
    t0 = time.perf_counter()
    ctx.build_grid(0.0)
    ctx.synchronize()
    t1 = time.perf_counter()
    ctx.gather_test(it, outputs=False, summary=False)
    t2 = time.perf_counter()
    ctx.synchronize()
    t3 = time.perf_counter()
    print(kern, it, f"grid {1e3*(t1-t0):.3f} ms  gather host-return {1e3*(t2-t1):.3f} ms  gather done {1e3*(t3-t1):.3f} ms")
