"""Dump GPU-traced and reference-traced photons for offline diffing (debug)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from oracle import Oracle  # noqa: E402
from paper_2504_04411_b200 import FppmContext  # noqa: E402
from paper_2504_04411_b200.scene import caustic_box, mixed_box  # noqa: E402

out = {}
for name, f in (("caustic", caustic_box), ("mixed", mixed_box)):
    sc = f()
    ctx = FppmContext(initial_radius=0.02, samples_per_iteration=1 << 16, max_hitpoints=16, max_photons=1 << 20)
    ctx.set_scene(sc)
    ctx.trace_photons(0xC0FFEE, 1, 30000, 8)
    g = ctx.get_photons()
    w = Oracle("reference").scene(sc.arrays()).trace(0xC0FFEE, 1, 30000, 8, threads=8)
    for k in g:
        out[f"{name}_gpu_{k}"] = g[k]
    for k in w:
        out[f"{name}_ref_{k}"] = w[k]
os.makedirs("gpurun_out", exist_ok=True)
np.savez_compressed("gpurun_out/trace_debug.npz", **out)
print("saved")
