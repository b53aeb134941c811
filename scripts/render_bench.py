"""C3 full iteration on the device (caustic box 1024^2, 8M paths): per-call ms."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch  # noqa: E402

from paper_2504_04411_b200 import FppmContext  # noqa: E402
from paper_2504_04411_b200.scene import bounding_radius, caustic_box, caustic_box_camera  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--steps", type=int, default=5)
p.add_argument("--res", type=int, default=1024)
p.add_argument("--paths", type=int, default=1 << 23)
p.add_argument("--kernel", default="auto")
a = p.parse_args()
sc, cam = caustic_box(), caustic_box_camera(a.res)
r1 = 0.002 * bounding_radius(sc)
ctx = FppmContext(initial_radius=r1, samples_per_iteration=a.paths, n_annuli=2, n_sectors=6, alpha_f=0.01,
                  r_min_base=0.001 * r1, max_depth=8, max_hitpoints=a.res * a.res, max_photons=4 * a.paths,
                  gather_kernel=a.kernel)
ctx.set_scene(sc)
ctx.set_camera(cam)
s = torch.cuda.ExternalStream(ctx.stream)
for it in range(1, a.steps + 1):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    t0 = time.perf_counter()
    ev[0].record(s)
    n = ctx.trace_photons(5, it, a.paths, 8)
    ev[1].record(s)
    ctx.trace_eye(5, it)
    ev[2].record(s)
    o, sm = ctx.iterate(it, outputs=False, summary=True)
    ev[3].record(s)
    ctx.film_add()
    ev[4].record(s)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(it, "trace %.2f eye %.2f iterate %.2f film %.2f total %.2f ms (wall %.2f) photons %d accepted %d cells %d"
          % tuple([ev[i].elapsed_time(ev[i + 1]) for i in range(4)] + [ev[0].elapsed_time(ev[4]), 1e3 * (t1 - t0),
                   n, sm["accepted"], sm["cells"]]))
