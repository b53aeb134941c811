"""Warm per-kernel device time of one C3 FPPM render iteration (caustic box
1024^2, 8M light paths, max depth 8; torch.profiler / CUPTI)."""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_04411_b200 import FppmContext  # noqa: E402
from paper_2504_04411_b200.scene import bounding_radius, caustic_box, caustic_box_camera  # noqa: E402

RES, J = int(os.environ.get("RES", "1024")), int(os.environ.get("J", str(1 << 23)))
sc, cam = caustic_box(), caustic_box_camera(RES)
r1 = 0.002 * bounding_radius(sc)
ctx = FppmContext(initial_radius=r1, samples_per_iteration=J, n_annuli=2, n_sectors=6, alpha_f=0.01,
                  r_min_base=0.001 * r1, max_depth=8, max_hitpoints=RES * RES, max_photons=4 * J)
ctx.set_scene(sc)
ctx.set_camera(cam)
for it in range(1, 4):
    ctx.render_iteration(5, it, J, 8)
ctx.synchronize()
steps = 3
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for it in range(4, 4 + steps):
        ctx.render_iteration(5, it, J, 8)
    ctx.synchronize()
tot, cnt = collections.defaultdict(float), collections.Counter()
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        tot[e.name] += e.device_time_total
        cnt[e.name] += 1
print(f"per iteration: {sum(tot.values()) / steps / 1000:.3f} ms")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:20]:
    print(f"{v / steps:9.1f} us  {cnt[k] // steps:3d}x  {k[:90]}")
