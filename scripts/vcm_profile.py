"""Warm per-kernel device time of one C4 VCM+ iteration (torch.profiler / CUPTI)."""
import collections, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2504_04411_b200 import FppmContext
from paper_2504_04411_b200.scene import bounding_radius, caustic_box, caustic_box_camera
RES, J = int(os.environ.get("RES", "1024")), int(os.environ.get("J", str(1 << 20)))
sc, cam = caustic_box(), caustic_box_camera(RES)
r1 = 0.002 * bounding_radius(sc)
ctx = FppmContext(initial_radius=r1, samples_per_iteration=J, n_annuli=1, n_sectors=4, alpha_f=0.05,
                  r_min_base=0.001 * r1, max_depth=8, max_hitpoints=RES * RES, max_photons=8 * J,
                  vcm_plus=True, mis_n_vm=J)
ctx.set_scene(sc)
ctx.set_camera(cam)
for it in range(1, 4):
    ctx.render_vcm_iteration(0x5EED, it, J)
ctx.synchronize()
steps = 3
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for it in range(4, 4 + steps):
        ctx.render_vcm_iteration(0x5EED, it, J)
    ctx.synchronize()
tot, cnt = collections.defaultdict(float), collections.Counter()
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        tot[e.name] += e.device_time_total
        cnt[e.name] += 1
print(f"per iteration: {sum(tot.values()) / steps / 1000:.3f} ms")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:16]:
    print(f"{v / steps:9.1f} us  {cnt[k] // steps:3d}x  {k[:90]}")
