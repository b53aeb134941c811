"""Warm per-kernel device time of one C2 FPPM step (torch.profiler / CUPTI
activity records of every kernel launched by libfppm_gpu.so)."""
import collections, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gc
gc.disable()
import torch
from paper_2504_04411_b200 import FppmContext, WORKLOADS
wl = WORKLOADS[os.environ.get("WL", "c2")]
ctx = FppmContext(**wl.context_kwargs())
wl.set_hitpoints(ctx)
steps = int(os.environ.get("STEPS", "3"))
for it in range(1, 4):
    ctx.generate_photons(wl.generator, wl.seed, it, wl.photons)
    ctx.build_grid(0.0)
    ctx.gather_test(it, outputs=False, summary=False)
ctx.synchronize()
acts = [torch.profiler.ProfilerActivity.CUDA]
import time
wall = 0.0
with torch.profiler.profile(activities=acts) as prof:
    for it in range(4, 4 + steps):
        ctx.generate_photons(wl.generator, wl.seed, it, wl.photons)
        ctx.synchronize()
        t0 = time.perf_counter()
        ctx.build_grid(0.0)
        ctx.gather_test(it, outputs=False, summary=False)
        ctx.synchronize()
        wall += time.perf_counter() - t0
print(f"wall per step (grid + gather, host-synchronised): {1e3 * wall / steps:.3f} ms")
tot = collections.defaultdict(float)
cnt = collections.Counter()
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        tot[e.name] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
        cnt[e.name] += 1
T = sum(v for k, v in tot.items() if "k_photons" not in k)
print(f"per step (excl. photon generation): {T / steps / 1000:.3f} ms")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v / steps:9.1f} us  {cnt[k] // steps:3d}x  {k[:90]}")
# idle time: the union of kernel intervals against the span of the timed steps
iv = sorted((e.time_range.start, e.time_range.end) for e in prof.events()
            if e.device_type == torch.autograd.DeviceType.CUDA and "k_photons" not in e.name)
if iv:
    busy, cs, ce = 0.0, iv[0][0], iv[0][1]
    for a, b in iv[1:]:
        if a > ce:
            busy += ce - cs
            cs, ce = a, b
        else:
            ce = max(ce, b)
    busy += ce - cs
    print(f"kernel-busy time per step (union of intervals): {busy / steps / 1000:.3f} ms")
