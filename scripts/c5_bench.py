"""C5 at full size on one GPU (16M hit points, 128M photons per iteration):
per-iteration device time of grid build + gather/F-test (photons generated
on the device beforehand, untimed)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch  # noqa: E402

from paper_2504_04411_b200 import WORKLOADS, FppmContext  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--steps", type=int, default=3)
p.add_argument("--scale", type=int, default=1, help="divide H and N by this")
a = p.parse_args()
wl = WORKLOADS["c5"]
H, N = wl.hitpoints // a.scale, wl.photons // a.scale
ctx = FppmContext(**wl.context_kwargs(max_hitpoints=H, max_photons=N))
ctx.c5_setup(wl.seed, H)
ctx.c5_hitpoints(0, H)
s = torch.cuda.ExternalStream(ctx.stream)
for it in range(1, a.steps + 1):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    e[0].record(s)
    ctx.generate_photons(5, wl.seed, it, N)
    e[1].record(s)
    ctx.build_grid(0.0)
    e[2].record(s)
    o, sm = ctx.gather_test(it, outputs=False, summary=True)
    e[3].record(s)
    torch.cuda.synchronize()
    g = ctx.gather_kernel_ms()
    print(f"it {it}: generate {e[0].elapsed_time(e[1]):.1f} ms, grid {e[1].elapsed_time(e[2]):.1f} ms, "
          f"gather+test {e[2].elapsed_time(e[3]):.1f} ms (kernel {g[-1]:.1f}), accepted {sm['accepted']}, "
          f"candidates {sm['candidates']}, rejected {sm['rejected']}, cells {sm['cells']}, "
          f"Gq/s {sm['accepted'] / (e[1].elapsed_time(e[3]) / 1e3) / 1e9:.2f}")
