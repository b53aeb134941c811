"""Light-phase timing alone (caustic box, 8M paths, max depth 8): per-call ms."""
import argparse
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch  # noqa: E402

from paper_2504_04411_b200 import FppmContext  # noqa: E402
from paper_2504_04411_b200.scene import caustic_box  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--steps", type=int, default=5)
p.add_argument("--paths", type=int, default=1 << 23)
a = p.parse_args()
ctx = FppmContext(initial_radius=0.01, samples_per_iteration=a.paths, max_hitpoints=1, max_photons=4 * a.paths)
ctx.set_scene(caustic_box())
s = torch.cuda.ExternalStream(ctx.stream)
ms = []
for it in range(a.steps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    n = ctx.trace_photons(0x5EED, it + 1, a.paths, 8)
    e1.record(s)
    torch.cuda.synchronize()
    ms.append(e0.elapsed_time(e1))
print("ms", [round(x, 3) for x in ms], "deposits", n)
