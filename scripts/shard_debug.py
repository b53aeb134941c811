import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..")); sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle")); sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import numpy as np, torch
from oracle import Oracle
from helpers import oracle_cfg
from paper_2504_04411_b200 import WORKLOADS, FppmContext
from paper_2504_04411_b200.distributed import owner_slice, photon_share
port = Oracle("port")
world, kernel = 2, sys.argv[1] if len(sys.argv) > 1 else "warp"
wl = WORKLOADS["c2"].scaled(raster=48, photons=1 << 16)
H = wl.hitpoints
ctxs = []
for _ in range(world):
    c = FppmContext(**wl.context_kwargs(gather_kernel=kernel)); c.generate_raster_hitpoints(wl.raster); ctxs.append(c)
single = FppmContext(**wl.context_kwargs(gather_kernel=kernel)); single.generate_raster_hitpoints(wl.raster)
sess = port.session(oracle_cfg(wl), port.gen_raster_hitpoints(wl.raster))
stride = ctxs[0].delta_stride
W = [1597, 1598]
for it in range(1, 4):
    rows = []
    for r, c in enumerate(ctxs):
        b, n = photon_share(wl.photons, r, world)
        c.generate_photons(wl.generator, wl.seed, it, n, begin=b); c.build_grid(0.0)
        d = torch.zeros((H, stride), dtype=torch.float64, device="cuda"); c.gather_deltas(it, d); rows.append(d)
    total = rows[0] + rows[1]
    got = {}
    for r, c in enumerate(ctxs):
        h0, n = owner_slice(H, r, world)
        o, _ = c.apply_deltas(it, h0, total[h0:h0 + n], stats=True)
        for k, v in o.items(): got.setdefault(k, []).append(v)
    got = {k: np.concatenate(v, 0) for k, v in got.items()}
    for c in ctxs: c.set_regions(radius=got["radius"])
    single.generate_photons(wl.generator, wl.seed, it, wl.photons)
    s_out, _ = single.iterate(it, stats=True)
    want = sess.iterate(it, port.gen_photons(wl.generator, wl.seed, it, 0, wl.photons))
    for h in W:
        print(it, h, "acc", got["accepted"][h], s_out["accepted"][h], want["accepted"][h], "gr", got["gather_radius"][h], want["gather_r"][h] if "gather_r" in want else None,
              "F", got["statistic"][h], want["statistic"][h], "Fc", want["critical"][h], "rej", got["rejected"][h], want["rejected"][h])
        print("   rows", [rr[h, :8].cpu().numpy() for rr in rows])
