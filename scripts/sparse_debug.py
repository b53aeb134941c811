import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..")); sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import numpy as np
from scenes import scene3d
from paper_2504_04411_b200 import FppmContext
hit, _ = scene3d(2, H=800, N=30000)
res = {}
for k in ("warp", "sparse"):
    ctx = FppmContext(initial_radius=0.03, samples_per_iteration=60000, n_annuli=1, n_sectors=4, alpha_f=0.05,
                      r_min_base=3e-5, max_hitpoints=800, max_photons=30000, gather_kernel=k)
    ctx.set_hitpoints(hit["pos"], hit["nrm"], hit["wo"], hit["thr"], hit["alb"], hit["eye_depth"], hit["gathered"])
    outs = []
    for it in range(1, 3):
        ph = scene3d(200 + it, H=800, N=30000)[1]
        ctx.set_photons(ph["pos"], ph["nrm"], ph["wi"], ph["pow"], ph["depth"])
        o, sm = ctx.iterate(it, stats=True)
        outs.append(o)
    res[k] = outs
for it in range(2):
    a, b = res["warp"][it], res["sparse"][it]
    for key in ("accepted", "stat_count", "stat_sum", "stat_sum_sq", "flux", "radius", "statistic"):
        x, y = a[key], b[key]
        bad = np.flatnonzero((np.abs(x.astype(float) - y.astype(float)) > 1e-9 * np.abs(x.astype(float)) + 1e-300).reshape(len(x), -1).any(-1))
        print(it + 1, key, len(bad), bad[:5], x[bad[:2]] if len(bad) else "", y[bad[:2]] if len(bad) else "")
