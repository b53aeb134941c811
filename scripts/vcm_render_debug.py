"""Debug: one VCM+ device iteration, NaN census of the intermediate buffers."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2504_04411_b200 import FppmContext
from paper_2504_04411_b200.scene import bounding_radius, caustic_box, caustic_box_camera
sc, cam = caustic_box(), caustic_box_camera(int(os.environ.get("RES", "24")))
J = int(os.environ.get("J", "5000"))
npix = cam.width * cam.height
r1 = 0.002 * bounding_radius(sc)
ctx = FppmContext(initial_radius=r1, samples_per_iteration=J, n_annuli=2, n_sectors=6, alpha_f=0.01,
                  r_min_base=0.001 * r1, max_depth=8, max_hitpoints=npix, max_photons=8 * J, vcm_plus=True, mis_n_vm=J)
ctx.set_scene(sc)
ctx.set_camera(cam)
ctx.render_vcm_iteration(17, 1, J, 8)
hp = ctx.get_hitpoints(emitted=True)
for k, v in hp.items():
    v = np.asarray(v, dtype=np.float64)
    print(k, v.shape, "nan", np.isnan(v).sum(), "max", np.nanmax(np.abs(v)) if v.size else 0)
img, n = ctx.film_mean()
print("film nan", np.isnan(img).sum(), "of", img.size)
r = ctx.regions()
print({k: (np.isnan(np.asarray(v, dtype=float)).sum()) for k, v in r.items()})
mis = ctx.get_photon_mis()
print({k: (np.isnan(v).sum(), np.nanmax(v)) for k, v in mis.items()})
