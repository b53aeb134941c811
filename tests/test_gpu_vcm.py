"""GPU parity of the VCM+ merge stage (integrator.cpp:595-627): every gathered
photon value is weighted by the MIS merge weight (path.cpp:103-111) computed
from the hit point's tested radius, then fed to the sector statistics and the
flux.  Compared with the oracle (and the reference build) on canonical and
general scenes with random MIS partials."""
import numpy as np
import pytest

from helpers import compare_iteration
from paper_2504_04411_b200 import FppmContext, InvalidArgument
from scenes import scene3d

pytestmark = pytest.mark.gpu


def _ctx(cfg, hit, H, kernel="auto"):
    ctx = FppmContext(gather_kernel=kernel, initial_radius=cfg["initial_radius"], samples_per_iteration=cfg["samples_per_iteration"],
                      n_annuli=cfg["n_annuli"], n_sectors=cfg["n_sectors"], alpha_f=cfg["alpha_f"],
                      r_min_base=cfg["r_min_base"], channels="rgb" if cfg.get("channels", 1) == 3 else "luminance",
                      max_hitpoints=H, max_photons=1 << 17, vcm_plus=True, mis_n_vm=cfg["mis_n_vm"],
                      mis_beta=cfg["mis_beta"])
    ctx.set_hitpoints(hit["pos"], hit["nrm"], hit["wo"], hit["thr"], hit["alb"], hit["eye_depth"],
                      hit.get("gathered"))
    return ctx


@pytest.mark.parametrize("kernel", ["auto", "warp"])
@pytest.mark.parametrize("beta", [1.0, 2.0])
@pytest.mark.parametrize("channels", [1, 3])
def test_vcm_canonical_matches_oracle(port, beta, channels, kernel):
    W, N = 48, 1 << 15
    hit = port.gen_raster_hitpoints(W)
    cfg = dict(n_annuli=2, n_sectors=4, alpha_f=0.01, initial_radius=0.02, r_min_base=2e-5,
               samples_per_iteration=N, threads=8, vcm_plus=1, mis_n_vm=N, mis_beta=beta, channels=channels)
    ctx = _ctx(cfg, hit, W * W, kernel)
    sess = port.session(cfg, hit)
    rng = np.random.default_rng(int(beta * 10) + channels)
    ev, em = rng.random(W * W) * 2, rng.random(W * W)
    ctx.set_hitpoint_mis(ev, em)
    sess.set_eye_mis(ev, em)
    for it in range(1, 4):
        ph = port.gen_photons(2, 0x5EED, it, 0, N)
        pv, pm, pc = rng.random(N) * 3, rng.random(N), rng.random(N)
        ctx.set_photons(ph["pos"], ph["nrm"], ph["wi"], ph["pow"], ph["depth"])
        ctx.set_photon_mis(pv, pm, pc)
        sess.set_photon_mis(pv, pm, pc)
        got, _ = ctx.iterate(it, stats=True)
        want = sess.iterate(it, ph)
        compare_iteration(got, want)
        assert want["accepted"].sum() > 0


@pytest.mark.parametrize("kernel", ["auto", "warp"])
def test_vcm_general_scene_matches_reference(port, ref, kernel):
    hit, _ = scene3d(4, H=400, N=15000)
    cfg = dict(n_annuli=2, n_sectors=6, alpha_f=0.05, initial_radius=0.03, r_min_base=3e-5,
               samples_per_iteration=15000, threads=4, vcm_plus=1, mis_n_vm=15000, mis_beta=2.0)
    ctx = _ctx(cfg, hit, 400, kernel)
    sess = ref.session(cfg, hit)
    rng = np.random.default_rng(3)
    ev, em = rng.random(400) * 2, rng.random(400)
    ctx.set_hitpoint_mis(ev, em)
    sess.set_eye_mis(ev, em)
    for it in range(1, 4):
        ph = scene3d(400 + it, H=400, N=15000)[1]
        pv, pm, pc = rng.random(15000) * 3, rng.random(15000), rng.random(15000)
        ctx.set_photons(ph["pos"], ph["nrm"], ph["wi"], ph["pow"], ph["depth"])
        ctx.set_photon_mis(pv, pm, pc)
        sess.set_photon_mis(pv, pm, pc)
        got, _ = ctx.iterate(it, stats=True)
        compare_iteration(got, sess.iterate(it, ph))


def test_vcm_requires_warp_kernel():
    with pytest.raises(InvalidArgument):
        FppmContext(initial_radius=0.02, samples_per_iteration=16, vcm_plus=True, mis_n_vm=16,
                    gather_kernel="fine")
