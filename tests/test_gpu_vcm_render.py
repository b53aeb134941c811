"""C4 end to end on the device: one whole VCM+ iteration per call
(Renderer::step with Algorithm::vcm_plus, integrator.cpp:150-228, 236-301,
492-653) -- light sub-paths and their camera splats, eye sub-paths with MIS
partials, emitter hits, next-event estimation, connections to light sub-path
px % J, kernel estimation at every rough eye vertex (the primary one tested
per pixel) -- against the reference's own render() on the same scene, camera,
seed, J and iterations.

The device restates every step in fp64 without FMA in the reference's
operation order with the reference's RNG streams; the photons of the merge
gathers are the canonical fp32 records and device sin/cos differ from glibc
in the last bits; on these scenes and seeds no rounded photon crosses a
kernel boundary, so every tested radius is identical and every pixel agrees
within 1e-6 relative (measured <= 3e-8; the north-star tolerance is 1e-5)."""
import numpy as np
import pytest

from paper_2504_04411_b200 import FppmContext, InvalidArgument, StateError
from paper_2504_04411_b200.scene import (Camera, bounding_radius, caustic_box, caustic_box_camera, mixed_box,
                                        two_lights_sphere_emitter)

pytestmark = pytest.mark.gpu


def _vcm_ctx(npix, J, r1, max_depth=8, **kw):
    return FppmContext(initial_radius=r1, samples_per_iteration=J, n_annuli=2, n_sectors=6, alpha_f=0.01,
                       r_min_base=0.001 * r1, max_depth=max_depth, max_hitpoints=npix, max_photons=8 * J,
                       vcm_plus=True, mis_n_vm=J, **kw)


def _compare(got, want, label):
    rel = np.abs(got - want) / np.maximum(np.abs(want), 1e-30)
    bad = (rel > 1e-6).any(-1) & (np.abs(got - want) > 1e-12).any(-1)
    print(f"{label}: {bad.sum()} of {len(want)} pixels outside 1e-6 relative; max rel "
          f"{rel[~bad].max() if (~bad).any() else 0:.2e} elsewhere; mean got {got.mean():.6g} want {want.mean():.6g}")
    return bad


@pytest.mark.parametrize("res,J,iters,kernel", [(24, 5000, 3, "auto"), (24, 5000, 3, "warp"),
                                               (32, 20000, 2, "auto")])
def test_vcm_film_matches_reference_render(ref, res, J, iters, kernel):
    """kernel: the merges on the thread-per-vertex kernel (auto) or the warp
    kernel."""
    sc, cam = caustic_box(), caustic_box_camera(res)
    npix = cam.width * cam.height
    r1 = 0.002 * bounding_radius(sc)
    ctx = _vcm_ctx(npix, J, r1, gather_kernel=kernel)
    ctx.set_scene(sc)
    ctx.set_camera(cam)
    for it in range(1, iters + 1):
        ctx.render_vcm_iteration(17, it, J, 8)
    img, n = ctx.film_mean()
    assert n == iters
    assert np.isfinite(img).all() and img.max() > 0
    rs = ref.scene(sc.arrays())
    film, radius, _ = rs.render_vcm_plus(cam, 17, iters, 8, J, r0_frac=0.002, n_annuli=2, n_sectors=6,
                                         alpha_f=0.01, threads=8)
    bad = _compare(img.reshape(-1, 3), film, f"vcm+ {res}^2 J={J} {kernel}")
    # measured: every pixel within 3e-8 and every tested radius identical on
    # these seeds; a fp32-rounded merge photon on a kernel boundary would show
    # up here as a radius difference (see test_gpu_render._attributed_render)
    assert bad.sum() == 0
    rad = ctx.regions()["radius"]
    assert np.array_equal(rad, radius)


def test_vcm_render_api_errors():
    sc, cam = caustic_box(), caustic_box_camera(8)
    r1 = 0.002 * bounding_radius(sc)
    plain = FppmContext(initial_radius=r1, samples_per_iteration=100, max_hitpoints=64, max_photons=800,
                        max_depth=8)
    plain.set_scene(sc)
    plain.set_camera(cam)
    with pytest.raises(StateError):
        plain.render_vcm_iteration(1, 1, 100, 8)     # not a vcm_plus context
    ctx = _vcm_ctx(64, 100, r1)
    with pytest.raises(StateError):
        ctx.render_vcm_iteration(1, 1, 100, 8)       # no scene / camera
    ctx.set_scene(sc)
    ctx.set_camera(cam)
    with pytest.raises(InvalidArgument):
        ctx.render_vcm_iteration(1, 1, 99, 8)        # J != samples_per_iteration
    with pytest.raises(InvalidArgument):
        ctx.render_vcm_iteration(1, 1, 100, 6)       # max_depth != the context's
    ctx.render_vcm_iteration(1, 1, 100, 8)
    img, n = ctx.film_mean()
    assert n == 1 and np.isfinite(img).all()


MIXED_CAM = Camera((0.0, 0.1, -0.9), (0.0, -0.1, 1.0), (0.0, 1.0, 0.0), 70.0, 24, 16)
TWO_CAM = Camera((0.0, 1.0, -3.0), (0.0, 0.4, 0.0), (0.0, 1.0, 0.0), 50.0, 20, 16)


@pytest.mark.parametrize("which", ["mixed", "two_lights"])
def test_vcm_other_scenes_match_reference_render(ref, which):
    """Every material path on the eye side (mirror / glass chains, emitter hits
    at depth > 1 with their MIS weight), a chromatic light (the reference
    auto-detects RGB test channels), and two emitters incl. a sphere light
    (emitter pick, sphere sampling in next-event estimation)."""
    sc, cam = (mixed_box(), MIXED_CAM) if which == "mixed" else (two_lights_sphere_emitter(), TWO_CAM)
    npix, J, iters = cam.width * cam.height, 8000, 2
    r1 = 0.002 * bounding_radius(sc)
    ctx = _vcm_ctx(npix, J, r1, channels="rgb" if which == "mixed" else "luminance")
    ctx.set_scene(sc)
    ctx.set_camera(cam)
    for it in range(1, iters + 1):
        ctx.render_vcm_iteration(29, it, J, 8)
    img, _ = ctx.film_mean()
    film, radius, _ = ref.scene(sc.arrays()).render_vcm_plus(cam, 29, iters, 8, J, r0_frac=0.002, n_annuli=2,
                                                             n_sectors=6, alpha_f=0.01, threads=8)
    bad = _compare(img.reshape(-1, 3), film, f"vcm+ {which}")
    assert bad.sum() == 0
    assert np.array_equal(ctx.regions()["radius"], radius)
