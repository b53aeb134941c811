"""C3 end to end on the device: eye pass (Renderer::pixel_pm's camera walk,
integrator.cpp:407-474), light phase, grid + gather + F-test, film
(film.cpp:21-50) -- against the reference.

* eye pass vs the reference's own camera / intersect / Bsdf code
  (oracle/_ref ref_eye_pass): no sin/cos on this walk, so hit points,
  throughputs and emitted radiance must agree to the last bits;
* full iterations vs the oracle session fed the GPU's canonical inputs (its
  fp32 photons and its hit points): counts, decisions, radii exact;
* the film vs the reference's render() (fp64 photons): the north-star
  radiance tolerance (1e-5 relative) on all but a reported handful of pixels
  where an fp32-rounded photon sits on a kernel boundary."""
import numpy as np
import pytest

from helpers import compare_iteration
from paper_2504_04411_b200 import FppmContext
from paper_2504_04411_b200.scene import Camera, bounding_radius, caustic_box, caustic_box_camera, mixed_box

pytestmark = pytest.mark.gpu

MIXED_CAM = Camera((0.0, 0.1, -0.9), (0.0, -0.1, 1.0), (0.0, 1.0, 0.0), 70.0, 48, 32)


def _ctx(npix, J, r1, max_depth=8, **kw):
    return FppmContext(initial_radius=r1, samples_per_iteration=J, n_annuli=2, n_sectors=6, alpha_f=0.01,
                       r_min_base=0.001 * r1, max_depth=max_depth, max_hitpoints=npix, max_photons=8 * J, **kw)


@pytest.mark.parametrize("which", ["caustic", "mixed"])
def test_eye_pass_matches_reference(ref, which):
    sc, cam = (caustic_box(), caustic_box_camera(40)) if which == "caustic" else (mixed_box(), MIXED_CAM)
    npix = cam.width * cam.height
    ctx = _ctx(npix, 1000, 0.002)
    ctx.set_scene(sc)
    ctx.set_camera(cam)
    rs = ref.scene(sc.arrays())
    for it in (1, 2):
        ctx.trace_eye(11, it)
        got = ctx.get_hitpoints(emitted=True)
        want = rs.eye_pass(cam, 11, it, 8)
        assert np.array_equal(got["gathered"], want["gathered"])
        assert np.array_equal(got["eye_depth"], want["eye_depth"])
        assert want["gathered"].mean() > 0.5
        for k in ("pos", "nrm", "wo", "thr", "alb", "emitted"):
            np.testing.assert_array_equal(got[k], want[k], err_msg=k)


def test_render_iterations_match_oracle(port):
    sc, cam = caustic_box(), caustic_box_camera(48)
    npix, J = cam.width * cam.height, 40000
    r1 = 0.002 * bounding_radius(sc)
    ctx = _ctx(npix, J, r1)
    ctx.set_scene(sc)
    ctx.set_camera(cam)
    cfg = dict(n_annuli=2, n_sectors=6, alpha_f=0.01, initial_radius=r1, r_min_base=0.001 * r1,
               samples_per_iteration=J, max_depth=8, threads=8)
    sess = None
    for it in range(1, 5):
        ctx.trace_photons(3, it, J, 8)
        ph = ctx.get_photons()
        ctx.trace_eye(3, it)
        hit = ctx.get_hitpoints()
        if sess is None:
            sess = port.session(cfg, hit)
        else:
            sess.set_hitpoints(hit)
        got, _ = ctx.iterate(it, stats=True)
        ctx.film_add()
        want = sess.iterate(it, ph)
        compare_iteration(got, want)
    img, n = ctx.film_mean()
    assert n == 4 and img.shape == (48, 48, 3) and np.isfinite(img).all() and img.max() > 0


def _attributed_render(ref, sc, cam, J, iters, seed, channels="luminance"):
    """The whole FPPM render on the device against the reference's render()
    (reference defaults 2x6, alpha_F = 0.01, r1 = 0.002 R_bb), with every
    difference attributed.

    Two reference sessions (oracle/_ref: the reference's own PhotonGrid and
    GatherRegion) replay each iteration on the reference eye pass: A with the
    reference tracer's fp64 photons, B with the device's fp32 photons.
      * A reproduces render() bit for bit (film and radii): the harness is the
        reference;
      * the device reproduces B exactly (counts, decisions, radii; fp64 sums
        to summation order): the device is the reference on its inputs;
      * the device's photons are the reference's rounded to fp32 (except
        coordinates within 1e-12 of zero: device vs glibc sin/cos);
    so every pixel whose radius or film differs structurally from render()
    must be a pixel where A and B accept a different photon set or decide
    differently -- a photon whose fp32 rounding crosses a cell, ball, disk,
    annulus or sector boundary.  Everywhere else the film differs only by the
    fp32 rounding of photon power: <= 1e-6 relative (measured ~4e-8)."""
    npix = cam.width * cam.height
    r1 = 0.002 * bounding_radius(sc)
    ctx = _ctx(npix, J, r1, channels=channels)
    ctx.set_scene(sc)
    ctx.set_camera(cam)
    rs = ref.scene(sc.arrays())
    cfg = dict(n_annuli=2, n_sectors=6, alpha_f=0.01, initial_radius=r1, r_min_base=0.001 * r1,
               samples_per_iteration=J, max_depth=8, threads=8, channels=3 if channels == "rgb" else 1)
    sA = sB = None
    film_a, film_b = np.zeros((npix, 3)), np.zeros((npix, 3))
    fp32_px = np.zeros(npix, bool)
    for it in range(1, iters + 1):
        got, _ = ctx.render_iteration(seed, it, J, 8, outputs=True, stats=True)
        hit = ctx.get_hitpoints(emitted=True)
        eye = rs.eye_pass(cam, seed, it, 8)
        for k in ("pos", "nrm", "wo", "thr", "alb", "emitted", "gathered", "eye_depth"):
            assert np.array_equal(hit[k], eye[k]), k
        ph32 = ctx.get_photons()
        ph64 = rs.trace(seed, it, J, 8)
        assert np.array_equal(ph32["depth"], ph64["depth"])
        for k in ("pos", "nrm", "wi", "pow"):
            d = ph32[k] != ph64[k].astype(np.float32)
            assert not (d & (np.abs(ph64[k]) > 1e-12)).any(), k
        if sA is None:
            sA, sB = ref.session(cfg, eye), ref.session(cfg, eye)
        else:
            sA.set_hitpoints(eye)
            sB.set_hitpoints(eye)
        wa, wb = sA.iterate(it, ph64), sB.iterate(it, ph32)
        compare_iteration(got, wb)
        fp32_px |= (wa["radius"] != wb["radius"]) | (wa["accepted"] != wb["accepted"]) | \
            (wa["rejected"] != wb["rejected"]) | (wa["tested"] != wb["tested"])
        film_a = film_a + (eye["emitted"] + wa["radiance"])   # Film::add_iteration (film.cpp:21-26)
        film_b = film_b + (eye["emitted"] + wb["radiance"])
    film, radius, _ = rs.render_fppm(cam, seed, iters, 8, J, r0_frac=0.002, n_annuli=2, n_sectors=6,
                                     alpha_f=0.01, threads=8)
    assert np.array_equal(film_a / iters, film), "session A is not the reference render()"
    assert np.array_equal(wa["radius"], radius)
    img, n = ctx.film_mean()
    assert n == iters
    got_film = img.reshape(-1, 3)
    np.testing.assert_allclose(got_film, film_b / iters, rtol=1e-12, atol=1e-300)
    rel = (np.abs(got_film - film) / np.maximum(np.abs(film), 1e-300)).max(-1)
    bad = rel > 1e-6
    rad = ctx.regions()["radius"]
    unexplained = (bad | (rad != radius)) & ~fp32_px
    mx = rel[~fp32_px].max() if (~fp32_px).any() else 0.0
    print(f"film vs render(): {bad.sum()} of {npix} pixels beyond 1e-6 relative, "
          f"{(rad != radius).sum()} radii differ; fp32 rounding changes the accepted set or a decision at "
          f"{fp32_px.sum()} pixels; unexplained {unexplained.sum()}; max rel elsewhere {mx:.1e}")
    assert not unexplained.any(), np.flatnonzero(unexplained)[:10]
    assert mx <= 1e-6
    return int(fp32_px.sum())


def test_film_matches_reference_render(ref):
    """The whole FPPM render against the reference's render(), every
    difference attributed (see _attributed_render)."""
    sc, cam = caustic_box(), caustic_box_camera(32)
    _attributed_render(ref, sc, cam, 30000, 4, 21)


def test_render_api_errors():
    from paper_2504_04411_b200 import InvalidArgument, StateError, CapacityError
    ctx = _ctx(64, 1000, 0.002)
    with pytest.raises(StateError):
        ctx.film_add()                      # no camera
    with pytest.raises(CapacityError):
        ctx.set_camera(Camera((0, 0, 0), (0, 0, 1), (0, 1, 0), 40.0, 16, 16))   # 256 px > 64
    ctx.set_camera(Camera((0, 0, 0), (0, 0, 1), (0, 1, 0), 40.0, 8, 8))
    with pytest.raises(StateError):
        ctx.trace_eye(1, 1)                 # no scene
    with pytest.raises(InvalidArgument):
        ctx.set_camera(Camera((0, 0, 0), (0, 0, 1), (0, 1, 0), 40.0, 0, 8))
    ctx.set_scene(caustic_box())
    ctx.trace_eye(1, 1)
    img, n = ctx.film_mean()
    assert n == 0 and not img.any()         # Film::mean with no iterations is black


SCENE_TEXT = """camera pos=(0,0.1,-0.9) look=(0,-0.1,1) up=(0,1,0) fov=70 res=40x30
material white lambertian albedo=(0.7,0.7,0.7)
material red lambertian albedo=(0.6,0.12,0.1)
material green lambertian albedo=(0.12,0.5,0.1)
material chrome mirror refl=(0.9,0.9,0.9)
material glass dielectric ior=1.5 tint=(0.98,0.96,0.94)
quad corner=(-1,-1,-1) e1=(0,0,2) e2=(2,0,0) material=white
quad corner=(-1,1,-1) e1=(2,0,0) e2=(0,0,2) material=white
quad corner=(-1,-1,1) e1=(0,2,0) e2=(2,0,0) material=white
quad corner=(-1,-1,-1) e1=(0,2,0) e2=(0,0,2) material=red
quad corner=(1,-1,-1) e1=(0,0,2) e2=(0,2,0) material=green
quad corner=(-0.3,0.99,-0.3) e1=(0.6,0,0) e2=(0,0,0.6) material=white emit=(12,9,6)
sphere center=(-0.4,-0.6,0.3) radius=0.34 material=chrome
sphere center=(0.45,-0.62,-0.1) radius=0.3 material=glass
"""


def test_scene_text_render_matches_reference(ref):
    """A scene in the reference's text format (chromatic light -> the RGB test
    channels the reference auto-detects), rendered on the device and by the
    reference's render(), every difference attributed."""
    from paper_2504_04411_b200.scene_text import parse_scene
    sc, cam = parse_scene(SCENE_TEXT)
    _attributed_render(ref, sc, cam, 20000, 3, 5, channels="rgb")
