"""The device renderer's algorithm family (render.py) against the reference:
the degeneracy identities of test_integrator.cpp:295-364 run on the device
(FPPM with forced rejection == SPPM photon for photon, VCM+ with forced
rejection == VCM, holding every test keeps r_1), SPPM / VCM / CPPM films
against the reference's own render(), the film's vc / vm split totals
(integrator.cpp:205-224, film.cpp:28-31), and the furnace box's closed form
(test_integrator.cpp:217-265)."""
import numpy as np
import pytest

from paper_2504_04411_b200 import FppmContext  # noqa: F401  (loads the library)
from paper_2504_04411_b200.api import RadiusSchedule, TestConfig
from paper_2504_04411_b200.render import render
from paper_2504_04411_b200.scene import bounding_radius, caustic_box, caustic_box_camera, schedule_radius_host
from paper_2504_04411_b200.scene_text import parse_scene

pytestmark = pytest.mark.gpu


def furnace_text(albedo=0.5, emit=1.0):
    """test_integrator.cpp:31-46: a closed cube, every face emits and reflects."""
    e = f"({emit},{emit},{emit})"
    a = f"({albedo},{albedo},{albedo})"
    return ("camera pos=(0,0,0) look=(0,0,1) up=(0,1,0) fov=60 res=8x8\n"
            f"material wall lambertian albedo={a}\n"
            f"quad corner=(-1,-1,-1) e1=(0,0,2) e2=(2,0,0) material=wall emit={e}\n"
            f"quad corner=(-1,1,-1) e1=(2,0,0) e2=(0,0,2) material=wall emit={e}\n"
            f"quad corner=(-1,-1,-1) e1=(2,0,0) e2=(0,2,0) material=wall emit={e}\n"
            f"quad corner=(-1,-1,1) e1=(0,2,0) e2=(2,0,0) material=wall emit={e}\n"
            f"quad corner=(-1,-1,-1) e1=(0,2,0) e2=(0,0,2) material=wall emit={e}\n"
            f"quad corner=(1,-1,-1) e1=(0,0,2) e2=(0,2,0) material=wall emit={e}\n")


def furnace_truncated(albedo, emit, max_depth):
    s, term = 0.0, emit
    for _ in range(max_depth):
        s += term
        term *= albedo
    return s


def test_forced_rejection_reproduces_the_fixed_schedule():
    """test_integrator.cpp:295-324 on the device: with the floor at r_1 the
    rejected branch is the schedule, so FPPM(always_reject) == SPPM bitwise."""
    sc, cam = parse_scene(furnace_text())
    r1 = 0.01 * bounding_radius(sc)
    iters = 8
    forced = render(sc, cam, "fppm", iters, seed=7, r0_frac=0.01, light_paths=4096,
                    test=TestConfig(override_decision="always_reject"), schedule=RadiusSchedule(r_min_base=r1))
    fixed = render(sc, cam, "sppm", iters, seed=7, r0_frac=0.01, light_paths=4096)
    assert np.array_equal(forced.image, fixed.image)
    for rf, rs in zip(forced.reports, fixed.reports):
        want = schedule_radius_host(r1, 0.75, rf.iteration + 1)
        assert np.all(rf.radius == want) and np.all(rs.radius == want)
        assert np.all(rf.rejected == 1)


def test_forced_rejection_in_vcm_plus_reproduces_vcm():
    """test_integrator.cpp:326-349 on the device."""
    sc, cam = parse_scene(furnace_text())
    r1 = 0.01 * bounding_radius(sc)
    forced = render(sc, cam, "vcm_plus", 6, seed=7, r0_frac=0.01,
                    test=TestConfig(override_decision="always_reject"), schedule=RadiusSchedule(r_min_base=r1))
    fixed = render(sc, cam, "vcm", 6, seed=7, r0_frac=0.01)
    assert np.array_equal(forced.image, fixed.image)
    for rf, rs in zip(forced.reports, fixed.reports):
        want = schedule_radius_host(r1, 0.75, rf.iteration + 1)
        assert np.all(rf.radius == want) and np.all(rs.radius == want)


def test_holding_every_test_keeps_r1():
    """test_integrator.cpp:351-364."""
    sc, cam = parse_scene(furnace_text())
    r1 = 0.01 * bounding_radius(sc)
    res = render(sc, cam, "fppm", 5, seed=7, r0_frac=0.01, light_paths=2048,
                 test=TestConfig(override_decision="never_reject"))
    for rep in res.reports:
        assert np.all(rep.radius == r1) and not rep.rejected.any()


@pytest.mark.parametrize("algorithm", ["sppm", "cppm", "vcm", "fppm", "vcm_plus"])
def test_algorithms_match_reference_render(ref, algorithm):
    """Each algorithm's film and final radii against the reference render()
    (caustic box 24^2): within 1e-6 relative on every pixel (measured <= 1e-7;
    the device photons are the reference's rounded to fp32), radii identical,
    the vc / vm split totals within 1e-6 like the film (the merge share
    carries the photon powers' fp32 rounding)."""
    sc, cam = caustic_box(), caustic_box_camera(24)
    J, iters = 6000, 3
    got = render(sc, cam, algorithm, iters, seed=11, max_depth=8, light_paths=J, r0_frac=0.002,
                 test=TestConfig(n_annuli=2, n_sectors=6, alpha_f=0.01))
    film, radius, vc, vm = ref.scene(sc.arrays()).render_ex(cam, algorithm, 11, iters, 8, J, r0_frac=0.002,
                                                            n_annuli=2, n_sectors=6, alpha_f=0.01, threads=8)
    g = got.image.reshape(-1, 3)
    rel = (np.abs(g - film) / np.maximum(np.abs(film), 1e-300)).max(-1)
    print(f"{algorithm}: max rel film diff {rel.max():.2e}, radii differ at {(got.reports[-1].radius != radius).sum()}")
    assert (rel <= 1e-6).all()
    assert np.array_equal(got.reports[-1].radius, radius)
    np.testing.assert_allclose(got.vc_total.ravel(), vc, rtol=1e-6, atol=1e-300)
    np.testing.assert_allclose(got.vm_total.ravel(), vm, rtol=1e-6, atol=1e-300)


def test_reports_and_film_agree_on_the_split():
    """test_integrator.cpp:386-411 (luminance is linear: vc + vm is the image)."""
    sc, cam = caustic_box(), caustic_box_camera(16)
    res = render(sc, cam, "vcm", 5, seed=3, max_depth=8, light_paths=4000, r0_frac=0.01)
    rep_vc = sum(r.vc_luminance for r in res.reports)
    rep_vm = sum(r.vm_luminance for r in res.reports)
    lum = (0.2126 * res.image[..., 0] + 0.7152 * res.image[..., 1] + 0.0722 * res.image[..., 2]).sum() * 5
    assert rep_vc > 0 and rep_vm > 0
    assert abs(res.vc_total.sum() - rep_vc) <= 1e-9 * rep_vc
    assert abs(res.vm_total.sum() - rep_vm) <= 1e-9 * rep_vm
    assert abs(lum - (rep_vc + rep_vm)) <= 1e-9 * lum


@pytest.mark.parametrize("algorithm,iters,J,r0,eps", [("fppm", 250, 2048, 0.05, 0.03),
                                                      ("sppm", 250, 2048, 0.05, 0.04),
                                                      ("vcm_plus", 150, 0, 0.05, 0.015)])
def test_furnace_closed_form(algorithm, iters, J, r0, eps):
    """test_integrator.cpp:217-265: every estimator converges to the truncated
    series L_e (1 + rho + ... + rho^9) in the furnace box."""
    sc, cam = parse_scene(furnace_text())
    expected = furnace_truncated(0.5, 1.0, 10)
    res = render(sc, cam, algorithm, iters, seed=7, max_depth=10, light_paths=J, r0_frac=r0)
    img = res.image
    assert np.isfinite(img).all() and (img >= 0).all()
    lum = (0.2126 * img[..., 0] + 0.7152 * img[..., 1] + 0.0722 * img[..., 2]).mean()
    assert abs(lum - expected) <= eps * expected, (lum, expected)
