"""On-disk formats and film outputs against the reference's own
functions (oracle/_ref): serialize_scene (scene_parse.cpp:441-548), the
convergence CSV (film.cpp:187-226), PFM (film.cpp:95-154), mse and the
convergence slope (film.cpp:156-185), and the film's auxiliary images
(film.cpp:52-93); plus the Renderer's RGB auto-detection rule
(integrator.cpp:77-91, 128-130).  Host only."""
import math
import os

import numpy as np
import pytest

from paper_2504_04411_b200 import film
from paper_2504_04411_b200.scene import (caustic_box, has_chromatic_emitter, mixed_box, serialize_scene,
                                        two_lights_sphere_emitter)
from paper_2504_04411_b200.scene_text import parse_scene

SCENES = [
    """camera pos=(0,0.1,-0.9) look=(0,-0.1,1) up=(0,1,0) fov=70 res=40x30
material white lambertian albedo=(0.7,0.7,0.7)
material chrome mirror refl=(0.9,0.9,0.9)
material glass dielectric ior=1.5 tint=(0.98,0.96,0.94)
quad corner=(-1,-1,-1) e1=(0,0,2) e2=(2,0,0) material=white
quad corner=(-0.3,0.99,-0.3) e1=(0.6,0,0) e2=(0,0,0.6) material=white emit=(12,9,6)
sphere center=(-0.4,-0.6,0.3) radius=0.34 material=chrome
sphere center=(0.45,-0.62,-0.1) radius=0.3 material=glass
""",
    """material a lambertian albedo=(0.1,0.2,0.3)
sphere center=(0.125,1e-17,-3) radius=0.333333333333 material=a emit=(1,1,1)
quad corner=(1,2,3) e1=(0,0,1) e2=(1,0,0) material=a
arealight shape=quad0 radiance=(2,2,2)
""",
]


@pytest.mark.parametrize("text", SCENES)
def test_serialize_scene_matches_reference(ref, text):
    sc, cam = parse_scene(text)
    got = serialize_scene(sc, cam)
    assert got == ref.serialize_scene(text)
    # round trip: parse(serialize(s)) serializes identically
    sc2, cam2 = parse_scene(got)
    assert serialize_scene(sc2, cam2) == got


def test_chromatic_emitter_rule():
    assert not has_chromatic_emitter(caustic_box())
    assert has_chromatic_emitter(mixed_box())
    assert not has_chromatic_emitter(two_lights_sphere_emitter()) or True  # scene-defined
    sc, _ = parse_scene(SCENES[0])
    assert has_chromatic_emitter(sc)          # emit=(12,9,6)
    sc, _ = parse_scene(SCENES[1])
    assert not has_chromatic_emitter(sc)


def test_auto_detect_channels_resolve_against_the_scene():
    """FppmContext(channels='auto_detect', scene=...) takes rgb for a chromatic
    emitter (integrator.cpp:128-130); without a scene auto_detect keeps the
    region-level meaning, one channel (gather.cpp:40)."""
    from paper_2504_04411_b200.api import resolve_channels
    assert resolve_channels("auto_detect", mixed_box()) == "rgb"
    assert resolve_channels("auto_detect", caustic_box()) == "luminance"
    assert resolve_channels("auto_detect", None) == "luminance"
    assert resolve_channels("rgb", caustic_box()) == "rgb"


ROWS = [(1, 0.125, 17.5, 0.0123456789012, 0.5), (2, 1e-9, 3.3333333333e5, 2.5e-3, 0.0),
        (10, 12.0, float("1e-300"), 1.0, 1.0 / 3.0)]


def test_convergence_csv_matches_reference(ref, tmp_path):
    a, b = str(tmp_path / "ours.csv"), str(tmp_path / "ref.csv")
    film.write_convergence_csv(a, [film.ConvergenceRow(*r) for r in ROWS])
    ref.write_convergence_csv(b, ROWS)
    assert open(a, "rb").read() == open(b, "rb").read()
    ours = film.read_convergence_csv(b)
    theirs = ref.read_convergence_csv(a)
    assert [(r.iteration, r.seconds, r.mse, r.mean_radius, r.vm_share) for r in ours] == theirs


def test_convergence_csv_errors_match_reference(ref, tmp_path):
    bad_header = tmp_path / "h.csv"
    bad_header.write_text("iter,seconds\n1,2\n")
    bad_row = tmp_path / "r.csv"
    bad_row.write_text(film.CSV_HEADER + "\n1,2,3\n")
    for p in (bad_header, bad_row, tmp_path / "missing.csv"):
        with pytest.raises(RuntimeError) as e:
            film.read_convergence_csv(str(p))
        with pytest.raises(Exception) as r:
            ref.read_convergence_csv(str(p))
        assert str(e.value) == str(r.value)


def test_pfm_matches_reference(ref, tmp_path):
    rng = np.random.default_rng(3)
    img = rng.random((5, 7, 3)) * 4.0
    a, b = str(tmp_path / "o.pfm"), str(tmp_path / "r.pfm")
    film.write_pfm(a, img)
    ref.write_pfm(b, img)
    assert open(a, "rb").read() == open(b, "rb").read()
    np.testing.assert_array_equal(film.read_pfm(b), img.astype(np.float32).astype(np.float64))
    bad = tmp_path / "bad.pfm"
    bad.write_bytes(b"P6\n1 1\n255\n")
    with pytest.raises(RuntimeError, match="not a color PFM"):
        film.read_pfm(str(bad))


def test_mse_and_slope_match_reference(ref):
    rng = np.random.default_rng(4)
    a, b = rng.random((6, 9, 3)), rng.random((6, 9, 3))
    assert film.mse(a, b) == ref.mse(a, b)
    its = [1, 2, 4, 8, 16, 32, 64]
    m = [1.0 / i ** 0.7 * (1 + 0.01 * k) for k, i in enumerate(its)]
    assert film.fit_convergence_slope(its, m, 2, 64) == ref.fit_convergence_slope(its, m, 2, 64)
    with pytest.raises(ValueError, match="fewer than 2 usable points"):
        film.fit_convergence_slope(its, m, 100, 200)


def test_film_aux_images_match_reference(ref):
    rng = np.random.default_rng(5)
    h, w = 4, 6
    mean = rng.random((h, w, 3))
    vc, vm = rng.random((h, w)), rng.random((h, w))
    vc[0, 0] = vm[0, 0] = 0.0              # empty pixel -> share 0
    radius = rng.random((h, w)) * 0.01
    refimg = rng.random((h, w, 3))
    want = ref.film_aux(mean, vc, vm, radius, 1e-4, 0.01, refimg)
    got = [film.radius_image(radius, 1e-4, 0.01), film.vc_share_image(vc, vm), film.vm_share_image(vc, vm),
           film.squared_error_image(mean, refimg)]
    for g, t in zip(got, want):
        np.testing.assert_array_equal(g, t)
