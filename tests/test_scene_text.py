"""The reference's scene text format (scene_parse.cpp) and PFM output
(film.cpp:95-115): our parser against the reference's own parse_scene
(oracle/_ref) -- same arrays for valid scenes, same ParseError messages for
invalid ones (CPU)."""
import numpy as np
import pytest

from paper_2504_04411_b200.scene import caustic_box
from paper_2504_04411_b200.scene_text import ParseError, parse_scene, read_pfm, write_pfm

BOX = """# a box with a glass ball
camera pos=(0.5,0.5,-1.4) look=(0.5,0.5,0) up=(0,1,0) fov=40 res=64x48
material white lambertian albedo=(0.75,0.75,0.75)
material red lambertian albedo=(0.75,0.25,0.25)
material chrome mirror refl=(0.9,0.9,0.9)
material glass dielectric ior=1.5 tint=(0.99,0.97,0.95)
material clear dielectric ior=1.33
quad corner=(0,0,0) e1=(0,0,1) e2=(1,0,0) material=white
quad corner=(0,0,0) e1=(0,1,0) e2=(0,0,1) material=red   # left wall
sphere center=(0.5,0.2,0.5) radius=0.2 material=glass
sphere center=(0.2,0.1,0.7) radius=.1 material=chrome emit=(1,2,3)
quad corner=(0.4,0.999,0.4) e1=(0.2,0,0) e2=(0,0,0.2) material=white emit=(15,15,15)
sphere center=(0.8,0.3,0.3) radius=1e-1 material=clear
arealight shape=quad1 radiance=(0.5,0.5,0.5)
"""

BAD = [
    "bogus x=1",
    "material m lambertian albedo=(1.5,0,0)",
    "material m lambertian",
    "material m lambertian albedo=(1,0,0) extra=3",
    "material m dielectric ior=0.9",
    "material m unknownkind a=1",
    "material m lambertian albedo=(0.5,0.5,0.5)\nmaterial m mirror refl=(1,1,1)",
    "material m lambertian albedo=(0.5,0.5,0.5)\nsphere center=(0,0,0) radius=-1 material=m",
    "material m lambertian albedo=(0.5,0.5,0.5)\nsphere center=(0,0,0) radius=1 material=q",
    "material m lambertian albedo=(0.5,0.5,0.5)\nquad corner=(0,0,0) e1=(1,0,0) e2=(2,0,0) material=m",
    "material m lambertian albedo=(0.5,0.5,0.5)\nquad corner=(0,0,0) e1=(1,0,0) e2=(0,1,0) material=m emit=(-1,0,0)",
    "material m lambertian albedo=(0.5,0.5,0.5)\nsphere center=(0,0,0) radius=1 material=m emit=3",
    "material m lambertian albedo=(0.5,0.5,0.5)\nsphere center=(0,0,0) radius=1 material=m emit=(1,1,1)\n"
    "arealight shape=sphere0 radiance=(1,1,1)",
    "arealight shape=quad7 radiance=(1,1,1)",
    "camera pos=(0,0,0) look=(0,0,1) up=(0,0,1) fov=40 res=8x8",
    "camera pos=(0,0,0) look=(0,0,1) up=(0,1,0) fov=180 res=8x8",
    "camera pos=(0,0,0) look=(0,0,1) up=(0,1,0) fov=40 res=8by8",
    "camera pos=(0,0,0) look=(0,0,1) up=(0,1,0) fov=40 res=0x8",
    "camera pos=(0,0,0 look=(0,0,1) up=(0,1,0) fov=40 res=8x8",
    "camera pos=(0,0,0) pos=(0,0,1) look=(0,0,1) up=(0,1,0) fov=40 res=8x8",
    "camera pos=(0,0,0) look=(0,0,1) up=(0,1,0) fov=inf res=8x8",
    "material m lambertian albedo=(0.5,0.5,0.5)\nsphere center=(0,0,0) radius=abc material=m",
]


def _f(x):
    return repr(float(x))


def _equal(a, b):
    for k in a:
        assert np.array_equal(np.asarray(a[k]), np.asarray(b[k])), k


def test_valid_scene_matches_reference_parser(ref):
    scene, cam = parse_scene(BOX)
    want, wcam = ref.parse_scene(BOX)
    _equal(scene.arrays(), want)
    got_cam = [*cam.position, *cam.look_at, *cam.up, cam.vfov_deg, cam.width, cam.height]
    assert np.array_equal(np.asarray(got_cam, np.float64), wcam)


def test_caustic_box_text_roundtrip(ref):
    """scene.caustic_box() written in the reference's format parses back to the
    same arrays in both parsers."""
    s = caustic_box().arrays()
    names = ["white", "red", "green", "glass"]
    kinds = {0: "lambertian albedo", 2: "dielectric ior=1.5 tint"}
    lines = []
    for i, (k, rgb) in enumerate(zip(s["material_kind"], s["material_rgb"])):
        lines.append(f"material {names[i]} {kinds[int(k)]}=({_f(rgb[0])},{_f(rgb[1])},{_f(rgb[2])})")
    emit = dict(zip(s["emitter_shape"].tolist(), s["emitter_radiance"].tolist()))
    for i, (k, p, m) in enumerate(zip(s["shape_kind"], s["shape"], s["shape_material"])):
        e = f" emit=({_f(emit[i][0])},{_f(emit[i][1])},{_f(emit[i][2])})" if i in emit else ""
        q = [_f(x) for x in p]
        if k == 0:
            lines.append(f"sphere center=({q[0]},{q[1]},{q[2]}) radius={q[3]} material={names[m]}{e}")
        else:
            lines.append(f"quad corner=({q[0]},{q[1]},{q[2]}) e1=({q[3]},{q[4]},{q[5]}) "
                         f"e2=({q[6]},{q[7]},{q[8]}) material={names[m]}{e}")
    text = "\n".join(lines)
    got, _ = parse_scene(text)
    want, _ = ref.parse_scene(text)
    _equal(got.arrays(), want)
    _equal(got.arrays(), s)


@pytest.mark.parametrize("text", BAD)
def test_errors_match_reference_messages(ref, text):
    from oracle import OracleError
    with pytest.raises(OracleError) as want:
        ref.parse_scene(text)
    with pytest.raises(ParseError) as got:
        parse_scene(text)
    assert str(got.value) == str(want.value)


def test_unsupported_primitives_are_rejected():
    for line in ("pointlight pos=(0,1,0) intensity=(1,1,1)",
                 "material p phong diffuse=(0.5,0.5,0.5) specular=(0.2,0.2,0.2) exp=10"):
        with pytest.raises(ParseError, match="not supported"):
            parse_scene(line)


def test_pfm_roundtrip(tmp_path):
    img = np.random.default_rng(0).random((5, 7, 3)) * 10
    write_pfm(tmp_path / "a.pfm", img)
    raw = (tmp_path / "a.pfm").read_bytes()
    assert raw.startswith(b"PF\n7 5\n-1.0\n") and len(raw) == len(b"PF\n7 5\n-1.0\n") + 5 * 7 * 12
    # bottom row first (film.cpp:103)
    first = np.frombuffer(raw[len(b"PF\n7 5\n-1.0\n"):][:12], "<f4")
    assert np.array_equal(first, img[4, 0].astype(np.float32))
    np.testing.assert_array_equal(read_pfm(tmp_path / "a.pfm"), img.astype(np.float32).astype(np.float64))
