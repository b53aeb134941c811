"""Scene description (paper_2504_04411_b200.scene) and the reference tracer
used as the checker for the GPU light phase (CPU, no GPU needed)."""
import numpy as np
import pytest

from paper_2504_04411_b200.scene import (DIELECTRIC, LAMBERTIAN, Scene, caustic_box, mixed_box,
                                         two_lights_sphere_emitter)


def test_scene_arrays_and_validation():
    s = caustic_box()
    a = s.arrays()
    assert a["shape"].shape == (7, 9) and a["material_rgb"].shape == (4, 3)
    assert list(a["emitter_shape"]) == [6]
    # the light quad faces down (e1 x e2 along -y, scene_geometry.cpp fill_hit)
    e1, e2 = a["shape"][6, 3:6], a["shape"][6, 6:9]
    assert np.cross(e1, e2)[1] < 0
    with pytest.raises(ValueError):
        Scene().material(7)
    with pytest.raises(ValueError):
        Scene().material(DIELECTRIC, ior=0.9)          # scene_parse: ior must exceed 1
    with pytest.raises(ValueError):
        Scene().sphere((0, 0, 0), 0.0, 0)


@pytest.mark.parametrize("make", [caustic_box, mixed_box, two_lights_sphere_emitter])
def test_reference_tracer_invariants(ref, make):
    sc = make()
    rs = ref.scene(sc.arrays())
    n_paths, max_depth = 4000, 6
    t = rs.trace(42, 3, n_paths, max_depth, threads=4)
    n = len(t["depth"])
    assert n > 0
    path, depth = t["path"].astype(np.int64), t["depth"].astype(np.int64)
    assert np.all(np.diff(path) >= 0)                               # flattened in path order
    same = np.diff(path) == 0
    assert np.all(np.diff(depth)[same] > 0)                         # depth grows along a path
    assert depth.min() >= 1 and depth.max() <= max_depth - 1        # light_depth = max_depth - 1
    np.testing.assert_allclose(np.linalg.norm(t["nrm"], axis=1), 1.0, rtol=1e-12)
    np.testing.assert_allclose(np.linalg.norm(t["wi"], axis=1), 1.0, rtol=1e-12)
    assert np.all(np.einsum("ij,ij->i", t["nrm"], t["wi"]) > 0)    # shading normal faces wi
    assert np.all(t["pow"] >= 0)
    # deposits are only on Lambertian surfaces (Bsdf::is_delta_only)
    kinds = np.asarray(sc.material_kind)
    assert set(np.unique(kinds)) >= {LAMBERTIAN}
    # same (seed, iteration, path) -> same vertices, independent of the range split
    half = rs.trace(42, 3, n_paths // 2, max_depth, threads=1, begin=n_paths // 2)
    sel = path >= n_paths // 2
    np.testing.assert_array_equal(half["pos"], t["pos"][sel])
    np.testing.assert_array_equal(half["path"], t["path"][sel])


def test_reference_tracer_power_closed_box(ref):
    """First-bounce photon power in a closed, all-diffuse room equals the
    emitted flux Phi = L * pi * A (each path carries L*pi*A / pick_prob and
    every path hits a wall): a statistical check of emission + throughput."""
    s = Scene()
    w = s.material(LAMBERTIAN, (0.5, 0.5, 0.5))
    s.quad((-1, -1, -1), (0, 0, 2), (2, 0, 0), w)
    s.quad((-1, 1, -1), (2, 0, 0), (0, 0, 2), w)
    s.quad((-1, -1, -1), (2, 0, 0), (0, 2, 0), w)
    s.quad((-1, -1, 1), (0, 2, 0), (2, 0, 0), w)
    s.quad((-1, -1, -1), (0, 2, 0), (0, 0, 2), w)
    s.quad((1, -1, -1), (0, 0, 2), (0, 2, 0), w)
    s.quad((-0.2, 0.99, -0.2), (0.4, 0, 0), (0, 0, 0.4), w, emit=(2.0, 2.0, 2.0))
    t = ref.scene(s.arrays()).trace(9, 1, 20000, 3, threads=4)
    first = t["depth"] == 1
    assert first.sum() == 20000
    phi = 2.0 * np.pi * 0.16
    np.testing.assert_allclose(t["pow"][first].mean(0), phi, rtol=1e-12)
