"""C5 workload generator (BASELINE configs[4]) in the C restatement: the
nearest-hit-point rule against brute force, the tangent-plane restriction,
the cluster/background mixture (CPU)."""
import numpy as np


def test_c5_generator_properties(port):
    c = port.c5(0x5EED, 3000)
    hp = c.hitpoints()
    assert hp["pos"].min() >= 0.0 and hp["pos"].max() < 1.0
    np.testing.assert_allclose(np.linalg.norm(hp["nrm"], axis=1), 1.0, rtol=1e-12)
    ph = c.photons(2, 0, 6000)
    P = ph["pos"].astype(np.float64)
    d2 = ((P[:, None, :] - hp["pos"][None, :, :]) ** 2).sum(-1)
    nn = d2.argmin(1)
    # deposit normal = nearest hit point's normal (exact nearest up to ties)
    assert np.array_equal(ph["nrm"], hp["nrm"][nn].astype(np.float32))
    off = np.abs(((P - hp["pos"][nn]) * hp["nrm"][nn]).sum(1))
    assert (off <= 0.05).mean() > 0.999           # rejection sampling (8 attempts)
    cosi = (ph["wi"].astype(np.float64) * hp["nrm"][nn]).sum(1)
    assert cosi.min() > -1e-6                     # wi in the normal's hemisphere
    inside = ((P >= 0) & (P < 1)).all(1)
    assert 0.9 < inside.mean() <= 1.0
    # 20 % uniform background: clustered photons have near neighbours
    assert np.array_equal(ph["depth"], np.ones(6000, np.uint32))


def test_c5_streams_are_counter_based(port):
    c = port.c5(7, 1000)
    a = c.photons(3, 0, 500)
    b = c.photons(3, 200, 300)
    for k in a:
        assert np.array_equal(a[k][200:], b[k]), k
    h = c.hitpoints(100, 50)
    assert np.array_equal(h["pos"], c.hitpoints()["pos"][100:150])
