"""CPU: BASELINE workload definitions and the canonical input generator
(oracle copy; the GPU copy is checked bit for bit in test_gpu_gather.py)."""
import math

import numpy as np

from paper_2504_04411_b200.workloads import C1, C2, WORKLOADS


def test_workloads_match_baseline_configs():
    # BASELINE.json configs[0] / configs[1]
    assert (C1.raster, C1.photons, C1.initial_radius) == (256, 1 << 20, 0.02)
    assert (C1.n_annuli, C1.n_sectors, C1.alpha_f, C1.iterations) == (1, 4, 0.05, 16)
    assert (C2.raster, C2.photons, C2.initial_radius) == (512, 1 << 22, 0.01)
    assert (C2.n_annuli * C2.n_sectors, C2.alpha_f, C2.iterations) == (8, 0.01, 64)
    assert set(WORKLOADS) == {"c1", "c2", "c5"}
    C5 = WORKLOADS["c5"]
    assert (C5.hitpoints, C5.photons, C5.initial_radius) == (1 << 24, 1 << 27, 0.005)   # 16M x 128M
    assert (C5.n_annuli * C5.n_sectors, C5.alpha_f, C5.iterations) == (8, 0.05, 32)
    kw = C2.context_kwargs()
    assert kw["r_min_base"] == 0.001 * C2.initial_radius  # integrator.cpp:125-126
    assert kw["samples_per_iteration"] == C2.photons


def test_pcg32_reference_sequence(port):
    # pcg32_srandom_r(42, 54) first outputs (O'Neill's reference demo)
    want = [0xa15c02b7, 0x7b47f409, 0xba1d3330, 0x83d2f293, 0xbfa4784b, 0xcbed606e]
    got = [port._pcg(42, 54, k) for k in range(6)]
    assert got == want


def test_deterministic_math_accuracy(port):
    rng = np.random.default_rng(0)
    u = rng.random(2000)
    for x in u:
        s, c = np.zeros(1), np.zeros(1)
        import ctypes as C
        port._sincos(float(x), s.ctypes.data_as(C.POINTER(C.c_double)),
                     c.ctypes.data_as(C.POINTER(C.c_double)))
        assert abs(s[0] - math.sin(2 * math.pi * x)) < 2e-15
        assert abs(c[0] - math.cos(2 * math.pi * x)) < 2e-15
    for x in np.concatenate([u, 10 ** rng.uniform(-9, 3, 200)]):
        assert abs(port._log(float(x)) - math.log(x)) <= 4e-16 * max(1.0, abs(math.log(x)))
    for x in rng.uniform(-5, 2, 200):
        assert abs(port._exp(float(x)) - math.exp(x)) <= 4e-16 * math.exp(x)


def test_c1_photon_distribution(port):
    ph = port.gen_photons(1, 0x5EED, 1, 0, 1 << 16)
    p = ph["pos"]
    assert np.all((p[:, :2] >= 0) & (p[:, :2] < 1)) and np.all(p[:, 2] == 0)
    assert abs(p[:, 0].mean() - 0.5) < 0.01 and abs(p[:, 1].mean() - 0.5) < 0.01
    wi = ph["wi"].astype(np.float64)
    assert np.all(wi[:, 2] >= 0)
    assert np.allclose(np.linalg.norm(wi, axis=1), 1.0, atol=1e-6)
    # cosine-distributed: E[cos] = 2/3
    assert abs(wi[:, 2].mean() - 2 / 3) < 0.01
    assert np.all(ph["nrm"] == np.array([0, 0, 1], np.float32)) and np.all(ph["depth"] == 1)


def test_c2_photon_distribution(port):
    n = 1 << 17
    ph = port.gen_photons(2, 0x5EED, 1, 0, n)
    x, y = ph["pos"][:, 0].astype(np.float64), ph["pos"][:, 1].astype(np.float64)
    blob = (x - 0.3) ** 2 + (y - 0.7) ** 2 < (0.15) ** 2
    # 30% Gaussian blob sigma 0.03 at (0.3, 0.7): radius 5 sigma holds ~all of it
    assert abs(blob.mean() - 0.3 - 0.7 * (math.pi * 0.15 ** 2 / 0.5) * (1 / 11)) < 0.01
    step = ~blob
    right = (x[step] > 0.5).mean()
    # step density 10x denser for x > 0.5 (70% component), small blob leakage
    assert abs(right - 10 / 11) < 0.02


def test_raster_hitpoints(port):
    hp = port.gen_raster_hitpoints(8)
    assert hp["pos"][0].tolist() == [1 / 16, 1 / 16, 0.0]
    assert hp["pos"][9].tolist() == [3 / 16, 3 / 16, 0.0]
    assert np.all(hp["nrm"] == [0, 0, 1]) and np.all(hp["eye_depth"] == 1)
