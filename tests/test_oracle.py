"""CPU: pin the oracle (plain-C restatement) against the reference.

Two independent pins:
  * the committed golden fixtures (tests/golden/golden.json, generated from
    the reference's own sources by tests/golden/make_golden.py), and
  * the reference build itself (oracle/_ref), when present, on fresh random
    inputs: grid keys/permutation, query order, sector binning, quantiles and
    whole FPPM iterations must agree bit for bit.
"""
import json
import math
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = json.load(open(os.path.join(HERE, "golden", "golden.json")))


def fh(s):
    return float.fromhex(s)


# ------------------------------------------------------------------ golden vectors
def test_sector_index_golden(port):
    for c in GOLDEN["sector_index"]:
        assert port.sector_index(c["u"], c["v"], c["r"], c["na"], c["ns"]) == c["sector"], c


def test_sector_index_errors(port):
    from oracle import DomainError, InvalidArgument
    with pytest.raises(DomainError):
        port.sector_index(1.1, 0.0, 1.0, 2, 6)
    with pytest.raises(InvalidArgument):
        port.sector_index(0.5, 0.0, 1.0, 0, 6)


def test_quantiles_golden(port):
    for c in GOLDEN["f_quantile"]:
        assert port.f_quantile(c["p"], c["d1"], c["d2"]) == fh(c["value"]), c
    for c in GOLDEN["chi2_quantile"]:
        assert port.chi2_quantile(c["p"], c["df"]) == fh(c["value"]), c


def test_quantile_closed_forms(port):
    # test_special_functions.cpp:41-64 and acceptance A1 (acceptance.cpp:296-303)
    assert math.isclose(port.chi2_quantile(0.5, 2.0), 2 * math.log(2), rel_tol=1e-8)
    assert math.isclose(port.chi2_quantile(0.99, 11.0), 24.724, rel_tol=5e-4)
    assert math.isclose(port.f_quantile(0.95, 2.0, 2.0), 19.0, rel_tol=1e-8)
    assert math.isclose(port.f_quantile(0.5, 1.0, 1.0), 1.0, rel_tol=1e-8)
    q = port.f_quantile(0.99, 11.0, 1e9)
    assert 2.24 < q < 2.26
    assert math.isclose(q, port.chi2_quantile(0.99, 11.0) / 11.0, rel_tol=1e-6)
    # SURVEY §8a critical values
    assert port.f_quantile(0.95, 3, 4 * (2 ** 20 - 1)) == 2.6049114173923344
    assert port.f_quantile(0.99, 7, 8 * (2 ** 22 - 1)) == 2.6393295580831913
    assert port.f_quantile(0.95, 7, 8 * (2 ** 27 - 1)) == 2.0095914927628806
    assert port.f_quantile(0.99, 11, 12 * 4095) == 2.2480842368732192


def test_quantile_round_trips(port):
    for p in (0.05, 0.5, 0.9, 0.99, 0.999):
        for df in (1.0, 2.0, 5.0, 11.0, 100.0):
            assert math.isclose(port.chi2_cdf(port.chi2_quantile(p, df), df), p, rel_tol=1e-7)
        for d1 in (1.0, 2.0, 11.0, 40.0):
            for d2 in (1.0, 2.0, 11.0, 1188.0, 1e8):
                assert math.isclose(port.f_cdf(port.f_quantile(p, d1, d2), d1, d2), p, rel_tol=1e-7)


def test_f_statistic_cases(port):
    h = GOLDEN["f_statistic_hand"]
    assert port.f_statistic(h["count"], h["sum"], h["sum_sq"], h["m"]) == fh(h["value"])
    assert math.isclose(fh(h["value"]), 4.5, rel_tol=1e-12)  # test_stat_tests.cpp:65-70
    assert port.f_statistic([2, 2], [4.0, 4.0], [8.0, 8.0], 2) == 0.0  # constant groups
    assert math.isinf(port.f_statistic([2, 2], [4.0, 6.0], [8.0, 18.0], 2))  # zero within
    assert port.f_statistic([0] * 4, [0.0] * 4, [0.0] * 4, 100) == 0.0


def test_schedule_and_frames_golden(port):
    for c in GOLDEN["schedule_radius"]:
        assert port.schedule_radius(c["base"], c["alpha"], c["i"]) == fh(c["value"])
    # test_gather.cpp:98-106: floor after iteration 3 is 4^-1/8
    assert math.isclose(port.schedule_radius(1.0, 0.75, 4), 4 ** -0.125, rel_tol=1e-12)
    for c in GOLDEN["frames"]:
        u, v = port.build_frame(np.array([fh(x) for x in c["n"]]))
        assert [x.hex() for x in u] == c["u"] and [x.hex() for x in v] == c["v"]


def test_grid_golden(port):
    gg = GOLDEN["grid"]
    pos = np.array(gg["pos"], np.float32).astype(np.float64)
    g = port.grid_build(pos, gg["cell"])
    keys, b, e, order = g.export()
    assert [int(k) for k in keys] == gg["keys"]
    assert b.tolist() == gg["begin"] and e.tolist() == gg["end"] and order.tolist() == gg["order"]
    for c, r, want in zip(gg["centers"], gg["radii"], gg["queries"]):
        assert g.query_ball(np.array(c), r).tolist() == want


@pytest.mark.parametrize("ri", [0, 1])
def test_fppm_runs_golden(port, ri):
    run = GOLDEN["runs"][ri]
    hp = port.gen_raster_hitpoints(run["raster"])
    cfg = dict(n_annuli=run["n_annuli"], n_sectors=run["n_sectors"], alpha_f=run["alpha_f"],
               initial_radius=run["initial_radius"], r_min_base=0.001 * run["initial_radius"],
               samples_per_iteration=run["photons"], threads=2)
    sess = port.session(cfg, hp)
    for it in run["iterations"]:
        ph = port.gen_photons(run["workload"], run["seed"], it["iteration"], 0, run["photons"])
        assert int(np.bitwise_xor.reduce(ph["pos"].view(np.uint32).ravel())) == it["photon_pos_digest"]
        out = sess.iterate(it["iteration"], ph)
        assert out["accepted"].tolist() == it["accepted"]
        assert out["rejected"].tolist() == it["rejected"]
        assert out["tested"].tolist() == it["tested"]
        assert out["t"].tolist() == it["t"]
        assert [x.hex() for x in out["radius"]] == it["radius"]
        assert [x.hex() for x in out["critical"]] == it["critical"]
        assert np.array_equal(out["flux"], np.array(it["flux"]))


# ------------------------------------------------------------------ vs the reference build
def test_port_matches_reference_scalars(port, ref):
    rng = np.random.default_rng(3)
    for _ in range(2000):
        r = 10 ** rng.uniform(-3, 1)
        u, v = rng.uniform(-r, r, 2) / math.sqrt(2)
        na, ns = int(rng.integers(1, 4)), int(rng.integers(1, 13))
        assert port.sector_index(u, v, r, na, ns) == ref.sector_index(u, v, r, na, ns)
    for _ in range(50):
        p = rng.uniform(0.5, 0.999)
        d1 = float(rng.integers(1, 40))
        d2 = float(rng.integers(2, 10 ** int(rng.integers(1, 9))))
        assert port.f_quantile(p, d1, d2) == ref.f_quantile(p, d1, d2)


def test_port_matches_reference_grid(port, ref):
    rng = np.random.default_rng(11)
    for n, ext, cell in ((3000, 2.0, 0.25), (5000, 1.0, 0.05), (1, 1.0, 0.5), (0, 1.0, 0.5)):
        pos = (ext * (2 * rng.random((n, 3)) - 1)).astype(np.float32).astype(np.float64)
        a, b = port.grid_build(pos, cell), ref.grid_build(pos, cell)
        for x, y in zip(a.export(), b.export()):
            assert np.array_equal(x, y)
        for _ in range(30):
            c = 1.2 * ext * (2 * rng.random(3) - 1)
            r = cell * rng.random()
            assert np.array_equal(a.query_ball(c, r), b.query_ball(c, r))


@pytest.mark.parametrize("wl,W,N,na,ns,alpha_f,r0,override", [
    (1, 32, 1 << 14, 1, 4, 0.05, 0.05, 0),
    (2, 32, 1 << 14, 2, 4, 0.01, 0.03, 0),
    (2, 24, 1 << 13, 2, 6, 0.01, 0.04, 0),
    (1, 16, 1 << 12, 2, 6, 0.01, 0.08, 1),
    (1, 16, 1 << 12, 2, 6, 0.01, 0.08, 2),
])
def test_port_matches_reference_fppm(port, ref, wl, W, N, na, ns, alpha_f, r0, override):
    hp = port.gen_raster_hitpoints(W)
    cfg = dict(n_annuli=na, n_sectors=ns, alpha_f=alpha_f, initial_radius=r0,
               r_min_base=0.001 * r0, samples_per_iteration=N, override_decision=override,
               threads=4)
    sp, sr = port.session(cfg, hp), ref.session(cfg, hp)
    for it in range(1, 4):
        ph = port.gen_photons(wl, 0x5EED, it, 0, N)
        a, b = sp.iterate(it, ph), sr.iterate(it, ph)
        for k in a:
            if k != "times":
                assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("over", [
    dict(), dict(channels=3), dict(policy=1, alpha_chi2=0.05), dict(policy=2),
    dict(max_depth=4, n_annuli=3, n_sectors=5), dict(samples_per_iteration=1),
])
def test_port_matches_reference_general_scene(port, ref, over):
    """Arbitrary normals, depth filter, back faces, not-gathered hit points and
    every end-of-iteration policy (gather.cpp:90/114/138): bit-identical."""
    from scenes import scene3d
    hit, _ = scene3d(11, H=500, N=20000)
    cfg = dict(n_annuli=2, n_sectors=6, alpha_f=0.05, initial_radius=0.03, r_min_base=3e-5,
               samples_per_iteration=20000, threads=4)
    cfg.update(over)
    sp, sr = port.session(cfg, hit), ref.session(cfg, hit)
    for it in range(1, 4):
        ph = scene3d(20 + it, H=500, N=20000)[1]
        a, b = sp.iterate(it, ph), sr.iterate(it, ph)
        assert a["accepted"].sum() > 0
        for k in a:
            if k != "times":
                assert np.array_equal(a[k], b[k]), k


def test_thread_count_invariance(port):
    """test_integrator.cpp:267-293 analogue: results independent of threads."""
    hp = port.gen_raster_hitpoints(24)
    base = dict(n_annuli=2, n_sectors=4, alpha_f=0.01, initial_radius=0.04, r_min_base=4e-5,
                samples_per_iteration=1 << 13)
    s1 = port.session(dict(base, threads=1), hp)
    s8 = port.session(dict(base, threads=8), hp)
    for it in (1, 2):
        ph = port.gen_photons(2, 7, it, 0, 1 << 13)
        a, b = s1.iterate(it, ph), s8.iterate(it, ph)
        for k in a:
            if k != "times":
                assert np.array_equal(a[k], b[k]), k


def test_mis_weight_merge_matches_reference(port, ref):
    """path.cpp:103-111 merge weight with eta_vm = n_vm pi r^2 (integrator.cpp:503)."""
    rng = np.random.default_rng(5)
    for beta in (1.0, 2.0):
        for _ in range(300):
            scale = rng.choice([0.0, 1e-3, 1.0, 1e3], 4)
            args = (int(rng.integers(0, 1 << 22)), beta, float(rng.random() * 0.05),
                    *map(float, rng.random(4) * scale), float(rng.random()), float(rng.random()))
            a, b = port.mis_weight_merge(*args), ref.mis_weight_merge(*args)
            assert a == b or (np.isnan(a) and np.isnan(b)), args


@pytest.mark.parametrize("beta", [1.0, 2.0])
def test_port_matches_reference_vcm_plus(port, ref, beta):
    """VCM+ merge stage: photon values weighted by the MIS merge weight of the
    tested radius (integrator.cpp:595-627); canonical raster + C2 photons with
    random MIS partials, bit-identical to the reference build."""
    W, N = 24, 1 << 13
    hp = port.gen_raster_hitpoints(W)
    cfg = dict(n_annuli=2, n_sectors=4, alpha_f=0.01, initial_radius=0.04, r_min_base=4e-5,
               samples_per_iteration=N, threads=4, vcm_plus=1, mis_n_vm=N, mis_beta=beta)
    sp, sr = port.session(cfg, hp), ref.session(cfg, hp)
    rng = np.random.default_rng(9)
    ev, em = rng.random(W * W) * 2, rng.random(W * W)
    sp.set_eye_mis(ev, em)
    sr.set_eye_mis(ev, em)
    for it in range(1, 4):
        ph = port.gen_photons(2, 0x5EED, it, 0, N)
        pv, pm, pc = rng.random(N) * 3, rng.random(N), rng.random(N)
        sp.set_photon_mis(pv, pm, pc)
        sr.set_photon_mis(pv, pm, pc)
        a, b = sp.iterate(it, ph), sr.iterate(it, ph)
        assert a["accepted"].sum() > 0
        for k in a:
            if k != "times":
                assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("algorithm", ["fppm", "vcm_plus"])
def test_reference_render_thread_invariance(ref, algorithm):
    """The reference's own render() -- the checker of the device's C3 / C4
    renders (tests/test_gpu_render.py, tests/test_gpu_vcm_render.py) -- is
    deterministic across thread counts (test_integrator.cpp:267-293), so its
    film is a fixed target for a given seed."""
    from paper_2504_04411_b200.scene import caustic_box, caustic_box_camera
    rs = ref.scene(caustic_box().arrays())
    cam = caustic_box_camera(8)
    render = rs.render_fppm if algorithm == "fppm" else rs.render_vcm_plus
    f1, r1, _ = render(cam, 3, 2, 8, 4000, r0_frac=0.01, n_annuli=1, n_sectors=4, alpha_f=0.05, threads=1)
    f4, r4, _ = render(cam, 3, 2, 8, 4000, r0_frac=0.01, n_annuli=1, n_sectors=4, alpha_f=0.05, threads=4)
    assert np.isfinite(f1).all() and f1.mean() > 0
    assert np.array_equal(f1, f4) and np.array_equal(r1, r4)
