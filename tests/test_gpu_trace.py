"""GPU photon emission + tracing (Renderer::light_phase, integrator.cpp:230-265;
trace_light_subpath, path.cpp:388-449) against the reference's OWN tracer
(oracle/_ref: the unmodified Scene/build_accel/trace_light_subpath sources)
on the same seeds, then the traced photons through the FPPM iteration.

Tolerance: the device evaluates sin/cos with CUDA's libm (<= 2 ulp) instead of
glibc, so directions differ in the last fp64 bits; every discrete decision
(hit primitive, Fresnel / roulette choice, deposit count and depth) must
match exactly, and the stored fp32 vertex fields within 1e-5 relative
(BASELINE north_star fp32 tolerance)."""
import numpy as np
import pytest

from helpers import compare_iteration
from paper_2504_04411_b200 import CapacityError, FppmContext, StateError
from paper_2504_04411_b200.scene import caustic_box, mixed_box, two_lights_sphere_emitter

pytestmark = pytest.mark.gpu

SCENES = {"caustic": caustic_box, "mixed": mixed_box, "two_lights": two_lights_sphere_emitter}


def _ctx(max_photons=1 << 20, **kw):
    return FppmContext(initial_radius=0.02, samples_per_iteration=1 << 16, n_annuli=1, n_sectors=4,
                       alpha_f=0.05, max_hitpoints=1 << 14, max_photons=max_photons, **kw)


def _close(got, want, name, rtol=1e-5, atol=1e-6):
    """fp32 fields within rtol; returns how many are not bit-identical to the
    reference's fp64 value rounded to fp32, ignoring |x| < 1e-12 (points on
    the z=0 / x=0 walls come out as +-1e-17 instead of 0 when one fp64 ulp of
    the ray direction differs)."""
    w = want.astype(np.float32)
    bad = np.abs(got.astype(np.float64) - w) > rtol * np.abs(w) + atol
    assert not bad.any(), f"{name}: {bad.sum()} values off, first rows {np.flatnonzero(bad.any(-1))[:5]}"
    tiny = (np.abs(want) < 1e-12) & (np.abs(got.astype(np.float64) - want) < 1e-15)
    return int(((got != w) & ~tiny).sum())


@pytest.mark.parametrize("scene", list(SCENES))
@pytest.mark.parametrize("max_depth", [8, 3])
def test_trace_matches_reference(ref, scene, max_depth):
    sc = SCENES[scene]()
    ctx = _ctx()
    ctx.set_scene(sc)
    rs = ref.scene(sc.arrays())
    n_paths = 30000
    for it in (1, 2):
        n = ctx.trace_photons(0xC0FFEE, it, n_paths, max_depth)
        want = rs.trace(0xC0FFEE, it, n_paths, max_depth, threads=8)
        assert n == len(want["depth"]) and n > 0
        got = ctx.get_photons()
        assert np.array_equal(got["depth"], want["depth"])
        ulps = sum(_close(got[k], want[k], k) for k in ("pos", "nrm", "wi", "pow"))
        # fp32 fields that are not bit-identical (a rounding-boundary case
        # needs an fp64 last-bit difference to straddle an fp32 tie)
        print(f"{scene} d={max_depth} it={it}: {n} photons, {ulps} fp32 fields not bit-identical")
        assert ulps <= 1e-4 * 12 * n


def test_trace_deterministic_and_iteration_keyed():
    sc = caustic_box()
    ctx = _ctx()
    ctx.set_scene(sc)
    ctx.trace_photons(5, 1, 20000, 8)
    a = ctx.get_photons()
    ctx.trace_photons(5, 1, 20000, 8)
    b = ctx.get_photons()
    for k in a:
        assert np.array_equal(a[k], b[k]), k
    ctx.trace_photons(5, 2, 20000, 8)
    c = ctx.get_photons()
    assert len(c["depth"]) != len(a["depth"]) or not np.array_equal(c["pos"], a["pos"])


@pytest.mark.parametrize("beta", [1.0, 2.0])
def test_trace_vcm_partials_match_reference(ref, beta):
    sc = mixed_box()
    n_paths, r = 20000, 0.015
    ctx = _ctx(vcm_plus=True, mis_n_vm=n_paths, mis_beta=beta)
    ctx.set_scene(sc)
    n = ctx.trace_photons(77, 3, n_paths, 8, mis_radius=r)
    want = ref.scene(sc.arrays()).trace(77, 3, n_paths, 8, n_vm=n_paths, beta=beta,
                                        eta_vm=n_paths * np.pi * r * r, threads=8)
    assert n == len(want["depth"])
    got = ctx.get_photon_mis()
    for i, k in enumerate(("d_vcm", "d_vm", "cont")):
        np.testing.assert_allclose(got[k], want["mis"][:, i], rtol=1e-7, atol=0, err_msg=k)


def test_traced_photons_through_fppm_iterations(port):
    """light phase -> grid -> gather -> F-test on scene surfaces: hit points
    are diffuse surface points of the caustic box (traced vertices of another
    seed); each iteration's GPU-traced photons also feed the oracle session."""
    sc = caustic_box()
    ctx = _ctx()
    ctx.set_scene(sc)
    ctx.trace_photons(1234, 0, 4000, 4)
    hp = ctx.get_photons()
    H = min(len(hp["depth"]), 3000)
    hit = dict(pos=hp["pos"][:H].astype(np.float64), nrm=hp["nrm"][:H].astype(np.float64),
               wo=hp["wi"][:H].astype(np.float64), thr=np.ones((H, 3)), alb=np.full((H, 3), 0.75),
               eye_depth=np.ones(H, np.uint32), gathered=np.ones(H, np.uint8))
    J = 60000
    cfg = dict(n_annuli=1, n_sectors=4, alpha_f=0.05, initial_radius=0.02, r_min_base=2e-5,
               samples_per_iteration=J, threads=8)
    ctx.set_hitpoints(hit["pos"], hit["nrm"], hit["wo"], hit["thr"], hit["alb"], hit["eye_depth"],
                      hit["gathered"])
    ctx.set_samples_per_iteration(J)
    sess = port.session(cfg, hit)
    for it in range(1, 4):
        ctx.trace_photons(99, it, J, 8)
        ph = ctx.get_photons()
        got, _ = ctx.iterate(it, stats=True)
        want = sess.iterate(it, ph)
        compare_iteration(got, want)
        assert (want["stat_count"].sum(-1) > 0).sum() > H // 4


def test_trace_errors():
    ctx = _ctx(max_photons=1000)
    with pytest.raises(StateError):
        ctx.trace_photons(1, 1, 10, 8)
    ctx.set_scene(caustic_box())
    with pytest.raises(CapacityError):
        ctx.trace_photons(1, 1, 100000, 8)
    assert ctx.trace_photons(1, 1, 1000, 1) == 0      # light_depth = max_depth - 1 = 0
    assert ctx.trace_photons(1, 1, 0, 8) == 0
