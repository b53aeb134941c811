"""GPU parity of the full FPPM iteration (grid + gather + F-test) vs the oracle.

Each test calls the CUDA path through the C ABI and compares with the C
restatement (and, where built, the reference's own code in oracle/_ref) on
identical canonical inputs."""
import numpy as np
import pytest

from helpers import compare_iteration, gpu_context, oracle_cfg
from paper_2504_04411_b200 import WORKLOADS

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("wl_name", ["c1", "c2"])
def test_generator_bitexact(port, wl_name):
    wl = WORKLOADS[wl_name].scaled(raster=8, photons=1 << 15)
    ctx = gpu_context(wl)
    ctx.generate_photons(wl.generator, wl.seed, 3, wl.photons, begin=777)
    got = ctx.get_photons()
    want = port.gen_photons(wl.generator, wl.seed, 3, 777, wl.photons)
    for k in ("pos", "nrm", "wi", "pow", "depth"):
        assert np.array_equal(got[k].view(np.uint32), want[k].view(np.uint32)), k


@pytest.mark.parametrize("kernel", ["fine", "warp", "3d"])
@pytest.mark.parametrize("wl_name,raster,photons,iters", [
    ("c1", 64, 1 << 16, 4),
    ("c2", 64, 1 << 17, 4),
    ("c2", 128, 1 << 19, 3),
])
def test_iterations_match_oracle(port, wl_name, raster, photons, iters, kernel):
    wl = WORKLOADS[wl_name].scaled(raster=raster, photons=photons)
    ctx = gpu_context(wl, gather_kernel=kernel)
    sess = port.session(oracle_cfg(wl), port.gen_raster_hitpoints(wl.raster))
    for it in range(1, iters + 1):
        ctx.generate_photons(wl.generator, wl.seed, it, wl.photons)
        got, summary = ctx.iterate(it, stats=True)
        want = sess.iterate(it, port.gen_photons(wl.generator, wl.seed, it, 0, wl.photons))
        compare_iteration(got, want)
        assert summary["accepted"] == int(want["accepted"].sum())
        assert summary["ambiguous_pairs"] == 0


def test_iterations_match_reference_build(port, ref):
    """Same check against the reference's own PhotonGrid/GatherRegion code."""
    wl = WORKLOADS["c2"].scaled(raster=32, photons=1 << 15)
    ctx = gpu_context(wl)
    sess = ref.session(oracle_cfg(wl), port.gen_raster_hitpoints(wl.raster))
    for it in range(1, 4):
        ctx.generate_photons(wl.generator, wl.seed, it, wl.photons)
        got, _ = ctx.iterate(it, stats=True)
        want = sess.iterate(it, port.gen_photons(wl.generator, wl.seed, it, 0, wl.photons))
        compare_iteration(got, want)


@pytest.mark.parametrize("z_mode,want_bytes", [
    ("zero", 32),        # every photon at z = 0: flat lean records
    ("offset", 32),      # one common non-zero z: flat records, dz != 0 in the ball test
    ("jitter", 48),      # photons off the plane by different amounts: 48-B lean records
    ("signed_zero", 48), # +0.0 and -0.0 are different bit patterns: not flat
])
def test_lean_record_layouts(port, z_mode, want_bytes):
    """The lean fine gather stages 32-B records when every photon shares one
    bit-identical z (common.cuh flat_record) and 48-B records otherwise; both
    layouts give the oracle's iteration (integrator.cpp:388-402)."""
    wl = WORKLOADS["c2"].scaled(raster=64, photons=1 << 17)
    ctx = gpu_context(wl)
    sess = port.session(oracle_cfg(wl), port.gen_raster_hitpoints(wl.raster))
    rng = np.random.default_rng(11)
    for it in range(1, 4):
        ph = port.gen_photons(wl.generator, wl.seed, it, 0, wl.photons)
        pos = ph["pos"].copy()
        if z_mode == "offset":
            pos[:, 2] = np.float32(0.0015)
        elif z_mode == "jitter":
            pos[:, 2] = rng.uniform(-0.004, 0.004, size=pos.shape[0]).astype(np.float32)
        elif z_mode == "signed_zero":
            pos[::2, 2] = np.float32(-0.0)
        ph["pos"] = pos
        ctx.set_photons(ph["pos"], ph["nrm"], ph["wi"], ph["pow"], ph["depth"])
        got, summary = ctx.iterate(it, stats=True)
        assert ctx.record_bytes() == want_bytes
        want = sess.iterate(it, ph)
        compare_iteration(got, want)
        assert summary["accepted"] == int(want["accepted"].sum())
