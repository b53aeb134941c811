"""C5 (BASELINE configs[4], 3D scaling stress) on the device: generator bit
for bit against the C restatement, then FPPM iterations on the sparse kernel
against the oracle (scaled sizes; the full config is 16M hit points x 128M
photons)."""
import numpy as np
import pytest

from helpers import compare_iteration, oracle_cfg
from paper_2504_04411_b200 import WORKLOADS, FppmContext

pytestmark = pytest.mark.gpu


def test_c5_generator_bitexact(port):
    seed, H, N = 0x5EED, 4096, 40000
    ctx = FppmContext(initial_radius=0.04, samples_per_iteration=N, max_hitpoints=H, max_photons=N)
    ctx.c5_setup(seed, H)
    ctx.c5_hitpoints(0, H)
    c = port.c5(seed, H)
    want = c.hitpoints()
    got = ctx.get_hitpoints()
    for k in ("pos", "nrm", "wo", "thr", "alb", "eye_depth", "gathered"):
        assert np.array_equal(got[k], want[k]), k
    for it, begin in ((1, 0), (4, 12345)):
        ctx.generate_photons(5, seed, it, N, begin=begin)
        g = ctx.get_photons()
        w = c.photons(it, begin, N)
        for k in ("pos", "nrm", "wi", "pow", "depth"):
            assert np.array_equal(g[k].view(np.uint32), w[k].view(np.uint32)), k


@pytest.mark.parametrize("kernel", ["auto", "warp"])
def test_c5_iterations_match_oracle(port, kernel):
    wl = WORKLOADS["c5"].scaled(raster=128, photons=1 << 17)  # H = 16384
    from dataclasses import replace
    wl = replace(wl, initial_radius=0.05)
    ctx = FppmContext(**wl.context_kwargs(gather_kernel=kernel))
    wl.set_hitpoints(ctx)
    c = port.c5(wl.seed, wl.hitpoints)
    sess = port.session(oracle_cfg(wl), c.hitpoints())
    for it in range(1, 4):
        ctx.generate_photons(5, wl.seed, it, wl.photons)
        got, summary = ctx.iterate(it, stats=True)
        want = sess.iterate(it, c.photons(it, 0, wl.photons))
        compare_iteration(got, want)
        assert summary["accepted"] == int(want["accepted"].sum()) > 0


def test_c5_api_errors():
    from paper_2504_04411_b200 import InvalidArgument, StateError
    ctx = FppmContext(initial_radius=0.04, samples_per_iteration=100, max_hitpoints=64, max_photons=100)
    with pytest.raises(StateError):
        ctx.generate_photons(5, 1, 1, 10)   # before c5_setup
    with pytest.raises(StateError):
        ctx.c5_hitpoints(0, 10)
    ctx.c5_setup(1, 100)
    with pytest.raises(InvalidArgument):
        ctx.c5_hitpoints(90, 20)            # beyond the generated set
    with pytest.raises(InvalidArgument):
        ctx.generate_photons(5, 2, 1, 10)   # seed differs from the setup
