"""Option B of the multi-GPU decomposition on one GPU: W
photon shares are gathered by W independent contexts (each with every hit
point), their partial-sum rows are summed (what ncclReduceScatter does across
ranks), each owner pools and tests its slice, and the new radii are copied to
every context (the all-gather).  Contexts run one after another -- no kernel
waits on another.  The stitched result must match the single-process oracle:
counts, decisions and radii exact; fp64 sums within summation-order
tolerance (the shares' partial sums are added in a different order)."""
import numpy as np
import pytest
import torch

from helpers import compare_iteration, oracle_cfg
from paper_2504_04411_b200 import WORKLOADS, FppmContext
from paper_2504_04411_b200.distributed import owner_slice, photon_share

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("kernel", ["fine", "warp", "sparse"])
def test_photon_sharded_matches_oracle(port, world, kernel):
    wl = WORKLOADS["c2"].scaled(raster=48, photons=1 << 16)
    H = wl.hitpoints
    ctxs = []
    for _ in range(world):
        c = FppmContext(**wl.context_kwargs(gather_kernel=kernel))
        c.generate_raster_hitpoints(wl.raster)
        ctxs.append(c)
    stride = ctxs[0].delta_stride
    assert stride == wl.groups + 2 * wl.groups + 3
    sess = port.session(oracle_cfg(wl), port.gen_raster_hitpoints(wl.raster))
    for it in range(1, 5):
        rows = []
        for r, c in enumerate(ctxs):
            b, n = photon_share(wl.photons, r, world)
            c.generate_photons(wl.generator, wl.seed, it, n, begin=b)
            c.build_grid(0.0)               # radii are replicated: same cell on every rank
            d = torch.zeros((H, stride), dtype=torch.float64, device="cuda")
            c.gather_deltas(it, d)
            rows.append(d)
        total = rows[0].clone()
        for d in rows[1:]:
            total += d
        got = {}
        for r, c in enumerate(ctxs):
            h0, n = owner_slice(H, r, world)
            o, _ = c.apply_deltas(it, h0, total[h0:h0 + n], stats=True)
            for k, v in o.items():
                got.setdefault(k, []).append(v)
        got = {k: np.concatenate(v, 0) for k, v in got.items()}
        # all-gather of the owners' radii
        for c in ctxs:
            c.set_regions(radius=got["radius"])
        want = sess.iterate(it, port.gen_photons(wl.generator, wl.seed, it, 0, wl.photons))
        compare_iteration(got, want, flux_rtol=1e-12)
        assert want["rejected"].sum() > 0 or it == 1


def test_deltas_of_one_share_equal_gather_test(port):
    """world 1: gather_deltas + apply_deltas(all) == gather_test, bit for bit
    (same kernel, same sums; only the state update moves to a second launch)."""
    wl = WORKLOADS["c1"].scaled(raster=32, photons=1 << 15)
    a = FppmContext(**wl.context_kwargs())
    b = FppmContext(**wl.context_kwargs())
    for c in (a, b):
        c.generate_raster_hitpoints(wl.raster)
    for it in range(1, 4):
        for c in (a, b):
            c.generate_photons(wl.generator, wl.seed, it, wl.photons)
            c.build_grid(0.0)
        want, _ = a.gather_test(it, stats=True)
        d = torch.zeros((wl.hitpoints, b.delta_stride), dtype=torch.float64, device="cuda")
        b.gather_deltas(it, d)
        got, _ = b.apply_deltas(it, 0, d, stats=True)
        for k in want:
            assert np.array_equal(got[k], want[k]), k
