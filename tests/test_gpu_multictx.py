"""Multi-GPU decompositions exercised on one GPU with several contexts
(the kernels do not wait on one another, so this is exactly
what each rank computes):

  * option A: K contexts, each owning a band of raster rows, receive every
    photon share in one packed buffer (the all-gather's layout), stage only
    the photons within the all-reduced r_max of their band
    (fppm_gpu_set_photons_packed), build their grid from the device cell and
    gather + test; the stitched counts, decisions and radii equal one context
    over the whole raster bit for bit, iteration after iteration (the fp64
    moment sums to rounding: their lane order follows the staged array);
  * the light phase sharded by path ranges (fppm_gpu_trace_photons_range):
    the shares concatenated in rank order are the single-call photon array.
"""
import numpy as np
import pytest
import torch

from paper_2504_04411_b200 import FppmContext, WORKLOADS
from paper_2504_04411_b200.distributed import pack_photons, photon_share, row_band, share_stride
from paper_2504_04411_b200.scene import caustic_box

pytestmark = pytest.mark.gpu

KEYS = ("radius", "gather_radius", "t", "tested", "rejected", "accepted", "critical")
# fp64 sums whose lane / window assignment follows the staged photon array:
# equal to rounding (the decisions and radii above are bit-exact)
NEAR = ("flux", "statistic")


def _hitpoints(W, r0, r1):
    j, i = np.meshgrid(np.arange(r0, r1), np.arange(W), indexing="ij")
    pos = np.zeros(((r1 - r0) * W, 3))
    pos[:, 0] = ((i.ravel() + 0.5) / W).astype(np.float32)
    pos[:, 1] = ((j.ravel() + 0.5) / W).astype(np.float32)
    return pos, np.tile([0.0, 0.0, 1.0], (len(pos), 1))


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("wl_name", ["c1", "c2"])
def test_option_a_bands_stitch_to_single_context(world, wl_name):
    wl = WORKLOADS[wl_name].scaled(raster=96, photons=1 << 17)
    W, N = wl.raster, wl.photons
    one = FppmContext(**wl.context_kwargs())
    one.set_hitpoints(*_hitpoints(W, 0, W))
    bands = [row_band(W, r, world) for r in range(world)]
    ranks = []
    for r0, r1 in bands:
        c = FppmContext(**wl.context_kwargs(max_hitpoints=(r1 - r0) * W))
        c.set_hitpoints(*_hitpoints(W, r0, r1))
        ranks.append(c)
    dev = torch.device("cuda", 0)
    stride = share_stride(N, world)
    part_n = [photon_share(N, r, world)[1] for r in range(world)]
    cells = [torch.zeros(1, dtype=torch.float64, device=dev) for _ in range(world)]
    kept_frac = []
    for it in range(1, 5):
        one.generate_photons(wl.generator, wl.seed, it, N)
        ph = one.get_photons()
        want, _ = one.iterate(it)
        # every rank's packed share, stacked in rank order = the all-gather output
        shares = []
        for r in range(world):
            b, n = photon_share(N, r, world)
            t = {k: torch.from_numpy(np.ascontiguousarray(ph[k][b:b + n])).to(dev) for k in ph}
            shares.append(pack_photons(t["pos"], t["nrm"], t["wi"], t["pow"], t["depth"].view(torch.int32), stride))
        full = torch.stack(shares, 0)
        for c, cell in zip(ranks, cells):
            c.max_radius_device(cell)
        torch.cuda.synchronize()
        rmax = torch.max(torch.cat(cells))  # the all-reduce(max)
        for cell in cells:
            cell.fill_(rmax.item())
        got = []
        for c, cell in zip(ranks, cells):
            kept = c.set_photons_packed(full, part_n, margin=cell)
            kept_frac.append(kept / N)
            c.build_grid_device(cell)
            o, _ = c.gather_test(it)
            got.append(o)
        for k in KEYS:
            stitched = np.concatenate([np.asarray(g[k]) for g in got], 0)
            assert np.array_equal(stitched, np.asarray(want[k])), (it, k)
        for k in NEAR:
            stitched = np.concatenate([np.asarray(g[k]) for g in got], 0)
            np.testing.assert_allclose(stitched, np.asarray(want[k]), rtol=1e-12, atol=0, err_msg=f"{it} {k}")
    print(f"world {world}: kept photon fraction per band mean {np.mean(kept_frac):.3f}")
    assert max(kept_frac) < 1.0
    one.close()
    for c in ranks:
        c.close()


def test_packed_staging_without_margin_is_the_plain_upload():
    wl = WORKLOADS["c2"].scaled(raster=64, photons=1 << 15)
    a = FppmContext(**wl.context_kwargs())
    b = FppmContext(**wl.context_kwargs())
    for c in (a, b):
        c.set_hitpoints(*_hitpoints(wl.raster, 0, wl.raster))
    a.generate_photons(wl.generator, wl.seed, 1, wl.photons)
    ph = a.get_photons()
    dev = torch.device("cuda", 0)
    world = 4
    stride = share_stride(wl.photons, world)
    part_n = [photon_share(wl.photons, r, world)[1] for r in range(world)]
    shares = []
    for r in range(world):
        s, n = photon_share(wl.photons, r, world)
        t = {k: torch.from_numpy(np.ascontiguousarray(ph[k][s:s + n])).to(dev) for k in ph}
        shares.append(pack_photons(t["pos"], t["nrm"], t["wi"], t["pow"], t["depth"].view(torch.int32), stride))
    torch.cuda.synchronize()
    assert b.set_photons_packed(torch.stack(shares, 0), part_n) == wl.photons
    got = b.get_photons()
    for k in ph:
        assert np.array_equal(got[k], ph[k]), k
    x, _ = a.iterate(1)
    y, _ = b.iterate(1)
    for k in KEYS + NEAR:
        assert np.array_equal(np.asarray(x[k]), np.asarray(y[k])), k
    a.close()
    b.close()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_light_phase_concatenates_to_the_single_trace(world):
    J, depth = 1 << 15, 8
    kw = dict(initial_radius=0.02, samples_per_iteration=J, n_annuli=1, n_sectors=4, alpha_f=0.05,
              max_hitpoints=16, max_photons=J * depth)
    one = FppmContext(**kw)
    one.set_scene(caustic_box())
    n_all = one.trace_photons(7, 3, J, depth)
    want = one.get_photons()
    parts = []
    for r in range(world):
        p0, n = photon_share(J, r, world)
        c = FppmContext(**kw)
        c.set_scene(caustic_box())
        c.trace_photons(7, 3, n, depth, path0=p0)
        parts.append(c.get_photons())
        c.close()
    assert sum(len(p["depth"]) for p in parts) == n_all
    for k in want:
        assert np.array_equal(np.concatenate([p[k] for p in parts], 0), want[k]), k
    one.close()
