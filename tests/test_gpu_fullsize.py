"""Parity at the BASELINE sizes (configs[0], [1], [4]) -- the sizes bench.py
times -- against the oracle.

The GPU runs the whole frame.  The oracle runs either the whole frame (C1)
or a seeded random subset of hit points (C2, C5) on the GPU's own canonical
inputs, with the GPU's r_max as its cell size.  A subset is exact: a region's
state depends only on its own photons (integrator.cpp:159-161,
gather.cpp:90-112), and the photons a subset hit point can see are those in
the 27 reference cells around its home cell, in insertion order
(photon_map.cpp:53-78).  For C5 the oracle is handed only the photons whose
reference cell lies within +-2 cells of a subset hit point's cell (an
order-preserving superset of every 27-neighbourhood), so its grid build stays
small; C1/C2 get every photon.

Bar (BASELINE north_star): bit-exact counts, decisions and radii, fp64 sums
within summation-order tolerance, decisions may differ only within 1e-6
relative of F_c (counted and printed)."""
import os

import numpy as np
import pytest

from helpers import compare_iteration, oracle_cfg
from paper_2504_04411_b200 import WORKLOADS, FppmContext, InvalidArgument

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

THREADS = max(1, min(os.cpu_count() or 1, 64))


def _cells(pos, inv):
    """cell_coord (photon_map.cpp:13-15): floor(x * (1/cell)) in fp64."""
    return np.floor(np.asarray(pos, np.float64) * inv).astype(np.int64)


def _pack(c):
    b = 1 << 20
    return ((c[:, 0] + b) << 42) | ((c[:, 1] + b) << 21) | (c[:, 2] + b)


def near_photon_mask(ph_pos, hit_pos, cell, chunk=1 << 24):
    """Photons whose reference cell is within +-2 cells of a hit point's cell."""
    inv = 1.0 / cell
    hc = _cells(hit_pos, inv)
    off = np.stack(np.meshgrid(*[np.arange(-2, 3)] * 3, indexing="ij"), -1).reshape(-1, 3)
    want = np.unique(_pack((hc[:, None, :] + off[None, :, :]).reshape(-1, 3)))
    mask = np.zeros(len(ph_pos), bool)
    for a in range(0, len(ph_pos), chunk):
        mask[a:a + chunk] = np.isin(_pack(_cells(ph_pos[a:a + chunk], inv)), want)
    return mask


def _sub(d, idx):
    return {k: (v[idx] if isinstance(v, np.ndarray) and v.ndim >= 1 and len(v) > 0 else v) for k, v in d.items()}


def _run(port, wl, iters, subset=None, filter_photons=False, extra=None):
    ctx = FppmContext(**wl.context_kwargs())
    wl.set_hitpoints(ctx)
    hit = ctx.get_hitpoints()
    idx = np.arange(wl.hitpoints) if subset is None else subset
    sess = port.session(oracle_cfg(wl, threads=THREADS), _sub(hit, idx))
    near_total, acc_total = 0, 0
    for it in range(1, iters + 1):
        ctx.generate_photons(wl.generator, wl.seed, it, wl.photons)
        got, summary = ctx.iterate(it, stats=True)
        ph = ctx.get_photons()
        if filter_photons:
            m = near_photon_mask(ph["pos"], hit["pos"][idx], summary["cell_size"])
            ph = {k: v[m] for k, v in ph.items()}
        want = sess.iterate(it, ph, cell=summary["cell_size"])
        near_total += compare_iteration(_sub(got, idx), want)
        acc_total += int(want["accepted"].sum())
        if subset is None:
            assert summary["accepted"] == int(want["accepted"].sum())
        assert summary["ambiguous_pairs"] == 0
        if extra:
            extra(it, got, want, summary)
    print(f"{wl.name}: {iters} iterations, {len(idx)} hit points checked, {acc_total} accepted pairs, "
          f"{near_total} decisions within 1e-6 of F_c")
    ctx.close()
    return acc_total


def test_c1_full_frame(port):
    """BASELINE configs[0] at its stated size: 256^2 hit points x 2^20 photons,
    every hit point checked, 4 iterations."""
    _run(port, WORKLOADS["c1"], 4)


def test_c2_full_size_subset(port):
    """BASELINE configs[1] -- the config bench.py times -- at 512^2 x 2^22,
    4 iterations; 16384 random hit points plus every hit point in the core of
    the Gaussian blob (the densest fine cells: multi-item waves)."""
    wl = WORKLOADS["c2"]
    W = wl.raster
    rng = np.random.default_rng(2024)
    sub = set(rng.choice(wl.hitpoints, 16384, replace=False).tolist())
    ij = np.arange(wl.hitpoints)
    x, y = (ij % W + 0.5) / W, (ij // W + 0.5) / W
    sub |= set(ij[(x - 0.3) ** 2 + (y - 0.7) ** 2 < 0.012 ** 2].tolist())
    subset = np.array(sorted(sub), np.uint32)

    def check_rows(it, got, want, summary):
        # per-hit-point counts reach the blob's tens of thousands
        assert int(want["accepted"].max()) > 20000

    assert _run(port, wl, 4, subset=subset, extra=check_rows) > 0


def test_c5_full_size_subset(port):
    """BASELINE configs[4] at 16M hit points x 2^27 photons, r0 = 0.005,
    2 iterations; 8192 random hit points (> 7e9 candidate pairs per launch on
    the GPU side: 64-bit counters)."""
    wl = WORKLOADS["c5"]
    rng = np.random.default_rng(5)
    subset = np.sort(rng.choice(wl.hitpoints, 8192, replace=False)).astype(np.uint32)
    assert _run(port, wl, 2, subset=subset, filter_photons=True) > 0


def test_radius_exceeding_cell_raises():
    """photon_map.cpp:57-58: a grid built with an explicit cell smaller than a
    gathered region's radius must fail the gather, not drop photons."""
    wl = WORKLOADS["c1"].scaled(raster=16, photons=4096)
    ctx = FppmContext(**wl.context_kwargs())
    ctx.generate_raster_hitpoints(wl.raster)
    ctx.generate_photons(wl.generator, wl.seed, 1, wl.photons)
    ctx.build_grid(0.5 * wl.initial_radius)
    with pytest.raises(InvalidArgument, match="query radius exceeds cell size"):
        ctx.gather_test(1)
    ctx.build_grid(wl.initial_radius)          # cell = radius: accepted (r > cell only)
    ctx.gather_test(1)
    r = ctx.regions()["radius"]
    r[3] = 2.0 * wl.initial_radius             # set_regions raises one radius
    ctx.set_regions(radius=r)
    with pytest.raises(InvalidArgument, match="query radius exceeds cell size"):
        ctx.gather_test(2)
