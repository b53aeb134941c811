"""Shared parity helpers (tests only)."""
import numpy as np

from paper_2504_04411_b200 import FppmContext


def oracle_cfg(wl, **over):
    cfg = dict(n_annuli=wl.n_annuli, n_sectors=wl.n_sectors, alpha_f=wl.alpha_f,
               initial_radius=wl.initial_radius, r_min_base=0.001 * wl.initial_radius,
               samples_per_iteration=wl.photons, k=wl.k, alpha=wl.alpha, threads=8)
    cfg.update(over)
    return cfg


def compare_iteration(got, want, *, flux_rtol=1e-11, stat_rtol=1e-9):
    """Parity bar (BASELINE north_star): bit-exact counts, decisions and radii
    (radii are fp64 results of identical operations); fp64 sums within
    summation-order tolerance; F within 1e-9 relative; decisions may differ
    only where |F - F_c| / F_c <= 1e-6 (reported)."""
    acc = got["accepted"].astype(np.uint64)
    assert np.array_equal(acc, want["accepted"]), \
        f"accepted differ at {np.flatnonzero(acc != want['accepted'])[:10]}"
    if "stat_count" in got and "stat_count" in want:
        assert np.array_equal(got["stat_count"], want["stat_count"])
        np.testing.assert_allclose(got["stat_sum"], want["stat_sum"], rtol=1e-12, atol=1e-300)
        np.testing.assert_allclose(got["stat_sum_sq"], want["stat_sum_sq"], rtol=1e-12, atol=1e-300)
    near = np.zeros(len(acc), bool)
    crit = want["critical"]
    with np.errstate(invalid="ignore", divide="ignore"):
        near = (want["tested"] == 1) & (np.abs(want["statistic"] - crit) <= 1e-6 * np.abs(crit))
    mism = (got["rejected"] != want["rejected"]) & ~near
    assert not mism.any(), f"decision mismatch at {np.flatnonzero(mism)[:10]}"
    assert np.array_equal(got["tested"], want["tested"])
    ok = ~near
    assert np.array_equal(got["radius"][ok], want["radius"][ok]), "radii differ"
    assert np.array_equal(got["t"][ok], want["t"][ok]), "t differs"
    np.testing.assert_allclose(got["flux"], want["flux"], rtol=flux_rtol, atol=1e-300)
    fin = np.isfinite(want["statistic"])
    np.testing.assert_allclose(got["statistic"][fin], want["statistic"][fin], rtol=stat_rtol, atol=0)
    assert np.array_equal(got["critical"], want["critical"])
    np.testing.assert_allclose(got["radiance"], want["radiance"].astype(np.float32), rtol=1e-5, atol=1e-30)
    return int(near.sum())


def gpu_context(wl, **over):
    ctx = FppmContext(**wl.context_kwargs(**over))
    ctx.generate_raster_hitpoints(wl.raster)
    return ctx
