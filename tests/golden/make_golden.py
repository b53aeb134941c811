#!/usr/bin/env python
"""Generate tests/golden/golden.json from the reference's own code.

Runs in the build container only (oracle/_ref is compiled from the unmodified
reference sources by oracle/Makefile).  The fixtures pin the C restatement
(oracle/fppm_oracle.c) and the GPU path on machines where the reference tree
is absent.  Sources of each vector:

* sector_index layout            test_gather.cpp:26-36
* quantile closed forms          test_special_functions.cpp:41-64, acceptance A1
* critical values per config     SURVEY.md §8a (stat_tests.cpp:72-82 memo path)
* F statistic hand value         test_stat_tests.cpp:65-70
* schedule floor                 test_gather.cpp:98-106
* grid internals / query order   test_photon_map.cpp:47-138 (random sets here)
* a small FPPM run on canonical inputs (C1/C2 scaled) through PhotonGrid +
  GatherRegion (ref_driver.cpp, restating integrator.cpp:388-489)
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from oracle import Oracle  # noqa: E402


def hexf(x):
    return float(x).hex()


def main():
    ref = Oracle("reference")
    port = Oracle("port")  # only for the canonical generator
    g = {"generated_by": "tests/golden/make_golden.py (oracle/_ref = reference proj/core)"}

    g["sector_index"] = [
        dict(u=u, v=v, r=r, na=na, ns=ns, sector=ref.sector_index(u, v, r, na, ns))
        for (u, v, r, na, ns) in [
            (0.999, 0.0, 1.0, 2, 6), (0.0, 0.4, 1.0, 2, 6), (0.0, -0.4, 1.0, 2, 6),
            (1.0, 0.0, 1.0, 2, 6), (0.0, 0.0, 1.0, 2, 6),
            # SURVEY §8a exact-sector table for n_s = 4
            (1e-3, 0.0, 1.0, 1, 4), (1e-3, -0.0, 1.0, 1, 4), (0.0, 1e-3, 1.0, 1, 4),
            (-0.0, 1e-3, 1.0, 1, 4), (-1e-3, 0.0, 1.0, 1, 4), (-1e-3, -0.0, 1.0, 1, 4),
            (0.0, -1e-3, 1.0, 1, 4), (-0.0, -1e-3, 1.0, 1, 4), (0.0, 0.0, 1.0, 1, 4),
            (-0.0, -0.0, 1.0, 1, 4), (0.3, 0.2, 1.0, 2, 4), (-0.3, 0.2, 1.0, 2, 4),
            (-0.3, -0.2, 1.0, 2, 4), (0.3, -0.2, 1.0, 2, 4), (0.6, 0.2, 1.0, 2, 4),
            (0.5, 0.5, 1.0, 2, 4),
        ]]
    g["sector_index_throws"] = [dict(u=1.1, v=0.0, r=1.0, na=2, ns=6, error="domain"),
                                dict(u=0.5, v=0.0, r=1.0, na=0, ns=6, error="invalid")]

    q = []
    for (p, d1, d2) in [(0.95, 2, 2), (0.5, 1, 1), (0.99, 11, 1e9), (0.99, 11, 49140),
                        (0.95, 3, 4 * (2 ** 20 - 1)), (0.95, 3, 4 * (2 * 2 ** 20 - 1)),
                        (0.95, 3, 4 * (4 * 2 ** 20 - 1)), (0.95, 3, 4 * (5 * 2 ** 20 - 1)),
                        (0.99, 7, 8 * (2 ** 22 - 1)), (0.95, 7, 8 * (2 ** 27 - 1)),
                        (0.95, 3, 4 * (8 * 2 ** 20 - 1)), (0.99, 11, 132), (0.95, 11, 4 * 99)]:
        q.append(dict(p=p, d1=d1, d2=d2, value=hexf(ref.f_quantile(p, d1, d2))))
    g["f_quantile"] = q
    g["chi2_quantile"] = [dict(p=p, df=df, value=hexf(ref.chi2_quantile(p, df)))
                          for (p, df) in [(0.5, 2.0), (0.99, 11.0), (0.99, 3.0), (0.99, 7.0)]]
    g["schedule_radius"] = [dict(base=b, alpha=a, i=i, value=hexf(ref.schedule_radius(b, a, i)))
                            for (b, a, i) in [(1.0, 0.75, 4), (0.02e-3, 0.75, 17), (0.01e-3, 0.75, 65),
                                              (0.5, 0.75, 200), (0.001, 0.75, 2)]]
    g["f_statistic_hand"] = dict(
        count=[2, 2], sum=[4.0, 10.0], sum_sq=[10.0, 52.0], m=2,
        value=hexf(ref.f_statistic([2, 2], [4.0, 10.0], [10.0, 52.0], 2)))
    frames = []
    rng = np.random.default_rng(5)
    for _ in range(8):
        n = rng.normal(size=3)
        n /= np.linalg.norm(n)
        u, v = ref.build_frame(n)
        frames.append(dict(n=[hexf(x) for x in n], u=[hexf(x) for x in u], v=[hexf(x) for x in v]))
    for n in ([0.0, 0.0, 1.0], [0.0, 0.0, -1.0]):
        u, v = ref.build_frame(np.array(n))
        frames.append(dict(n=[hexf(x) for x in n], u=[hexf(x) for x in u], v=[hexf(x) for x in v]))
    g["frames"] = frames

    # grid internals + ball queries (test_photon_map.cpp style sets)
    rng = np.random.default_rng(31)
    pos = (2.0 * (2 * rng.random((600, 3)) - 1)).astype(np.float32)
    cell = 0.3
    grid = ref.grid_build(pos.astype(np.float64), cell)
    keys, b, e, order = grid.export()
    centers = 2.2 * (2 * rng.random((40, 3)) - 1)
    radii = cell * (0.3 + 0.7 * rng.random(40))
    radii[:4] = cell
    g["grid"] = dict(pos=pos.tolist(), cell=cell, keys=[int(k) for k in keys], begin=b.tolist(),
                     end=e.tolist(), order=order.tolist(), centers=centers.tolist(),
                     radii=radii.tolist(),
                     queries=[ref_q.tolist() for ref_q in
                              (grid.query_ball(centers[i], radii[i]) for i in range(40))])

    # small FPPM runs on canonical inputs
    runs = []
    for (wl, W, N, na, ns, alpha_f, r0, iters) in [(1, 16, 4096, 1, 4, 0.05, 0.08, 4),
                                                   (2, 24, 8192, 2, 4, 0.01, 0.05, 4)]:
        hp = port.gen_raster_hitpoints(W)
        cfg = dict(n_annuli=na, n_sectors=ns, alpha_f=alpha_f, initial_radius=r0,
                   r_min_base=0.001 * r0, samples_per_iteration=N, threads=4)
        sess = ref.session(cfg, hp)
        its = []
        for it in range(1, iters + 1):
            ph = port.gen_photons(wl, 0x5EED, it, 0, N)
            out = sess.iterate(it, ph)
            its.append(dict(
                iteration=it,
                photon_pos_digest=int(np.bitwise_xor.reduce(ph["pos"].view(np.uint32).ravel())),
                accepted=out["accepted"].tolist(), rejected=out["rejected"].tolist(),
                tested=out["tested"].tolist(), t=out["t"].tolist(),
                radius=[hexf(x) for x in out["radius"]],
                critical=[hexf(x) for x in out["critical"]],
                statistic=[float(x) for x in out["statistic"]],
                flux=out["flux"].tolist()))
        runs.append(dict(workload=wl, raster=W, photons=N, n_annuli=na, n_sectors=ns,
                         alpha_f=alpha_f, initial_radius=r0, seed=0x5EED, iterations=its))
    g["runs"] = runs
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(g, f)
    print("wrote", os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
