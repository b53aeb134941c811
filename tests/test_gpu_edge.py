"""GPU parity of the full gather path on general (non-canonical) inputs and
edge cases, vs the oracle (and the reference build where present).

The canonical workloads put every hit point on the z=0 plane; these cases
exercise the general 3D path: arbitrary normals (full tangent frame and the
30-degree normal guard), the depth filter, back-facing wo / wi, per-hit-point
throughput and albedo, not-gathered hit points, rgb channels, every
end-of-iteration policy and override, empty photon sets, photons exactly on
the closed-ball rim, coincident photons, negative / large coordinates and
the m < 2 hold."""
import numpy as np
import pytest

from helpers import compare_iteration
from scenes import _unit, scene3d
from paper_2504_04411_b200 import FppmContext

pytestmark = pytest.mark.gpu

POLICY = {"ftest": 0, "chi2": 1, "schedule": 2}
OVERRIDE = {"none": 0, "always_reject": 1, "never_reject": 2}


def make_pair(port_or_ref, hit, cfg, kernel="auto", device_policy=None):
    ctx = FppmContext(initial_radius=cfg["initial_radius"],
                      samples_per_iteration=cfg["samples_per_iteration"],
                      n_annuli=cfg["n_annuli"], n_sectors=cfg["n_sectors"],
                      alpha_f=cfg["alpha_f"], alpha_chi2=cfg.get("alpha_chi2", 0.01),
                      channels="rgb" if cfg.get("channels", 1) == 3 else "luminance",
                      override_decision={v: k for k, v in OVERRIDE.items()}[cfg.get("override_decision", 0)],
                      k=cfg.get("k", 0.7), alpha=cfg.get("alpha", 0.75), r_min_base=cfg["r_min_base"],
                      max_depth=cfg.get("max_depth", 10),
                      policy={v: k for k, v in POLICY.items()}[cfg.get("policy", 0)],
                      max_hitpoints=len(hit["pos"]), max_photons=1 << 17, gather_kernel=kernel)
    ctx.set_hitpoints(hit["pos"], hit["nrm"], hit["wo"], hit["thr"], hit["alb"],
                      hit["eye_depth"], hit.get("gathered"))
    return ctx, port_or_ref.session(cfg, hit)


def run_iters(ctx, sess, ph_of_it, iters):
    near = 0
    for it in range(1, iters + 1):
        ph = ph_of_it(it)
        ctx.set_photons(ph["pos"], ph["nrm"], ph["wi"], ph["pow"], ph["depth"])
        got, summ = ctx.iterate(it, stats=True)
        want = sess.iterate(it, ph)
        near += compare_iteration(got, want)
        assert summ["accepted"] == int(want["accepted"].sum())
    return near


BASE = dict(n_annuli=2, n_sectors=6, alpha_f=0.05, initial_radius=0.03, r_min_base=3e-5,
            samples_per_iteration=60000, threads=8)


@pytest.mark.parametrize("kernel", ["fine", "warp", "3d"])
def test_general_3d_scene(port, kernel):
    hit, _ = scene3d(1)
    ctx, sess = make_pair(port, hit, BASE, kernel)
    run_iters(ctx, sess, lambda it: scene3d(100 + it)[1], 4)


@pytest.mark.parametrize("over", [
    dict(channels=3),
    dict(n_annuli=1, n_sectors=4),
    dict(n_annuli=3, n_sectors=5),
    dict(n_annuli=1, n_sectors=2),
    dict(n_annuli=4, n_sectors=8),
    dict(policy=1, alpha_chi2=0.05),
    dict(policy=2),
    dict(override_decision=1),
    dict(override_decision=2),
    dict(max_depth=4),
    dict(samples_per_iteration=1),   # m = t J < 2 on the first test -> hold untested
    dict(k=0.5, alpha=0.5, r_min_base=0.01),
])
def test_config_variants(port, over):
    cfg = dict(BASE, **over)
    hit, _ = scene3d(2, H=800, N=30000)
    ctx, sess = make_pair(port, hit, cfg)
    run_iters(ctx, sess, lambda it: scene3d(200 + it, H=800, N=30000)[1], 3)


def test_negative_and_far_coordinates(port):
    hit, _ = scene3d(3, H=600, N=20000, offset=(-1000.25, 37.0, -3.5), scale=0.5)
    ctx, sess = make_pair(port, hit, BASE)
    run_iters(ctx, sess,
              lambda it: scene3d(300 + it, H=600, N=20000, offset=(-1000.25, 37.0, -3.5), scale=0.5)[1], 3)


def test_reference_build_general_scene(port, ref):
    hit, _ = scene3d(4, H=400, N=15000)
    cfg = dict(BASE, channels=3)
    ctx, sess = make_pair(ref, hit, cfg)
    run_iters(ctx, sess, lambda it: scene3d(400 + it, H=400, N=15000)[1], 3)


def _empty_photons():
    return dict(pos=np.zeros((0, 3), np.float32), nrm=np.zeros((0, 3), np.float32),
                wi=np.zeros((0, 3), np.float32), pow=np.zeros((0, 3), np.float32),
                depth=np.zeros(0, np.uint32))


def test_empty_photon_set(port):
    hit, ph = scene3d(5, H=300, N=5000)
    ctx, sess = make_pair(port, hit, BASE)
    run_iters(ctx, sess, lambda it: _empty_photons() if it % 2 else ph, 4)


def test_no_gathered_hitpoints(port):
    hit, ph = scene3d(6, H=300, N=5000, frac_gathered=0.0)
    ctx, sess = make_pair(port, hit, BASE)
    run_iters(ctx, sess, lambda it: ph, 2)


def test_closed_ball_rim_and_coincident_photons(port):
    """Photons exactly at distance r (binary-exact), exactly at the centre,
    on cell boundaries, and 64 coincident copies of one position."""
    W = 8
    xs = (np.arange(W) + 0.5) / W
    gx, gy = np.meshgrid(xs, xs)
    H = W * W
    hit = dict(pos=np.stack([gx.ravel(), gy.ravel(), np.zeros(H)], 1), nrm=np.tile([0.0, 0, 1], (H, 1)),
               wo=np.tile([0.0, 0, 1], (H, 1)), thr=np.ones((H, 3)), alb=np.full((H, 3), 0.5),
               eye_depth=np.ones(H, np.uint32))
    r = 0.0625  # 2^-4: exact in fp32 and fp64
    pts = []
    for cx, cy in hit["pos"][:, :2]:
        for dx, dy in ((r, 0), (-r, 0), (0, r), (0, -r), (0, 0), (r / 2, r / 2), (r, r / 1024)):
            pts.append((cx + dx, cy + dy, 0.0))
    pts += [(0.25, 0.25, 0.0)] * 64 + [(0.5, 0.5, 0.0), (0.0, 0.0, 0.0), (1.0, 1.0, 0.0)]
    P = np.array(pts)
    n = len(P)
    rng = np.random.default_rng(7)
    ph = dict(pos=P.astype(np.float32), nrm=np.tile(np.float32([0, 0, 1]), (n, 1)),
              wi=_unit(rng.normal(size=(n, 3)) * [1, 1, 0] + [0, 0, 1.5]).astype(np.float32),
              pow=(rng.random((n, 3)) + 0.5).astype(np.float32), depth=np.ones(n, np.uint32))
    cfg = dict(BASE, initial_radius=r, r_min_base=r * 1e-3, samples_per_iteration=n)
    ctx, sess = make_pair(port, hit, cfg)
    ctx.set_photons(ph["pos"], ph["nrm"], ph["wi"], ph["pow"], ph["depth"])
    got, _ = ctx.iterate(1, stats=True)
    want = sess.iterate(1, ph)
    compare_iteration(got, want)
    # the rim photons are inside the closed ball
    assert int(want["accepted"][0]) >= 6


def test_normal_guard_and_depth_filters(port):
    """Flipped photon normals fail the 30-degree guard against their own hit
    point (only stray cross-region pairs survive); max_depth 2 keeps only
    depth-1 photons of eye-depth-1 hit points."""
    hit, ph = scene3d(8, H=200, N=8000)
    ctx, sess = make_pair(port, hit, BASE)
    ctx.set_photons(ph["pos"], ph["nrm"], ph["wi"], ph["pow"], ph["depth"])
    base, _ = ctx.iterate(1, stats=True)
    flipped = dict(ph, nrm=-ph["nrm"])
    ctx, sess = make_pair(port, hit, BASE)
    ctx.set_photons(flipped["pos"], flipped["nrm"], flipped["wi"], flipped["pow"], flipped["depth"])
    got, _ = ctx.iterate(1, stats=True)
    compare_iteration(got, sess.iterate(1, flipped))
    assert got["accepted"].sum() * 20 < base["accepted"].sum()
    shallow = dict(BASE, max_depth=2)
    ctx, sess = make_pair(port, hit, shallow)
    ctx.set_photons(ph["pos"], ph["nrm"], ph["wi"], ph["pow"], ph["depth"])
    got, _ = ctx.iterate(1, stats=True)
    compare_iteration(got, sess.iterate(1, ph))
    assert np.all(got["accepted"][hit["eye_depth"] > 1] == 0)
