"""General 3D synthetic scenes for parity tests (numpy only, tests only)."""
import numpy as np


def _unit(v):
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


def _frame(n):
    # any orthonormal pair: the tests only need points in the tangent disk
    a = np.where(np.abs(n[:, :1]) > 0.9, np.array([[0.0, 1.0, 0.0]]), np.array([[1.0, 0.0, 0.0]]))
    u = _unit(np.cross(n, a))
    return u, np.cross(n, u)


def scene3d(seed, H=1500, N=60000, r=0.03, offset=(0.0, 0.0, 0.0), scale=1.0, frac_gathered=0.85):
    rng = np.random.default_rng(seed)
    pos = rng.random((H, 3)) * scale + np.asarray(offset)
    nrm = _unit(rng.normal(size=(H, 3)))
    nrm[: H // 4] = [0.0, 0.0, 1.0]                       # some planar-fast-path regions
    nrm[H // 4: H // 3] = [0.0, 0.0, -1.0]               # the frame's n.z < 0 branch
    wo = _unit(nrm + 0.8 * rng.normal(size=(H, 3)))       # some back-facing (cos_o <= 0)
    hit = dict(pos=pos, nrm=nrm, wo=wo, thr=rng.random((H, 3)) + 0.1,
               alb=rng.random((H, 3)), eye_depth=rng.integers(1, 5, H).astype(np.uint32),
               gathered=(rng.random(H) < frac_gathered).astype(np.uint8))
    # photons: 80% in the tangent disks of random hit points, 20% uniform
    owner = rng.integers(0, H, N)
    u, v = _frame(nrm)
    rr = 1.4 * r * np.sqrt(rng.random(N))
    phi = 2 * np.pi * rng.random(N)
    p = (pos[owner] + (rr * np.cos(phi))[:, None] * u[owner] + (rr * np.sin(phi))[:, None] * v[owner]
         + (0.3 * r * rng.normal(size=N))[:, None] * nrm[owner])
    far = rng.random(N) < 0.2
    p[far] = rng.random((far.sum(), 3)) * scale + np.asarray(offset)
    pn = _unit(nrm[owner] + 0.45 * rng.normal(size=(N, 3)))   # ~guard-limited mix
    wi = _unit(pn + 0.9 * rng.normal(size=(N, 3)))            # some cos_i <= 0
    ph = dict(pos=p.astype(np.float32), nrm=pn.astype(np.float32), wi=wi.astype(np.float32),
              pow=(rng.random((N, 3)) * 2).astype(np.float32),
              depth=rng.integers(1, 10, N).astype(np.uint32))
    return hit, ph
