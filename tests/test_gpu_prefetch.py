"""fppm_gpu_prefetch_photons / fppm_gpu_adopt_photons: the next batch's
upload overlaps the current iteration; adopting it by token gives exactly the
results of a plain set_photons; any other photon call discards it; a stale
token and host arrays rewritten after the prefetch are refused."""
import ctypes as C

import numpy as np
import pytest

from paper_2504_04411_b200 import FppmContext, WORKLOADS
from paper_2504_04411_b200 import _native as N

pytestmark = pytest.mark.gpu


def _batch(seed, it, n, generator=2):
    from oracle import Oracle
    ph = Oracle("port").gen_photons(generator, seed, it, 0, n)
    keys = ("pos", "nrm", "wi", "pow", "depth")
    return {k: np.ascontiguousarray(ph[k], dtype=np.uint32 if k == "depth" else np.float32) for k in keys}


def _ph(b):
    return N.Photons(*[b[k].ctypes.data for k in ("pos", "nrm", "wi", "pow", "depth")])


def _run(prefetch):
    wl = WORKLOADS["c2"].scaled(raster=64, photons=1 << 15)
    ctx = FppmContext(**wl.context_kwargs())
    ctx.generate_raster_hitpoints(wl.raster)
    batches = [_batch(wl.seed, it, wl.photons, wl.generator) for it in range(1, 5)]
    outs = []
    token = C.c_uint64(0)
    for i, b in enumerate(batches):
        if token.value:
            N.check(ctx._lib.fppm_gpu_adopt_photons(ctx._h, token.value), ctx._h)
            token.value = 0
        else:
            N.check(ctx._lib.fppm_gpu_set_photons(ctx._h, C.byref(_ph(b)), wl.photons), ctx._h)
        if prefetch and i + 1 < len(batches):
            N.check(ctx._lib.fppm_gpu_prefetch_photons(ctx._h, C.byref(_ph(batches[i + 1])), wl.photons,
                                                       C.byref(token)), ctx._h)
        ctx.N = wl.photons
        got, _ = ctx.iterate(i + 1, stats=True)
        outs.append(got)
    ctx.close()
    return outs


def test_prefetch_matches_plain_uploads():
    a, b = _run(False), _run(True)
    for x, y in zip(a, b):
        for k in x:
            assert np.array_equal(np.asarray(x[k]), np.asarray(y[k])), k


def test_prefetch_superseded():
    wl = WORKLOADS["c2"].scaled(raster=32, photons=1 << 12)
    ctx = FppmContext(**wl.context_kwargs())
    ctx.generate_raster_hitpoints(wl.raster)
    b1, b2 = _batch(wl.seed, 1, wl.photons, wl.generator), _batch(wl.seed, 2, wl.photons, wl.generator)
    N.check(ctx._lib.fppm_gpu_set_photons(ctx._h, C.byref(_ph(b1)), wl.photons), ctx._h)
    tok = C.c_uint64(0)
    N.check(ctx._lib.fppm_gpu_prefetch_photons(ctx._h, C.byref(_ph(b2)), wl.photons, C.byref(tok)), ctx._h)
    ctx.generate_photons(wl.generator, wl.seed, 3, wl.photons)   # discards the prefetch
    assert ctx._lib.fppm_gpu_adopt_photons(ctx._h, tok.value) == 5  # FPPM_ERR_STATE: superseded
    got, _ = ctx.iterate(1)
    ref = FppmContext(**wl.context_kwargs())
    ref.generate_raster_hitpoints(wl.raster)
    ref.generate_photons(wl.generator, wl.seed, 3, wl.photons)
    want, _ = ref.iterate(1)
    assert np.array_equal(got["accepted"], want["accepted"])


def test_rewritten_prefetch_buffer_is_refused():
    """A caller that reuses the host buffer after prefetching gets
    FPPM_ERR_STATE at adoption instead of the stale upload, and a plain
    set_photons of the rewritten buffer then gives the new batch's results."""
    wl = WORKLOADS["c2"].scaled(raster=32, photons=1 << 12)
    ctx = FppmContext(**wl.context_kwargs())
    ctx.generate_raster_hitpoints(wl.raster)
    b1, b2, b3 = (_batch(wl.seed, it, wl.photons, wl.generator) for it in (1, 2, 3))
    N.check(ctx._lib.fppm_gpu_set_photons(ctx._h, C.byref(_ph(b1)), wl.photons), ctx._h)
    buf = {k: v.copy() for k, v in b2.items()}
    tok = C.c_uint64(0)
    N.check(ctx._lib.fppm_gpu_prefetch_photons(ctx._h, C.byref(_ph(buf)), wl.photons, C.byref(tok)), ctx._h)
    ctx.synchronize()
    for k in buf:                       # the buffer is refilled with the next batch
        buf[k][...] = b3[k]
    assert ctx._lib.fppm_gpu_adopt_photons(ctx._h, tok.value) == 5
    assert "changed after" in ctx._lib.fppm_gpu_last_error(ctx._h).decode()
    assert ctx._lib.fppm_gpu_adopt_photons(ctx._h, tok.value) == 5   # consumed
    N.check(ctx._lib.fppm_gpu_set_photons(ctx._h, C.byref(_ph(buf)), wl.photons), ctx._h)
    ctx.N = wl.photons
    got, _ = ctx.iterate(1)
    ref = FppmContext(**wl.context_kwargs())
    ref.generate_raster_hitpoints(wl.raster)
    N.check(ref._lib.fppm_gpu_set_photons(ref._h, C.byref(_ph(b3)), wl.photons), ref._h)
    ref.N = wl.photons
    want, _ = ref.iterate(1)
    assert np.array_equal(got["accepted"], want["accepted"])
    assert np.array_equal(got["radius"], want["radius"])
    ctx.close()
    ref.close()


def test_stale_token_is_refused():
    wl = WORKLOADS["c2"].scaled(raster=16, photons=1 << 10)
    ctx = FppmContext(**wl.context_kwargs())
    b1, b2 = _batch(wl.seed, 1, wl.photons, wl.generator), _batch(wl.seed, 2, wl.photons, wl.generator)
    N.check(ctx._lib.fppm_gpu_set_photons(ctx._h, C.byref(_ph(b1)), wl.photons), ctx._h)
    t1, t2 = C.c_uint64(0), C.c_uint64(0)
    N.check(ctx._lib.fppm_gpu_prefetch_photons(ctx._h, C.byref(_ph(b2)), wl.photons, C.byref(t1)), ctx._h)
    N.check(ctx._lib.fppm_gpu_prefetch_photons(ctx._h, C.byref(_ph(b2)), wl.photons, C.byref(t2)), ctx._h)
    assert t2.value != t1.value
    assert ctx._lib.fppm_gpu_adopt_photons(ctx._h, t1.value) == 5
    N.check(ctx._lib.fppm_gpu_adopt_photons(ctx._h, t2.value), ctx._h)
    ctx.close()
