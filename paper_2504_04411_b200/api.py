"""Host-side mirror of the reference hot-path interface over the C ABI.

Reference interface (proj/core/include/fppm/*.hpp) -> this module:

* ``fppm::RadiusSchedule`` / ``fppm::TestConfig`` (gather.hpp:16-41)
  -> :class:`RadiusSchedule` / :class:`TestConfig`
* ``fppm::PhotonGrid`` (photon_map.hpp:15-42) -> :class:`PhotonGrid`
* ``fppm::GatherRegion`` (gather.hpp:69-112), one per pixel
  -> :class:`GatherRegionBatch`, all regions of a frame on one GPU
* ``Renderer::step``'s gather path (integrator.cpp:159-175, 262-264,
  388-402, 435-489) -> :class:`FppmContext` (``iterate``)

Errors follow the reference exception classes: :class:`InvalidArgument`
(std::invalid_argument) and :class:`DomainError` (std::domain_error).
Arrays may be NumPy (host; copied through the C ABI) or CUDA tensors
exposing ``data_ptr()`` (device; copied device-to-device).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _native as N
from ._native import (CapacityError, CudaError, DomainError, FppmError,  # noqa: F401
                      InvalidArgument, NoDeviceError, StateError)

NORMAL_GUARD_COS = 0.86602540378443865  # integrator.cpp:47


@dataclass
class RadiusSchedule:
    """gather.hpp:16-20."""

    k: float = 0.7
    alpha: float = 0.75
    r_min_base: float = 0.0


@dataclass
class TestConfig:
    """gather.hpp:34-41 (channels: 'luminance' | 'rgb'; override: 'none' |
    'always_reject' | 'never_reject')."""

    __test__ = False  # not a pytest class
    n_annuli: int = 2
    n_sectors: int = 6
    alpha_f: float = 0.01
    alpha_chi2: float = 0.01
    channels: str = "luminance"
    override_decision: str = "none"


# auto_detect at the region level is one channel (GatherRegion, gather.cpp:40);
# the Renderer resolves it against the scene first (resolve_channels)
_CHANNELS = {"luminance": N.CHANNELS_LUMINANCE, "auto_detect": N.CHANNELS_LUMINANCE,
             "rgb": N.CHANNELS_RGB}


def resolve_channels(channels: str, scene=None) -> str:
    """Renderer's TestChannels::auto_detect (integrator.cpp:128-130): rgb when
    the scene has a chromatic emitter, else luminance.  Without a scene the
    region-level meaning applies (one channel, gather.cpp:40)."""
    if channels != "auto_detect":
        return channels
    if scene is None:
        return "luminance"
    from .scene import has_chromatic_emitter
    return "rgb" if has_chromatic_emitter(scene) else "luminance"
_OVERRIDE = {"none": N.OVERRIDE_NONE, "always_reject": N.OVERRIDE_ALWAYS_REJECT,
             "never_reject": N.OVERRIDE_NEVER_REJECT}
_POLICY = {"ftest": N.POLICY_FTEST, "chi2": N.POLICY_CHI2, "schedule": N.POLICY_SCHEDULE}


def _is_device(a) -> bool:
    return hasattr(a, "data_ptr") and getattr(a, "is_cuda", False)


def _ptr(a):
    if a is None:
        return None
    if _is_device(a):
        return a.data_ptr()
    return a.ctypes.data


def _host(a, dtype, shape=None):
    a = np.ascontiguousarray(a, dtype=dtype)
    if shape is not None:
        a = a.reshape(shape)
    return a


class FppmContext:
    """One GPU context owning every region (hit point) of a frame.

    Parameters mirror ``IntegratorConfig``/``TestConfig``/``RadiusSchedule``;
    ``samples_per_iteration`` is J (integrator.cpp:480).
    """

    def __init__(self, *, initial_radius: float, samples_per_iteration: int,
                 n_annuli: int = 2, n_sectors: int = 6, alpha_f: float = 0.01,
                 alpha_chi2: float = 0.01, channels: str = "luminance",
                 override_decision: str = "none", policy: str = "ftest",
                 k: float = 0.7, alpha: float = 0.75, r_min_base: Optional[float] = None,
                 max_depth: int = 10, normal_guard_cos: float = NORMAL_GUARD_COS,
                 max_hitpoints: int = 1, max_photons: int = 1, max_cells: int = 0,
                 device: int = 0, stream: Optional[int] = None, gather_kernel: str = "auto",
                 vcm_plus: bool = False, mis_n_vm: int = 0, mis_beta: float = 1.0, scene=None):
        self._lib = N.lib()
        cfg = N.Config()
        cfg.n_annuli, cfg.n_sectors = n_annuli, n_sectors
        cfg.alpha_f, cfg.alpha_chi2 = alpha_f, alpha_chi2
        cfg.channels = _CHANNELS[resolve_channels(channels, scene)]
        cfg.override_decision = _OVERRIDE[override_decision]
        cfg.policy = _POLICY[policy]
        cfg.k, cfg.alpha = k, alpha
        # integrator.cpp:125-126: r_min_base <= 0 resolves to 0.001 r_1
        cfg.r_min_base = (0.001 * initial_radius) if r_min_base is None else r_min_base
        cfg.initial_radius = initial_radius
        cfg.samples_per_iteration = samples_per_iteration
        cfg.max_depth, cfg.normal_guard_cos = max_depth, normal_guard_cos
        cfg.max_hitpoints, cfg.max_photons, cfg.max_cells = max_hitpoints, max_photons, max_cells
        cfg.device = device
        cfg.stream = stream
        cfg.gather_kernel = {"auto": 0, "warp": 1, "fine": 4, "3d": 5, "sparse": 5}[gather_kernel]
        cfg.vcm_plus, cfg.mis_n_vm, cfg.mis_beta = int(bool(vcm_plus)), int(mis_n_vm), float(mis_beta)
        self.config = cfg
        self.device = device
        self.G = n_annuli * n_sectors
        self.C = cfg.channels
        self._h = C.c_void_p()
        N.check(self._lib.fppm_gpu_create(C.byref(cfg), C.byref(self._h)))
        self.H = 0
        self.N = 0
        self._keep = []

    # ------------------------------------------------------------ lifecycle
    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            self._lib.fppm_gpu_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _check(self, status):
        N.check(status, self._h)

    @property
    def stream(self) -> int:
        return self._lib.fppm_gpu_stream(self._h) or 0

    def synchronize(self):
        self._check(self._lib.fppm_gpu_synchronize(self._h))

    def counters(self) -> dict:
        """Cumulative pair counters of this context."""
        c = np.zeros(4, np.uint64)
        self._check(self._lib.fppm_gpu_counters(self._h, c.ctypes.data))
        return dict(accepted=int(c[0]), candidates=int(c[1]), exact=int(c[2]), ambiguous=int(c[3]))

    @staticmethod
    def kernel_launches() -> int:
        return int(N.lib().fppm_gpu_kernel_launches())

    def record_bytes(self) -> int:
        """Bytes per sorted photon record staged by the fine gather of the
        current grid: 64 general, 48 lean, 32 flat lean, 0 other kernels."""
        return int(self._lib.fppm_gpu_record_bytes(self._h))

    def gather_kernel_ms(self) -> list:
        """Durations (ms) of the dominant gather kernel of the gathers issued
        since the previous call (CUDA events on the context stream)."""
        buf = (C.c_float * 64)()
        n = C.c_uint32(0)
        self._check(self._lib.fppm_gpu_gather_kernel_ms(self._h, buf, 64, C.byref(n)))
        return [float(buf[i]) for i in range(n.value)]

    def device_view(self) -> dict:
        v = N.DeviceView()
        self._check(self._lib.fppm_gpu_device_view_get(self._h, C.byref(v)))
        return {f: getattr(v, f) for f, _ in v._fields_}

    # ------------------------------------------------------------ regions
    def set_hitpoints(self, pos, normal, wo=None, throughput=None, albedo=None,
                      eye_depth=None, gathered=None):
        """move_to for every region (gather.cpp:54-57) plus the per-hit-point
        Bsdf/throughput of the eye vertex (integrator.cpp:433-448)."""
        dev = _is_device(pos)
        if dev:
            arrs = dict(pos=pos, normal=normal, wo=wo, throughput=throughput, albedo=albedo,
                        eye_depth=eye_depth, gathered=gathered)
            n = pos.shape[0]
        else:
            pos = _host(pos, np.float64, (-1, 3))
            n = pos.shape[0]
            normal = _host(normal, np.float64, (-1, 3))
            wo = normal if wo is None else _host(wo, np.float64, (-1, 3))
            throughput = np.ones((n, 3)) if throughput is None else _host(throughput, np.float64, (-1, 3))
            albedo = np.ones((n, 3)) if albedo is None else _host(albedo, np.float64, (-1, 3))
            eye_depth = np.ones(n, np.uint32) if eye_depth is None else _host(eye_depth, np.uint32)
            gathered = None if gathered is None else _host(gathered, np.uint8)
            arrs = dict(pos=pos, normal=normal, wo=wo, throughput=throughput, albedo=albedo,
                        eye_depth=eye_depth, gathered=gathered)
        hp = N.HitPoints(*[_ptr(arrs[k]) for k in ("pos", "normal", "wo", "throughput",
                                                    "albedo", "eye_depth", "gathered")])
        fn = self._lib.fppm_gpu_set_hitpoints_device if dev else self._lib.fppm_gpu_set_hitpoints
        self._check(fn(self._h, C.byref(hp), n))
        if not dev:
            self.synchronize()  # host arrays may be pageable temporaries
        self.H = n

    def set_hitpoint_mis(self, d_vcm, d_vm):
        """VCM+: eye-vertex MIS partials per hit point."""
        a = [_host(d_vcm, np.float64), _host(d_vm, np.float64)]
        self._check(self._lib.fppm_gpu_set_hitpoint_mis(self._h, a[0].ctypes.data, a[1].ctypes.data,
                                                        len(a[0])))

    def set_photon_mis(self, d_vcm, d_vm, cont):
        """VCM+: light-vertex MIS partials and survival per photon (photon order)."""
        a = [_host(x, np.float64) for x in (d_vcm, d_vm, cont)]
        self._check(self._lib.fppm_gpu_set_photon_mis(self._h, a[0].ctypes.data, a[1].ctypes.data,
                                                      a[2].ctypes.data, len(a[0])))
        self.synchronize()  # host arrays may be pageable temporaries

    def c5_setup(self, seed: int, n_hitpoints: int):
        """Generate the C5 workload's hit point set, its NN grid and clusters."""
        self._check(self._lib.fppm_gpu_c5_setup(self._h, seed, n_hitpoints))

    def c5_hitpoints(self, h0: int, n: int):
        self._check(self._lib.fppm_gpu_c5_hitpoints(self._h, h0, n))
        self.H = n

    def generate_raster_hitpoints(self, W: int):
        self._check(self._lib.fppm_gpu_generate_raster_hitpoints(self._h, W))
        self.H = W * W

    def reset_regions(self):
        self._check(self._lib.fppm_gpu_reset_regions(self._h))

    def regions(self):
        H, CG = self.H, self.G * self.C
        r = np.zeros(H)
        t = np.zeros(H, np.uint64)
        cnt = np.zeros((H, CG), np.uint64)
        s = np.zeros((H, CG))
        q = np.zeros((H, CG))
        self._check(self._lib.fppm_gpu_get_regions(self._h, r.ctypes.data, t.ctypes.data,
                                                   cnt.ctypes.data, s.ctypes.data, q.ctypes.data))
        return dict(radius=r, t=t, stat_count=cnt, stat_sum=s, stat_sum_sq=q)

    def set_regions(self, radius=None, t=None, stat_count=None, stat_sum=None, stat_sum_sq=None):
        H, CG = self.H, self.G * self.C
        a = [None if radius is None else _host(radius, np.float64, (H,)),
             None if t is None else _host(t, np.uint64, (H,)),
             None if stat_count is None else _host(stat_count, np.uint64, (H, CG)),
             None if stat_sum is None else _host(stat_sum, np.float64, (H, CG)),
             None if stat_sum_sq is None else _host(stat_sum_sq, np.float64, (H, CG))]
        self._check(self._lib.fppm_gpu_set_regions(self._h, *[_ptr(x) for x in a]))

    def max_radius(self) -> float:
        r = C.c_double()
        self._check(self._lib.fppm_gpu_max_radius(self._h, C.byref(r)))
        return r.value

    def max_radius_device(self, out) -> None:
        """Max live radius into device memory (a float64 CUDA tensor of one
        element), stream-ordered on the context stream, no host sync."""
        self._check(self._lib.fppm_gpu_max_radius_device(self._h, C.c_void_p(out.data_ptr())))

    def build_grid_device(self, cell) -> None:
        """Grid whose cell is read on the device from `cell` (float64 CUDA
        tensor of one element, e.g. the all-reduced max of every rank's
        max_radius_device)."""
        self._check(self._lib.fppm_gpu_build_grid_device(self._h, C.c_void_p(cell.data_ptr())))

    # ------------------------------------------------------------ photons + grid
    def set_photons(self, pos, normal, wi, power, depth):
        dev = _is_device(pos)
        if dev:
            arrs = [pos, normal, wi, power, depth]
            n = pos.shape[0]
        else:
            arrs = [_host(pos, np.float32, (-1, 3)), _host(normal, np.float32, (-1, 3)),
                    _host(wi, np.float32, (-1, 3)), _host(power, np.float32, (-1, 3)),
                    _host(depth, np.uint32)]
            n = arrs[0].shape[0]
        ph = N.Photons(*[_ptr(a) for a in arrs])
        fn = self._lib.fppm_gpu_set_photons_device if dev else self._lib.fppm_gpu_set_photons
        self._check(fn(self._h, C.byref(ph), n))
        if not dev:
            self.synchronize()
        self.N = n

    def generate_photons(self, workload: int, seed: int, iteration: int, n: int, begin: int = 0):
        self._check(self._lib.fppm_gpu_generate_photons(self._h, workload, seed, iteration, begin, n))
        self.N = n

    def set_scene(self, scene):
        """Upload an analytic scene (paper_2504_04411_b200.scene.Scene)."""
        from .scene import to_struct
        st, keep = to_struct(scene)
        self._check(self._lib.fppm_gpu_set_scene(self._h, C.byref(st)))
        del keep

    def trace_photons(self, seed: int, iteration: int, n_paths: int, max_depth: int,
                      mis_radius: float = 0.0, path0: int = 0) -> int:
        """Renderer::light_phase (integrator.cpp:230-265) on the device: traces
        light sub-paths [path0, path0 + n_paths) and stages their non-delta
        vertices, in path order, as the photons of the next grid build.
        Returns the count."""
        n = C.c_uint32()
        self._check(self._lib.fppm_gpu_trace_photons_range(self._h, seed, iteration, path0, n_paths, max_depth,
                                                           mis_radius, C.byref(n)))
        self.N = n.value
        return n.value

    def set_photons_packed(self, packed, part_n, margin=None) -> int:
        """Stage photon shares packed [parts][13][stride] (a uint32/int32/float32
        CUDA tensor, e.g. one all-gather of pack_photons() outputs), in part
        order; with `margin` (float64 CUDA tensor of one element) only the
        photons within the hit points' box grown by it are kept.  Returns the
        staged count."""
        parts = len(part_n)
        stride = packed.shape[-1]
        arr = (C.c_uint32 * max(parts, 1))(*part_n)
        n = C.c_uint32()
        self._check(self._lib.fppm_gpu_set_photons_packed(
            self._h, C.c_void_p(packed.data_ptr()), parts, stride, arr,
            C.c_void_p(margin.data_ptr()) if margin is not None else None, C.byref(n)))
        self.N = n.value
        return n.value

    def set_camera(self, camera):
        """Pinhole camera (scene.Camera); clears the film."""
        from .scene import Camera  # noqa: F401
        c = N.CameraStruct((C.c_double * 3)(*camera.position), (C.c_double * 3)(*camera.look_at),
                           (C.c_double * 3)(*camera.up), float(camera.vfov_deg), int(camera.width),
                           int(camera.height))
        self._check(self._lib.fppm_gpu_set_camera(self._h, C.byref(c)))
        self.camera = camera

    def trace_eye(self, seed: int, iteration: int):
        """pixel_pm's camera walk (integrator.cpp:407-474): one hit point per
        pixel (gathered = 0 where the walk found no rough surface)."""
        self._check(self._lib.fppm_gpu_trace_eye(self._h, seed, iteration))
        self.H = self.camera.width * self.camera.height

    def get_hitpoints(self, emitted: bool = False) -> dict:
        H = self.H
        o = dict(pos=np.zeros((H, 3)), nrm=np.zeros((H, 3)), wo=np.zeros((H, 3)), thr=np.zeros((H, 3)),
                 alb=np.zeros((H, 3)), eye_depth=np.zeros(H, np.uint32), gathered=np.zeros(H, np.uint8))
        hp = N.HitPoints(*[o[k].ctypes.data for k in ("pos", "nrm", "wo", "thr", "alb", "eye_depth",
                                                       "gathered")])
        em = np.zeros((H, 3)) if emitted else None
        self._check(self._lib.fppm_gpu_get_hitpoints(self._h, C.byref(hp), _ptr(em)))
        if emitted:
            o["emitted"] = em
        return o

    def film_add(self):
        self._check(self._lib.fppm_gpu_film_add(self._h))

    def film_mean(self):
        """(image [height, width, 3] fp64, iterations)."""
        n = self.camera.width * self.camera.height
        out = np.zeros((n, 3))
        it = C.c_uint64()
        self._check(self._lib.fppm_gpu_film_mean(self._h, out.ctypes.data, C.byref(it)))
        return out.reshape(self.camera.height, self.camera.width, 3), it.value

    def film_splits(self):
        """(vc, vm): per-pixel cumulative luminance of the non-merge and the
        merge estimates (Film::vc_total / vm_total), [height, width] each."""
        n = self.camera.width * self.camera.height
        vc, vm = np.zeros(n), np.zeros(n)
        self._check(self._lib.fppm_gpu_film_splits(self._h, vc.ctypes.data, vm.ctypes.data))
        return vc.reshape(self.camera.height, self.camera.width), vm.reshape(self.camera.height, self.camera.width)

    def render_iteration(self, seed: int, iteration: int, light_paths: int, max_depth: Optional[int] = None,
                         outputs: bool = False, stats: bool = False):
        """One full FPPM iteration of Renderer::step on the device: light
        phase, eye pass, grid + gather + F-test, film."""
        self.trace_photons(seed, iteration, light_paths, max_depth or self.config.max_depth)
        self.trace_eye(seed, iteration)
        o, sm = self.iterate(iteration, outputs=outputs, stats=stats, summary=outputs or stats)
        self.film_add()
        return o, sm

    def render_vcm_iteration(self, seed: int, iteration: int, light_paths: int, max_depth: Optional[int] = None):
        """One whole VCM+ iteration of Renderer::step (Algorithm::vcm_plus) on the
        device: light sub-paths + camera splats, eye sub-paths with emitter
        hits, next-event estimation and connections, merges at every rough eye
        vertex (the primary one tested per pixel), film
        (fppm_gpu_render_vcm)."""
        n = C.c_uint32()
        self._check(self._lib.fppm_gpu_render_vcm(self._h, seed, iteration, light_paths,
                                                  max_depth or self.config.max_depth, C.byref(n)))
        self.N = n.value
        self.H = self.camera.width * self.camera.height

    def get_photon_mis(self) -> dict:
        n = self.N
        o = dict(d_vcm=np.zeros(n), d_vm=np.zeros(n), cont=np.zeros(n))
        self._check(self._lib.fppm_gpu_get_photon_mis(self._h, o["d_vcm"].ctypes.data, o["d_vm"].ctypes.data,
                                                      o["cont"].ctypes.data))
        return o

    def get_photons(self) -> dict:
        n = self.N
        o = dict(pos=np.zeros((n, 3), np.float32), nrm=np.zeros((n, 3), np.float32),
                 wi=np.zeros((n, 3), np.float32), pow=np.zeros((n, 3), np.float32),
                 depth=np.zeros(n, np.uint32))
        self._check(self._lib.fppm_gpu_get_photons(self._h, *[o[k].ctypes.data for k in
                                                              ("pos", "nrm", "wi", "pow", "depth")]))
        return o

    def build_grid(self, cell_size: float = 0.0):
        self._check(self._lib.fppm_gpu_build_grid(self._h, cell_size))

    def export_grid(self):
        """(keys, begin, end, order) in the reference PhotonGrid layout."""
        nc = C.c_uint64()
        self._check(self._lib.fppm_gpu_export_grid(self._h, None, None, None, None, C.byref(nc)))
        keys = np.zeros(nc.value, np.uint64)
        b = np.zeros(nc.value, np.uint32)
        e = np.zeros(nc.value, np.uint32)
        order = np.zeros(self.N, np.uint32)
        self._check(self._lib.fppm_gpu_export_grid(self._h, keys.ctypes.data, b.ctypes.data,
                                                   e.ctypes.data, order.ctypes.data, C.byref(nc)))
        return keys, b, e, order

    def query_ball(self, centers, radii, cap: Optional[int] = None):
        centers = _host(centers, np.float64, (-1, 3))
        radii = _host(radii, np.float64)
        nq = len(radii)
        offsets = np.zeros(nq + 1, np.uint64)
        total = C.c_uint64()
        self._check(self._lib.fppm_gpu_query_ball(self._h, centers.ctypes.data, radii.ctypes.data,
                                                  nq, offsets.ctypes.data, None, 0, C.byref(total)))
        idx = np.zeros(max(total.value, 1), np.uint32)
        self._check(self._lib.fppm_gpu_query_ball(self._h, centers.ctypes.data, radii.ctypes.data,
                                                  nq, offsets.ctypes.data, idx.ctypes.data,
                                                  total.value, C.byref(total)))
        return [idx[offsets[q]:offsets[q + 1]].copy() for q in range(nq)]

    # ------------------------------------------------------------ hot path
    def _out(self, outputs: bool, stats: bool, gather: bool, n: Optional[int] = None):
        if not outputs and not stats:
            return None, None
        H, CG = (self.H if n is None else n), self.G * self.C
        o = {}
        if outputs:
            o.update(radius=np.zeros(H), gather_radius=np.zeros(H), t=np.zeros(H, np.uint64),
                     tested=np.zeros(H, np.uint8), rejected=np.zeros(H, np.uint8),
                     statistic=np.zeros(H), critical=np.zeros(H))
            if gather:
                o.update(flux=np.zeros((H, 3)), radiance=np.zeros((H, 3), np.float32),
                         accepted=np.zeros(H, np.uint32))
        if stats:
            o.update(stat_count=np.zeros((H, CG), np.uint64), stat_sum=np.zeros((H, CG)),
                     stat_sum_sq=np.zeros((H, CG)))
        io = N.IterOut(*[o[f].ctypes.data if f in o else None for f, _ in N.IterOut._fields_])
        return o, io

    def gather_test(self, iteration: int, outputs: bool = True, stats: bool = False,
                    summary: bool = True):
        o, io = self._out(outputs, stats, True)
        sm = N.Summary() if summary else None
        self._check(self._lib.fppm_gpu_gather_test(self._h, iteration,
                                                   C.byref(io) if io is not None else None,
                                                   C.byref(sm) if sm is not None else None))
        if o is not None:
            self.synchronize()  # outputs are written asynchronously
        return o, (sm.as_dict() if sm is not None else None)

    def iterate(self, iteration: int, outputs: bool = True, stats: bool = False,
                summary: bool = True):
        """One FPPM iteration: grid at the max live radius + gather + test."""
        o, io = self._out(outputs, stats, True)
        sm = N.Summary() if summary else None
        self._check(self._lib.fppm_gpu_iterate(self._h, iteration,
                                               C.byref(io) if io is not None else None,
                                               C.byref(sm) if sm is not None else None))
        if o is not None:
            self.synchronize()  # outputs are written asynchronously
        return o, (sm.as_dict() if sm is not None else None)

    # ---------------------------------------- multi-GPU option B (photon-sharded)
    @property
    def delta_stride(self) -> int:
        return int(self._lib.fppm_gpu_delta_stride(self._h))

    def _stream_handoff(self, rows, to_ctx: bool):
        """Order the context stream after torch's current stream (to_ctx) or
        the other way round, without a host synchronization."""
        if not _is_device(rows):
            return
        import torch
        ctx_stream = torch.cuda.ExternalStream(self.stream, device=rows.device)
        cur = torch.cuda.current_stream(rows.device)
        src, dst = (cur, ctx_stream) if to_ctx else (ctx_stream, cur)
        ev = torch.cuda.Event()
        ev.record(src)
        dst.wait_event(ev)

    def radius_tensor(self):
        """torch view (no copy) of the context's live radii [H] fp64 on the
        device: the all-gather of option B writes into it."""
        import torch

        class _View:
            def __init__(self, ptr, n):
                self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False),
                                                 "version": 3, "strides": None}
        v = self.device_view()
        return torch.as_tensor(_View(v["radius"], self.H), device=f"cuda:{self.device}")

    def gather_deltas(self, iteration: int, rows):
        """Partial sums of this context's photons for every hit point into the
        device tensor ``rows`` ([H, delta_stride] fp64); no state change.
        Stream-ordered with torch's current stream on both sides."""
        self._stream_handoff(rows, True)
        self._check(self._lib.fppm_gpu_gather_deltas(self._h, iteration, _ptr(rows)))
        self._stream_handoff(rows, False)

    def apply_deltas(self, iteration: int, h0: int, rows, outputs: bool = True, stats: bool = False,
                     summary: bool = False):
        """Pool rows (device [n, delta_stride], summed over ranks) into regions
        [h0, h0 + n) and run the end-of-iteration policy; outputs cover the slice."""
        n = int(rows.shape[0])
        o, io = self._out(outputs, stats, True, n=n)
        self._stream_handoff(rows, True)
        sm = N.Summary() if summary else None
        self._check(self._lib.fppm_gpu_apply_deltas(self._h, iteration, h0, n, _ptr(rows),
                                                    C.byref(io) if io is not None else None,
                                                    C.byref(sm) if sm is not None else None))
        if o is not None:
            self.synchronize()
        return o, (sm.as_dict() if sm is not None else None)

    def accumulate(self, region, y, value):
        region = _host(region, np.uint32)
        y = _host(y, np.float64, (-1, 2))
        value = _host(value, np.float64, (-1, 3))
        self._check(self._lib.fppm_gpu_accumulate(self._h, region.ctypes.data, y.ctypes.data,
                                                  value.ctypes.data, len(region)))

    def set_samples_per_iteration(self, J: int):
        self._check(self._lib.fppm_gpu_set_samples_per_iteration(self._h, J))

    def end_iteration(self, iteration: int, outputs: bool = True, stats: bool = False):
        o, io = self._out(outputs, stats, False)
        self._check(self._lib.fppm_gpu_end_iteration(self._h, iteration,
                                                     C.byref(io) if io is not None else None))
        if o is not None:
            self.synchronize()
        return o


# ---------------------------------------------------------------------------
class PhotonGrid:
    """Mirror of fppm::PhotonGrid (photon_map.hpp:15-42) on the GPU.

    ``vertices`` is an (n, 3) array of positions or a dict with ``pos`` and
    optionally ``normal``/``wi``/``power``/``depth``.
    """

    def __init__(self, vertices, cell_size: float, device: int = 0):
        if not (cell_size > 0.0):
            raise InvalidArgument("PhotonGrid: cell size must be positive")
        v = vertices if isinstance(vertices, dict) else {"pos": vertices}
        pos = _host(v["pos"], np.float32, (-1, 3))
        n = len(pos)
        z3 = np.zeros((n, 3), np.float32)
        self._v = dict(pos=pos, normal=v.get("normal", z3), wi=v.get("wi", z3),
                       power=v.get("power", z3), depth=v.get("depth", np.zeros(n, np.uint32)))
        self._cell = float(cell_size)
        self._ctx = FppmContext(initial_radius=cell_size, samples_per_iteration=1, n_annuli=1,
                                n_sectors=4, max_hitpoints=1, max_photons=max(n, 1), device=device)
        self._ctx.set_photons(**self._v)
        self._ctx.build_grid(self._cell)

    def size(self) -> int:
        return len(self._v["pos"])

    def cell_size(self) -> float:
        return self._cell

    def vertices(self) -> dict:
        return self._v

    def query_ball(self, center, r: float) -> np.ndarray:
        """Indices with |pos - center|^2 <= r^2 in reference visit order."""
        return self._ctx.query_ball(np.asarray(center, np.float64).reshape(1, 3), [r])[0]

    def query_ball_batch(self, centers, radii):
        return self._ctx.query_ball(centers, radii)

    def internals(self):
        """(keys_, begin/end of cells_, order_) of the reference layout."""
        return self._ctx.export_grid()


class GatherRegionBatch:
    """``count`` fppm::GatherRegion objects (gather.hpp:69-112) on the GPU.

    Same constructor validation as GatherRegion (gather.cpp:35-52); all
    regions share TestConfig/RadiusSchedule/initial radius.
    """

    def __init__(self, test: TestConfig, schedule: RadiusSchedule, initial_radius: float,
                 count: int = 1, samples_per_iteration: int = 1, policy: str = "ftest",
                 device: int = 0):
        if not (initial_radius > 0):
            raise InvalidArgument("GatherRegion requires a positive initial radius")
        if not (0 < schedule.k < 1):
            raise InvalidArgument("RadiusSchedule requires k in (0,1)")
        if not (0.5 <= schedule.alpha < 1):
            raise InvalidArgument("RadiusSchedule requires alpha in [0.5,1)")
        if not (0 < schedule.r_min_base <= initial_radius):
            raise InvalidArgument("RadiusSchedule requires 0 < r_min_base <= r_1")
        if test.n_annuli * test.n_sectors < 2:
            raise InvalidArgument("GatherRegion requires at least 2 sectors")
        self.test, self.schedule = test, schedule
        self._J = samples_per_iteration
        self._ctx = FppmContext(
            initial_radius=initial_radius, samples_per_iteration=samples_per_iteration,
            n_annuli=test.n_annuli, n_sectors=test.n_sectors, alpha_f=test.alpha_f,
            alpha_chi2=test.alpha_chi2, channels=test.channels,
            override_decision=test.override_decision, k=schedule.k, alpha=schedule.alpha,
            r_min_base=schedule.r_min_base, policy=policy, max_hitpoints=count, max_photons=1,
            device=device)
        z = np.zeros((count, 3))
        n = np.tile([0.0, 0.0, 1.0], (count, 1))
        self._ctx.set_hitpoints(z, n)
        self.count = count

    def accumulate(self, region, y, value):
        """GatherRegion::accumulate for samples (region index, y=(u,v), rgb)."""
        self._ctx.accumulate(region, y, value)

    def end_iteration(self, i: int, samples_per_iteration: int):
        if samples_per_iteration != self._J:
            self._ctx.set_samples_per_iteration(samples_per_iteration)
            self._J = samples_per_iteration
        return self._ctx.end_iteration(i)

    def radius(self):
        return self._ctx.regions()["radius"]

    def held_iterations(self):
        return self._ctx.regions()["t"]

    def sector_count(self) -> int:
        return self.test.n_annuli * self.test.n_sectors

    def channel_count(self) -> int:
        return 3 if self.test.channels == "rgb" else 1

    def sector_stats(self, region: int, channel: int = 0):
        """(count, sum, sum_sq) arrays of one region's channel."""
        r = self._ctx.regions()
        G = self.sector_count()
        sl = slice(channel * G, (channel + 1) * G)
        return r["stat_count"][region, sl], r["stat_sum"][region, sl], r["stat_sum_sq"][region, sl]


def schedule_radius(base: float, alpha: float, i: int) -> float:
    """gather.cpp:11-13 (host libm, bit-identical to the reference)."""
    return N.lib().fppm_gpu_schedule_radius(base, alpha, i)


def f_quantile(p: float, d1: float, d2: float) -> float:
    st = C.c_int(0)
    v = N.lib().fppm_gpu_f_quantile(p, d1, d2, C.byref(st))
    N.check(st.value)
    return v


def chi2_quantile(p: float, df: float) -> float:
    st = C.c_int(0)
    v = N.lib().fppm_gpu_chi2_quantile(p, df, C.byref(st))
    N.check(st.value)
    return v
