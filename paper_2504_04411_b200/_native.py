"""ctypes binding of libfppm_gpu.so (include/fppm_gpu.h).

The shared library is built in-tree by ``paper_2504_04411_b200/csrc/Makefile``
(``__graft_entry__.build()``).  There is no CPU fallback: importing the
binding without the library, or creating a context without an sm_100 GPU,
raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FPPM_GPU_LIB") or os.path.join(HERE, "libfppm_gpu.so")

FPPM_OK = 0
FPPM_ERR_INVALID_ARGUMENT = 1
FPPM_ERR_DOMAIN = 2
FPPM_ERR_CUDA = 3
FPPM_ERR_CAPACITY = 4
FPPM_ERR_STATE = 5
FPPM_ERR_NO_DEVICE = 6

CHANNELS_LUMINANCE = 1
CHANNELS_RGB = 3
OVERRIDE_NONE, OVERRIDE_ALWAYS_REJECT, OVERRIDE_NEVER_REJECT = 0, 1, 2
POLICY_FTEST, POLICY_CHI2, POLICY_SCHEDULE = 0, 1, 2
WORKLOAD_C1, WORKLOAD_C2 = 1, 2

_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_u8p = C.POINTER(C.c_uint8)


class FppmError(RuntimeError):
    """Base class; ``status`` holds the fppm_status code."""

    status = -1


class InvalidArgument(FppmError, ValueError):
    """Reference std::invalid_argument."""

    status = FPPM_ERR_INVALID_ARGUMENT


class DomainError(FppmError, ArithmeticError):
    """Reference std::domain_error."""

    status = FPPM_ERR_DOMAIN


class CudaError(FppmError):
    status = FPPM_ERR_CUDA


class CapacityError(FppmError):
    status = FPPM_ERR_CAPACITY


class StateError(FppmError):
    status = FPPM_ERR_STATE


class NoDeviceError(FppmError):
    status = FPPM_ERR_NO_DEVICE


_ERRORS = {c.status: c for c in (InvalidArgument, DomainError, CudaError, CapacityError,
                                 StateError, NoDeviceError)}


class Config(C.Structure):
    _fields_ = [
        ("n_annuli", C.c_int32), ("n_sectors", C.c_int32),
        ("alpha_f", C.c_double), ("alpha_chi2", C.c_double),
        ("channels", C.c_int32), ("override_decision", C.c_int32), ("policy", C.c_int32),
        ("k", C.c_double), ("alpha", C.c_double), ("r_min_base", C.c_double),
        ("initial_radius", C.c_double), ("samples_per_iteration", C.c_uint64),
        ("max_depth", C.c_uint32), ("normal_guard_cos", C.c_double),
        ("max_hitpoints", C.c_uint32), ("max_photons", C.c_uint32), ("max_cells", C.c_uint32),
        ("device", C.c_int32), ("stream", C.c_void_p), ("gather_kernel", C.c_int32),
        ("vcm_plus", C.c_int32), ("mis_n_vm", C.c_int32), ("mis_beta", C.c_double),
    ]


class HitPoints(C.Structure):
    _fields_ = [("pos", C.c_void_p), ("normal", C.c_void_p), ("wo", C.c_void_p),
                ("throughput", C.c_void_p), ("albedo", C.c_void_p),
                ("eye_depth", C.c_void_p), ("gathered", C.c_void_p)]


class Photons(C.Structure):
    _fields_ = [("pos", C.c_void_p), ("normal", C.c_void_p), ("wi", C.c_void_p),
                ("power", C.c_void_p), ("depth", C.c_void_p)]


class IterOut(C.Structure):
    _fields_ = [("radius", C.c_void_p), ("gather_radius", C.c_void_p), ("t", C.c_void_p),
                ("tested", C.c_void_p), ("rejected", C.c_void_p), ("statistic", C.c_void_p),
                ("critical", C.c_void_p), ("flux", C.c_void_p), ("radiance", C.c_void_p),
                ("accepted", C.c_void_p), ("stat_count", C.c_void_p), ("stat_sum", C.c_void_p),
                ("stat_sum_sq", C.c_void_p)]


class Summary(C.Structure):
    _fields_ = [("accepted", C.c_uint64), ("candidates", C.c_uint64),
                ("exact_pairs", C.c_uint64), ("ambiguous_pairs", C.c_uint64),
                ("tested", C.c_uint32), ("rejected", C.c_uint32),
                ("cell_size", C.c_double), ("r_max_next", C.c_double), ("cells", C.c_uint64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class DeviceView(C.Structure):
    _fields_ = [("photon_pos", C.c_void_p), ("photon_normal", C.c_void_p),
                ("photon_wi", C.c_void_p), ("photon_power", C.c_void_p),
                ("photon_depth", C.c_void_p), ("radius", C.c_void_p), ("counters", C.c_void_p)]


class CameraStruct(C.Structure):
    _fields_ = [("position", C.c_double * 3), ("look_at", C.c_double * 3), ("up", C.c_double * 3),
                ("vfov_deg", C.c_double), ("width", C.c_int32), ("height", C.c_int32)]


# (name, restype, argtypes)
_SIGS = [
    ("fppm_gpu_abi_version", C.c_int, []),
    ("fppm_gpu_status_string", C.c_char_p, [C.c_int]),
    ("fppm_gpu_create", C.c_int, [C.POINTER(Config), C.POINTER(C.c_void_p)]),
    ("fppm_gpu_destroy", C.c_int, [C.c_void_p]),
    ("fppm_gpu_last_error", C.c_char_p, [C.c_void_p]),
    ("fppm_gpu_synchronize", C.c_int, [C.c_void_p]),
    ("fppm_gpu_stream", C.c_void_p, [C.c_void_p]),
    ("fppm_gpu_device_view_get", C.c_int, [C.c_void_p, C.POINTER(DeviceView)]),
    ("fppm_gpu_set_hitpoints", C.c_int, [C.c_void_p, C.POINTER(HitPoints), C.c_uint32]),
    ("fppm_gpu_set_hitpoints_device", C.c_int, [C.c_void_p, C.POINTER(HitPoints), C.c_uint32]),
    ("fppm_gpu_generate_raster_hitpoints", C.c_int, [C.c_void_p, C.c_uint32]),
    ("fppm_gpu_reset_regions", C.c_int, [C.c_void_p]),
    ("fppm_gpu_get_regions", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("fppm_gpu_set_regions", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("fppm_gpu_max_radius", C.c_int, [C.c_void_p, _dp]),
    ("fppm_gpu_max_radius_device", C.c_int, [C.c_void_p, C.c_void_p]),
    ("fppm_gpu_build_grid_device", C.c_int, [C.c_void_p, C.c_void_p]),
    ("fppm_gpu_set_photons", C.c_int, [C.c_void_p, C.POINTER(Photons), C.c_uint32]),
    ("fppm_gpu_set_photons_device", C.c_int, [C.c_void_p, C.POINTER(Photons), C.c_uint32]),
    ("fppm_gpu_set_photons_packed", C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint64, C.c_void_p,
                                              C.c_void_p, C.POINTER(C.c_uint32)]),
    ("fppm_gpu_prefetch_photons", C.c_int, [C.c_void_p, C.POINTER(Photons), C.c_uint32, _u64p]),
    ("fppm_gpu_adopt_photons", C.c_int, [C.c_void_p, C.c_uint64]),
    ("fppm_gpu_generate_photons", C.c_int, [C.c_void_p, C.c_int32, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32]),
    ("fppm_gpu_generate_photons_to", C.c_int, [C.c_void_p, C.c_int32, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32, C.POINTER(Photons)]),
    ("fppm_gpu_get_photons", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("fppm_gpu_build_grid", C.c_int, [C.c_void_p, C.c_double]),
    ("fppm_gpu_export_grid", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, _u64p]),
    ("fppm_gpu_query_ball", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p, C.c_uint64, _u64p]),
    ("fppm_gpu_gather_test", C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(IterOut), C.POINTER(Summary)]),
    ("fppm_gpu_iterate", C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(IterOut), C.POINTER(Summary)]),
    ("fppm_gpu_accumulate", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32]),
    ("fppm_gpu_set_samples_per_iteration", C.c_int, [C.c_void_p, C.c_uint64]),
    ("fppm_gpu_end_iteration", C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(IterOut)]),
    ("fppm_gpu_set_policy", C.c_int, [C.c_void_p, C.c_int32]),
    ("fppm_gpu_sector_index", C.c_int, [C.c_double, C.c_double, C.c_double, C.c_int32, C.c_int32,
                                        C.POINTER(C.c_int32)]),
    ("fppm_gpu_build_frame", C.c_int, [_dp, _dp, _dp]),
    ("fppm_gpu_kernel_launches", C.c_uint64, []),
    ("fppm_gpu_record_bytes", C.c_int, [C.c_void_p]),
    ("fppm_gpu_gather_kernel_ms", C.c_int, [C.c_void_p, C.POINTER(C.c_float), C.c_uint32, C.POINTER(C.c_uint32)]),
    ("fppm_gpu_counters", C.c_int, [C.c_void_p, C.c_void_p]),
    ("fppm_gpu_set_hitpoint_mis", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32]),
    ("fppm_gpu_set_photon_mis", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32]),
    ("fppm_gpu_set_scene", C.c_int, [C.c_void_p, C.c_void_p]),
    ("fppm_gpu_trace_photons", C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_double,
                                         C.POINTER(C.c_uint32)]),
    ("fppm_gpu_trace_photons_range", C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32,
                                               C.c_uint32, C.c_double, C.POINTER(C.c_uint32)]),
    ("fppm_gpu_get_photon_mis", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("fppm_gpu_c5_setup", C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32]),
    ("fppm_gpu_c5_hitpoints", C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32]),
    ("fppm_gpu_set_camera", C.c_int, [C.c_void_p, C.c_void_p]),
    ("fppm_gpu_trace_eye", C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64]),
    ("fppm_gpu_film_add", C.c_int, [C.c_void_p]),
    ("fppm_gpu_render_vcm", C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_void_p]),
    ("fppm_gpu_get_hitpoints", C.c_int, [C.c_void_p, C.POINTER(HitPoints), C.c_void_p]),
    ("fppm_gpu_film_mean", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64)]),
    ("fppm_gpu_film_splits", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    ("fppm_gpu_delta_stride", C.c_uint32, [C.c_void_p]),
    ("fppm_gpu_gather_deltas", C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p]),
    ("fppm_gpu_apply_deltas", C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_void_p,
                                        C.POINTER(IterOut), C.POINTER(Summary)]),
    ("fppm_gpu_schedule_radius", C.c_double, [C.c_double, C.c_double, C.c_uint64]),
    ("fppm_gpu_f_quantile", C.c_double, [C.c_double, C.c_double, C.c_double, C.POINTER(C.c_int)]),
    ("fppm_gpu_chi2_quantile", C.c_double, [C.c_double, C.c_double, C.POINTER(C.c_int)]),
]

EXPORTED = [s[0] for s in _SIGS]

_lib = None


def lib():
    """Load libfppm_gpu.so once; raise loudly when it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                "(there is no CPU fallback for the hot path)")
        L = C.CDLL(LIB_PATH)
        for name, res, args in _SIGS:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(status, ctx=None):
    if status == FPPM_OK:
        return
    msg = lib().fppm_gpu_status_string(status).decode()
    if ctx:
        detail = lib().fppm_gpu_last_error(ctx)
        if detail:
            msg = f"{msg}: {detail.decode()}"
    raise _ERRORS.get(status, FppmError)(msg)
