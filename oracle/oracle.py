"""ctypes bindings for the parity checkers -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this module, and only as the checker or
the CPU baseline.  The product package never imports it.

Two checkers share one Python interface:

* ``Oracle("port")``      -> oracle/liboracle.so, the plain-C restatement
  (fppm_oracle.c) of the reference path;
* ``Oracle("reference")`` -> oracle/_ref/libfppm_ref.so, the reference's own
  proj/core sources compiled unmodified plus the extern "C" driver
  oracle/ref_driver.cpp.
"""
from __future__ import annotations

import ctypes as C
import os
import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PORT = os.path.join(HERE, "liboracle.so")
LIB_REF = os.path.join(HERE, "_ref", "libfppm_ref.so")

_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_u8p = C.POINTER(C.c_uint8)
_ip = C.POINTER(C.c_int)


def _ptr(a, t):
    if a is None:
        return C.cast(None, t)
    return a.ctypes.data_as(t)


class Config(C.Structure):
    """Mirror of orc_config / RefConfig."""

    _fields_ = [
        ("n_annuli", C.c_int), ("n_sectors", C.c_int), ("alpha_f", C.c_double),
        ("channels", C.c_int), ("override_decision", C.c_int),
        ("k", C.c_double), ("alpha", C.c_double), ("r_min_base", C.c_double),
        ("initial_radius", C.c_double), ("samples_per_iteration", C.c_uint64),
        ("max_depth", C.c_uint32), ("normal_guard_cos", C.c_double),
        ("threads", C.c_int), ("alpha_chi2", C.c_double), ("policy", C.c_int),
        ("vcm_plus", C.c_int), ("mis_n_vm", C.c_int), ("mis_beta", C.c_double),
    ]


class IterOut(C.Structure):
    _fields_ = [
        ("radius", _dp), ("gather_r", _dp), ("t", _u64p), ("tested", _u8p),
        ("rejected", _u8p), ("statistic", _dp), ("critical", _dp),
        ("flux", _dp), ("radiance", _dp), ("accepted", _u64p),
        ("stat_count", _u64p), ("stat_sum", _dp), ("stat_sum_sq", _dp),
    ]


class OracleError(RuntimeError):
    pass


class InvalidArgument(OracleError, ValueError):
    pass


class DomainError(OracleError, ArithmeticError):
    pass


def _raise(code):
    if code == 1:
        raise InvalidArgument("invalid argument")
    if code == 2:
        raise DomainError("domain error")
    if code:
        raise OracleError(f"oracle error {code}")


class Oracle:
    """Uniform Python view over liboracle.so ('port') or _ref ('reference')."""

    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = LIB_PORT if kind == "port" else LIB_REF
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing; run `make -C oracle`")
        self.lib = L = C.CDLL(path)
        self.p = "orc_" if kind == "port" else "ref_"
        p = self.p
        def fn(name, res, args):
            f = getattr(L, p + name)
            f.restype = res
            f.argtypes = args
            return f
        self._sector = fn("sector_index", C.c_int, [C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, _ip])
        self._sched = fn("schedule_radius", C.c_double, [C.c_double, C.c_double, C.c_uint64])
        self._fq = fn("f_quantile", C.c_double, [C.c_double, C.c_double, C.c_double, _ip])
        self._cq = fn("chi2_quantile", C.c_double, [C.c_double, C.c_double, _ip])
        self._fcdf = fn("f_cdf", C.c_double, [C.c_double, C.c_double, C.c_double, _ip])
        self._ccdf = fn("chi2_cdf", C.c_double, [C.c_double, C.c_double, _ip])
        self._ib = fn("reg_inc_beta", C.c_double, [C.c_double, C.c_double, C.c_double, _ip])
        self._lg = fn("reg_lower_gamma", C.c_double, [C.c_double, C.c_double, _ip])
        self._fs = fn("f_statistic", C.c_double, [_u64p, _dp, _dp, C.c_int, C.c_uint64, _ip])
        self._c2s = fn("chi2_statistic", C.c_double, [_u64p, C.c_int, _ip])
        self._frame = fn("build_frame", None, [_dp, _dp, _dp])
        self._gb = fn("grid_build", C.c_void_p, [_dp, C.c_size_t, C.c_double, _ip])
        self._gf = fn("grid_free", None, [C.c_void_p])
        self._gc = fn("grid_cell_count", C.c_size_t, [C.c_void_p])
        self._ge = fn("grid_export", None, [C.c_void_p, _u64p, _u32p, _u32p, _u32p])
        self._gq = fn("grid_query_ball", C.c_size_t, [C.c_void_p, _dp, C.c_double, _u32p, C.c_size_t, _ip])
        self._sc = fn("session_create", C.c_void_p, [C.POINTER(Config), C.c_size_t, _dp, _dp, _dp, _dp, _dp, _u32p, _u8p, _ip])
        self._sf = fn("session_free", None, [C.c_void_p])
        self._smr = fn("session_max_radius", C.c_double, [C.c_void_p])
        self._seye = fn("session_set_eye_mis", None, [C.c_void_p, _dp, _dp])
        self._shp = fn("session_set_hitpoints", None, [C.c_void_p, _dp, _dp, _dp, _dp, _dp, _u32p, _u8p])
        self._sphm = fn("session_set_photon_mis", None, [C.c_void_p, _dp, _dp, _dp, C.c_size_t])
        self._mwm = fn("mis_weight_merge", C.c_double, [C.c_int, C.c_double, C.c_double, C.c_double,
                                                        C.c_double, C.c_double, C.c_double,
                                                        C.c_double, C.c_double])
        if kind == "port":
            self._si = fn("session_iterate", C.c_int, [C.c_void_p, C.c_uint64, _fp, _fp, _fp, _fp, _u32p, C.c_size_t, C.c_double, _u32p, C.c_size_t, C.POINTER(IterOut)])
            self._gen = fn("gen_photons", None, [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, _fp, _fp, _fp, _fp, _u32p])
            self._ghp = fn("gen_raster_hitpoints", None, [C.c_uint32, _dp, _dp, _dp, _dp, _dp, _u32p])
            self._pcg = fn("pcg32_at", C.c_uint32, [C.c_uint64, C.c_uint64, C.c_uint64])
            self._sincos = fn("dm_sincos2pi", None, [C.c_double, _dp, _dp])
            self._log = fn("dm_log", C.c_double, [C.c_double])
            self._exp = fn("dm_exp", C.c_double, [C.c_double])
            self._fcrit = fn("f_critical", C.c_double, [C.c_int64, C.c_int64, C.c_double])
            self._c5c = fn("c5_create", C.c_void_p, [C.c_uint64, C.c_uint32])
            self._c5f = fn("c5_free", None, [C.c_void_p])
            self._c5h = fn("c5_hitpoints", None, [C.c_void_p, C.c_uint32, C.c_uint32] + [C.c_void_p] * 6)
            self._c5p = fn("c5_photons", None, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64] + [C.c_void_p] * 5)
        else:
            self._si = fn("session_iterate", C.c_int, [C.c_void_p, C.c_uint64, _fp, _fp, _fp, _fp, _u32p, C.c_size_t, C.c_double, _u32p, C.c_size_t, C.POINTER(IterOut), _dp, _dp])
            self._si64 = fn("session_iterate_f64", C.c_int, [C.c_void_p, C.c_uint64, _dp, _dp, _dp, _dp, _u32p, C.c_size_t, C.c_double, _u32p, C.c_size_t, C.POINTER(IterOut), _dp, _dp])
            self._anova = fn("anova_f_test", None, [_u64p, _dp, _dp, C.c_int, C.c_uint64, C.c_double, _dp, _ip])
            self._hw = fn("hardware_threads", C.c_uint, [])
            self._scn = fn("scene_create", C.c_void_p, [C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p,
                                                        C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p,
                                                        C.c_uint32, C.c_void_p, C.c_void_p])
            self._scnf = fn("scene_free", None, [C.c_void_p])
            self._eye = fn("eye_pass", None, [C.c_void_p, _dp, C.c_double, C.c_int, C.c_int, C.c_uint64,
                                              C.c_uint64, C.c_uint32] + [C.c_void_p] * 8)
            self._render = fn("render_fppm", C.c_int, [C.c_void_p, _dp, C.c_double, C.c_int, C.c_int,
                                                       C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint64,
                                                       C.c_double, C.c_int, C.c_int, C.c_double, C.c_int,
                                                       C.c_void_p, C.c_void_p, _dp])
            self._render_vcm = fn("render_vcm_plus", C.c_int, [C.c_void_p, _dp, C.c_double, C.c_int, C.c_int,
                                                               C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint64,
                                                               C.c_double, C.c_int, C.c_int, C.c_double, C.c_int,
                                                               C.c_void_p, C.c_void_p, _dp])
            self._brad = fn("bounding_radius", C.c_double, [C.c_void_p])
            self._ser = fn("serialize_scene", C.c_long, [C.c_char_p, C.c_char_p, C.c_size_t])
            self._wcsv = fn("write_convergence_csv", C.c_int, [C.c_char_p, C.c_size_t] + [C.c_void_p] * 5)
            self._rcsv = fn("read_convergence_csv", C.c_long, [C.c_char_p, C.c_size_t] + [C.c_void_p] * 5 +
                            [C.c_char_p, C.c_size_t])
            self._wpfm = fn("write_pfm", C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_void_p])
            self._mse = fn("mse", C.c_double, [C.c_int, C.c_int, C.c_void_p, C.c_void_p])
            self._slope = fn("fit_slope", C.c_double, [C.c_size_t, C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, _ip])
            self._faux = fn("film_aux", None, [C.c_int, C.c_int] + [C.c_void_p] * 4 + [C.c_double, C.c_double] +
                            [C.c_void_p] * 5)
            self._render_ex = fn("render_ex", C.c_int, [C.c_void_p, C.c_int, _dp, C.c_double, C.c_int, C.c_int,
                                                        C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint64, C.c_double,
                                                        C.c_int, C.c_int, C.c_double, C.c_int, C.c_double, C.c_int,
                                                        C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p])
            self._sparse = fn("scene_parse", C.c_void_p, [C.c_char_p, C.c_char_p, C.c_size_t])
            self._sexport = fn("scene_export", None, [C.c_void_p] + [C.c_void_p] * 10)
            self._trace = fn("trace_photons", C.c_size_t, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint32,
                                                           C.c_uint32, C.c_uint32, C.c_int, C.c_double,
                                                           C.c_double, C.c_int, C.c_size_t] + [C.c_void_p] * 7)

    # ---------------------------------------------------------- scalars
    def _call(self, f, *a):
        err = C.c_int(0)
        v = f(*a, C.byref(err))
        _raise(err.value)
        return v

    def sector_index(self, u, v, r, na, ns):
        return self._call(self._sector, u, v, r, na, ns)

    def schedule_radius(self, base, alpha, i):
        return self._sched(base, alpha, i)

    def f_quantile(self, p, d1, d2):
        return self._call(self._fq, p, d1, d2)

    def chi2_quantile(self, p, df):
        return self._call(self._cq, p, df)

    def f_cdf(self, x, d1, d2):
        return self._call(self._fcdf, x, d1, d2)

    def chi2_cdf(self, x, df):
        return self._call(self._ccdf, x, df)

    def reg_inc_beta(self, a, b, x):
        return self._call(self._ib, a, b, x)

    def reg_lower_gamma(self, a, x):
        return self._call(self._lg, a, x)

    def mis_weight_merge(self, n_vm, beta, r, e_vcm, e_vm, l_vcm, l_vm, fwd, rev):
        return self._mwm(n_vm, beta, r, e_vcm, e_vm, l_vcm, l_vm, fwd, rev)

    def f_statistic(self, count, s, q, m):
        s = np.ascontiguousarray(s, np.float64)
        q = np.ascontiguousarray(q, np.float64)
        c = np.ascontiguousarray(count if count is not None else np.zeros(len(s)), np.uint64)
        return self._call(self._fs, _ptr(c, _u64p), _ptr(s, _dp), _ptr(q, _dp), len(s), m)

    def chi2_statistic(self, counts):
        c = np.ascontiguousarray(counts, np.uint64)
        return self._call(self._c2s, _ptr(c, _u64p), len(c))

    def build_frame(self, n):
        n = np.ascontiguousarray(n, np.float64)
        u = np.zeros(3); v = np.zeros(3)
        self._frame(_ptr(n, _dp), _ptr(u, _dp), _ptr(v, _dp))
        return u, v

    # ---------------------------------------------------------- grid
    def grid_build(self, pos, cell):
        pos = np.ascontiguousarray(pos, np.float64).reshape(-1, 3)
        err = C.c_int(0)
        h = self._gb(_ptr(pos, _dp), len(pos), cell, C.byref(err))
        _raise(err.value)
        return _Grid(self, h, len(pos))

    # ---------------------------------------------------------- session
    def session(self, cfg: dict, hit):
        return _Session(self, cfg, hit)

    # ---------------------------------------------------------- generators (port only)
    def c5(self, seed, H):
        if self.kind != "port":
            raise NotImplementedError("the C5 generator is part of the C restatement")
        return _C5(self, seed, H)

    # ---- formats and film outputs (reference build only; tests/test_formats.py)
    def serialize_scene(self, text: str) -> str:
        n = self._ser(text.encode(), None, 0)
        if n < 0:
            raise OracleError("reference parse_scene failed")
        buf = C.create_string_buffer(n + 1)
        self._ser(text.encode(), buf, n + 1)
        return buf.value.decode()

    def write_convergence_csv(self, path, rows):
        it = np.ascontiguousarray([r[0] for r in rows], np.uint64)
        cols = [np.ascontiguousarray([r[k] for r in rows], np.float64) for k in range(1, 5)]
        if self._wcsv(path.encode(), len(rows), it.ctypes.data, *[c.ctypes.data for c in cols]):
            raise OracleError("reference write_convergence_csv failed")

    def read_convergence_csv(self, path, cap=4096):
        it = np.zeros(cap, np.uint64)
        cols = [np.zeros(cap) for _ in range(4)]
        err = C.create_string_buffer(512)
        n = self._rcsv(path.encode(), cap, it.ctypes.data, *[c.ctypes.data for c in cols], err, 512)
        if n < 0:
            raise OracleError(err.value.decode())
        return [(int(it[i]), *[float(c[i]) for c in cols]) for i in range(n)]

    def write_pfm(self, path, img):
        a = np.ascontiguousarray(img, np.float64)
        if self._wpfm(path.encode(), a.shape[1], a.shape[0], a.ctypes.data):
            raise OracleError("reference write_pfm failed")

    def mse(self, a, b):
        a, b = np.ascontiguousarray(a, np.float64), np.ascontiguousarray(b, np.float64)
        return self._mse(a.shape[1], a.shape[0], a.ctypes.data, b.ctypes.data)

    def fit_convergence_slope(self, its, m, lo, hi):
        its, m = np.ascontiguousarray(its, np.uint64), np.ascontiguousarray(m, np.float64)
        err = C.c_int(0)
        v = self._slope(len(its), its.ctypes.data, m.ctypes.data, lo, hi, C.byref(err))
        if err.value:
            raise OracleError("fit_convergence_slope")
        return v

    def film_aux(self, mean, vc, vm, radius, r_min, r_1, ref_img):
        h, w = mean.shape[:2]
        args = [np.ascontiguousarray(x, np.float64) for x in (mean, vc, vm, radius)]
        ref_img = np.ascontiguousarray(ref_img, np.float64)
        outs = [np.zeros((h, w, 3)) for _ in range(4)]
        self._faux(w, h, *[a.ctypes.data for a in args], r_min, r_1, ref_img.ctypes.data, *[o.ctypes.data for o in outs])
        return outs

    def parse_scene_error(self, text: str):
        """The reference parser's ParseError message for `text` ('' when it
        parses).  Runs in a child interpreter that loads only ctypes: in a
        process that has imported numpy, a ParseError unwinding out of
        parse_scene crashes (reproduced only under Python + numpy; C++ hosts
        catch it normally)."""
        import subprocess
        import sys
        code = ("import ctypes as C, sys\n"
                f"L = C.CDLL({LIB_REF!r})\n"
                "f = L.ref_scene_parse; f.restype = C.c_void_p\n"
                "f.argtypes = [C.c_char_p, C.c_char_p, C.c_size_t]\n"
                "b = C.create_string_buffer(1024)\n"
                "h = f(sys.stdin.buffer.read(), b, 1024)\n"
                "sys.stdout.write('' if h else b.value.decode())\n")
        r = subprocess.run([sys.executable, "-c", code], input=text.encode(), capture_output=True, check=True)
        return r.stdout.decode()

    def parse_scene(self, text: str):
        """The reference's parse_scene: (arrays, camera 12-vector or None), or
        raises OracleError with the reference's ParseError message."""
        msg = self.parse_scene_error(text)
        if msg:
            raise OracleError(msg)
        err = C.create_string_buffer(512)
        h = self._sparse(text.encode(), err, 512)
        if not h:
            raise OracleError(err.value.decode())
        sc = _Scene.__new__(_Scene)
        sc.o, sc.h, sc.a = self, h, None
        cnt = np.zeros(4, np.int32)
        self._sexport(h, cnt.ctypes.data, *([None] * 9))
        nm, npr, ne, hc = (int(x) for x in cnt)
        a = dict(material_kind=np.zeros(nm, np.int32), material_rgb=np.zeros((nm, 3)), material_ior=np.zeros(nm),
                 shape_kind=np.zeros(npr, np.int32), shape=np.zeros((npr, 9)), shape_material=np.zeros(npr, np.int32),
                 emitter_shape=np.zeros(ne, np.int32), emitter_radiance=np.zeros((ne, 3)))
        cam = np.zeros(12)
        self._sexport(h, cnt.ctypes.data, *[a[k].ctypes.data for k in (
            "material_kind", "material_rgb", "material_ior", "shape_kind", "shape", "shape_material",
            "emitter_shape", "emitter_radiance")], cam.ctypes.data)
        return a, (cam if hc else None)

    def scene(self, arrays: dict):
        if self.kind != "reference":
            raise NotImplementedError("photon tracing is checked against the reference build only")
        return _Scene(self, arrays)

    def gen_photons(self, workload, seed, iteration, begin, count):
        pos = np.zeros((count, 3), np.float32); nrm = np.zeros((count, 3), np.float32)
        wi = np.zeros((count, 3), np.float32); pw = np.zeros((count, 3), np.float32)
        depth = np.zeros(count, np.uint32)
        self._gen(workload, seed, iteration, begin, count, _ptr(pos, _fp), _ptr(nrm, _fp),
                  _ptr(wi, _fp), _ptr(pw, _fp), _ptr(depth, _u32p))
        return dict(pos=pos, nrm=nrm, wi=wi, pow=pw, depth=depth)

    def gen_raster_hitpoints(self, W):
        H = W * W
        a = {k: np.zeros((H, 3), np.float64) for k in ("pos", "nrm", "wo", "thr", "alb")}
        a["eye_depth"] = np.zeros(H, np.uint32)
        self._ghp(W, *[_ptr(a[k], _dp) for k in ("pos", "nrm", "wo", "thr", "alb")],
                  _ptr(a["eye_depth"], _u32p))
        return a


class _C5:
    """C5 workload generator (oracle restatement of generate.cu's C5 kernels)."""

    def __init__(self, o, seed, H):
        self.o, self.seed, self.H = o, seed, H
        self.h = o._c5c(seed, H)

    def __del__(self):
        if getattr(self, "h", None):
            self.o._c5f(self.h)
            self.h = None

    def hitpoints(self, h0=0, n=None):
        n = self.H - h0 if n is None else n
        out = dict(pos=np.zeros((n, 3)), nrm=np.zeros((n, 3)), wo=np.zeros((n, 3)), thr=np.zeros((n, 3)),
                   alb=np.zeros((n, 3)), eye_depth=np.zeros(n, np.uint32))
        self.o._c5h(self.h, h0, n, *[out[k].ctypes.data for k in ("pos", "nrm", "wo", "thr", "alb", "eye_depth")])
        out["gathered"] = np.ones(n, np.uint8)
        return out

    def photons(self, iteration, begin, count):
        out = dict(pos=np.zeros((count, 3), np.float32), nrm=np.zeros((count, 3), np.float32),
                   wi=np.zeros((count, 3), np.float32), pow=np.zeros((count, 3), np.float32),
                   depth=np.zeros(count, np.uint32))
        self.o._c5p(self.h, iteration, begin, count,
                    *[out[k].ctypes.data for k in ("pos", "nrm", "wi", "pow", "depth")])
        return out


class _Scene:
    """The reference's own Scene + build_accel + trace_light_subpath (oracle/_ref)."""

    def __init__(self, o, arrays):
        self.o = o
        a = self.a = {k: np.ascontiguousarray(v) for k, v in arrays.items()}
        self.h = o._scn(len(a["material_kind"]), a["material_kind"].ctypes.data, a["material_rgb"].ctypes.data,
                        a["material_ior"].ctypes.data, len(a["shape_kind"]), a["shape_kind"].ctypes.data,
                        a["shape"].ctypes.data, a["shape_material"].ctypes.data, len(a["emitter_shape"]),
                        a["emitter_shape"].ctypes.data, a["emitter_radiance"].ctypes.data)

    def __del__(self):
        if getattr(self, "h", None):
            self.o._scnf(self.h)
            self.h = None

    def trace(self, seed, iteration, n_paths, max_depth, n_vm=0, beta=1.0, eta_vm=0.0, threads=0, begin=0):
        """light_phase's flattened vertices (fp64) for paths [begin, begin + n_paths)."""
        end = begin + n_paths
        n = self.o._trace(self.h, seed, iteration, begin, end, max_depth, n_vm, beta, eta_vm, threads, 0,
                          *([None] * 7))
        out = dict(pos=np.zeros((n, 3)), nrm=np.zeros((n, 3)), wi=np.zeros((n, 3)), pow=np.zeros((n, 3)),
                   depth=np.zeros(n, np.uint32), path=np.zeros(n, np.uint32), mis=np.zeros((n, 3)))
        self.o._trace(self.h, seed, iteration, begin, end, max_depth, n_vm, beta, eta_vm, threads, n,
                      *[out[k].ctypes.data for k in ("pos", "nrm", "wi", "pow", "depth", "path", "mis")])
        return out


def _cam9(cam):
    return np.ascontiguousarray(np.concatenate([cam.position, cam.look_at, cam.up]).astype(np.float64))


def _scene_eye(self, cam, seed, iteration, max_depth):
    """pixel_pm's camera walk per pixel (hit points + emitted radiance)."""
    n = cam.width * cam.height
    out = dict(pos=np.zeros((n, 3)), nrm=np.zeros((n, 3)), wo=np.zeros((n, 3)), thr=np.zeros((n, 3)),
               alb=np.zeros((n, 3)), eye_depth=np.zeros(n, np.uint32), gathered=np.zeros(n, np.uint8),
               emitted=np.zeros((n, 3)))
    c9 = _cam9(cam)
    self.o._eye(self.h, c9.ctypes.data_as(_dp), cam.vfov_deg, cam.width, cam.height, seed, iteration, max_depth,
                *[out[k].ctypes.data for k in ("pos", "nrm", "wo", "thr", "alb", "eye_depth", "gathered",
                                                "emitted")])
    return out


def _scene_render(self, cam, seed, iterations, max_depth, light_paths, r0_frac=0.002, n_annuli=2, n_sectors=6,
                  alpha_f=0.01, threads=0, algorithm="fppm"):
    """The reference's render() with Algorithm::fppm (or vcm_plus): (film mean,
    last radii, seconds)."""
    n = cam.width * cam.height
    film = np.zeros((n, 3))
    radius = np.zeros(n)
    secs = C.c_double()
    c9 = _cam9(cam)
    fn = {"fppm": self.o._render, "vcm_plus": self.o._render_vcm}[algorithm]
    rc = fn(self.h, c9.ctypes.data_as(_dp), cam.vfov_deg, cam.width, cam.height, seed, iterations,
                        max_depth, light_paths, r0_frac, n_annuli, n_sectors, alpha_f, threads,
                        film.ctypes.data, radius.ctypes.data, C.byref(secs))
    if rc:
        raise OracleError("reference render failed")
    return film, radius, secs.value


def _scene_render_ex(self, cam, algorithm, seed, iterations, max_depth, light_paths, r0_frac=0.002, n_annuli=2,
                     n_sectors=6, alpha_f=0.01, override="none", r_min_base=0.0, threads=0):
    """render() for fppm / vcm_plus / sppm / vcm / cppm with a test override:
    (film mean [npix][3], last radii, vc totals, vm totals)."""
    n = cam.width * cam.height
    film, radius, vc, vm = np.zeros((n, 3)), np.zeros(n), np.zeros(n), np.zeros(n)
    algo = {"fppm": 0, "vcm_plus": 1, "sppm": 2, "vcm": 3, "cppm": 4}[algorithm]
    ov = {"none": 0, "always_reject": 1, "never_reject": 2}[override]
    c9 = _cam9(cam)
    rc = self.o._render_ex(self.h, algo, c9.ctypes.data_as(_dp), cam.vfov_deg, cam.width, cam.height, seed,
                           iterations, max_depth, light_paths, r0_frac, n_annuli, n_sectors, alpha_f, ov,
                           r_min_base, threads, film.ctypes.data, radius.ctypes.data, vc.ctypes.data, vm.ctypes.data)
    if rc:
        raise OracleError("reference render failed")
    return film, radius, vc, vm


_Scene.render_ex = _scene_render_ex
_Scene.eye_pass = _scene_eye
_Scene.render_fppm = _scene_render
_Scene.render_vcm_plus = lambda self, *a, **k: _scene_render(self, *a, algorithm="vcm_plus", **k)
_Scene.bounding_radius = lambda self: self.o._brad(self.h)


class _Grid:
    def __init__(self, o, h, n):
        self.o, self.h, self.n = o, h, n

    def __del__(self):
        if getattr(self, "h", None):
            self.o._gf(self.h)
            self.h = None

    def export(self):
        nc = self.o._gc(self.h)
        keys = np.zeros(nc, np.uint64); b = np.zeros(nc, np.uint32)
        e = np.zeros(nc, np.uint32); order = np.zeros(self.n, np.uint32)
        self.o._ge(self.h, _ptr(keys, _u64p), _ptr(b, _u32p), _ptr(e, _u32p), _ptr(order, _u32p))
        return keys, b, e, order

    def query_ball(self, c, r):
        c = np.ascontiguousarray(c, np.float64)
        cap = max(self.n, 1)
        out = np.zeros(cap, np.uint32)
        err = C.c_int(0)
        k = self.o._gq(self.h, _ptr(c, _dp), r, _ptr(out, _u32p), cap, C.byref(err))
        _raise(err.value)
        return out[:k].copy()


OUT_FIELDS = ("radius", "gather_r", "t", "tested", "rejected", "statistic",
              "critical", "flux", "radiance", "accepted", "stat_count",
              "stat_sum", "stat_sum_sq")


class _Session:
    def __init__(self, o, cfg, hit):
        self.o = o
        c = Config()
        defaults = dict(n_annuli=2, n_sectors=6, alpha_f=0.01, channels=1,
                        override_decision=0, k=0.7, alpha=0.75, r_min_base=0.0,
                        initial_radius=0.02, samples_per_iteration=1, max_depth=10,
                        normal_guard_cos=0.86602540378443865, threads=1, alpha_chi2=0.01,
                        policy=0, vcm_plus=0, mis_n_vm=0, mis_beta=1.0)
        defaults.update(cfg)
        for k_, v in defaults.items():
            setattr(c, k_, v)
        self.cfg = c
        self.G = c.n_annuli * c.n_sectors
        self.C = c.channels
        self.H = len(hit["pos"])
        self._keep = {k: np.ascontiguousarray(hit[k], np.float64) for k in ("pos", "nrm", "wo", "thr", "alb")}
        self._keep["eye_depth"] = np.ascontiguousarray(hit["eye_depth"], np.uint32)
        g = hit.get("gathered")
        self._keep["gathered"] = None if g is None else np.ascontiguousarray(g, np.uint8)
        err = C.c_int(0)
        kp = self._keep
        self.h = o._sc(C.byref(c), self.H, *[_ptr(kp[k], _dp) for k in ("pos", "nrm", "wo", "thr", "alb")],
                       _ptr(kp["eye_depth"], _u32p), _ptr(kp["gathered"], _u8p), C.byref(err))
        _raise(err.value)

    def __del__(self):
        if getattr(self, "h", None):
            self.o._sf(self.h)
            self.h = None

    def max_radius(self):
        return self.o._smr(self.h)

    def set_hitpoints(self, hit):
        """move_to for every region (new eye-pass hit points; state kept)."""
        kp = {k: np.ascontiguousarray(hit[k], np.float64) for k in ("pos", "nrm", "wo", "thr", "alb")}
        kp["eye_depth"] = np.ascontiguousarray(hit["eye_depth"], np.uint32)
        g = hit.get("gathered")
        kp["gathered"] = None if g is None else np.ascontiguousarray(g, np.uint8)
        assert len(kp["pos"]) == self.H
        self._keep = kp
        self.o._shp(self.h, *[_ptr(kp[k], _dp) for k in ("pos", "nrm", "wo", "thr", "alb")],
                    _ptr(kp["eye_depth"], _u32p), _ptr(kp["gathered"], _u8p))

    def set_eye_mis(self, d_vcm, d_vm):
        """VCM+: eye-vertex MIS partials per hit point."""
        self._eye = [np.ascontiguousarray(d_vcm, np.float64), np.ascontiguousarray(d_vm, np.float64)]
        self.o._seye(self.h, *[_ptr(a, _dp) for a in self._eye])

    def set_photon_mis(self, d_vcm, d_vm, cont):
        """VCM+: light-vertex MIS partials + survival per photon (used by the
        next iterate; arrays are kept alive here)."""
        self._pm = [np.ascontiguousarray(a, np.float64) for a in (d_vcm, d_vm, cont)]
        self.o._sphm(self.h, *[_ptr(a, _dp) for a in self._pm], len(self._pm[0]))

    def iterate(self, iteration, ph, cell=0.0, subset=None):
        n = self.H if subset is None else len(subset)
        CG = self.G * self.C
        out = dict(radius=np.zeros(n), gather_r=np.zeros(n), t=np.zeros(n, np.uint64),
                   tested=np.zeros(n, np.uint8), rejected=np.zeros(n, np.uint8),
                   statistic=np.zeros(n), critical=np.zeros(n), flux=np.zeros((n, 3)),
                   radiance=np.zeros((n, 3)), accepted=np.zeros(n, np.uint64),
                   stat_count=np.zeros((n, CG), np.uint64), stat_sum=np.zeros((n, CG)),
                   stat_sum_sq=np.zeros((n, CG)))
        io = IterOut()
        for k in OUT_FIELDS:
            t = IterOut._fields_[[f[0] for f in IterOut._fields_].index(k)][1]
            setattr(io, k, _ptr(out[k], t))
        # fp64: the reference tracer's own LightVertex values (reference build only)
        f64 = ph["pos"].dtype == np.float64 and self.o.kind != "port"
        ft, pt = (np.float64, _dp) if f64 else (np.float32, _fp)
        arrs = [np.ascontiguousarray(ph[k], ft) for k in ("pos", "nrm", "wi", "pow")]
        depth = np.ascontiguousarray(ph["depth"], np.uint32)
        sub = None if subset is None else np.ascontiguousarray(subset, np.uint32)
        N = len(depth)
        args = [self.h, iteration, *[_ptr(a, pt) for a in arrs], _ptr(depth, _u32p), N,
                float(cell), _ptr(sub, _u32p), 0 if sub is None else len(sub), C.byref(io)]
        if self.o.kind == "port":
            rc = self.o._si(*args)
            times = None
        else:
            gs, ts = C.c_double(0), C.c_double(0)
            rc = (self.o._si64 if f64 else self.o._si)(*args, C.byref(gs), C.byref(ts))
            times = (gs.value, ts.value)
        _raise(rc)
        out["times"] = times
        return out
