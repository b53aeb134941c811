"""Analytic scenes for the light phase (fppm_scene, include/fppm_gpu.h).

Mirrors the subset of the reference's Scene (proj/core/include/fppm/scene.hpp:
16-103) the photon tracer supports: spheres and quads, Lambertian / mirror /
dielectric materials and area emitters attached to primitives.  Scenes are
plain host arrays; FppmContext.set_scene uploads them once.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

LAMBERTIAN, MIRROR, DIELECTRIC = 0, 1, 2
SPHERE, QUAD = 0, 1


@dataclass
class Scene:
    material_kind: list = field(default_factory=list)
    material_rgb: list = field(default_factory=list)
    material_ior: list = field(default_factory=list)
    shape_kind: list = field(default_factory=list)
    shape: list = field(default_factory=list)
    shape_material: list = field(default_factory=list)
    emitter_shape: list = field(default_factory=list)
    emitter_radiance: list = field(default_factory=list)
    material_name: list = field(default_factory=list)

    # ---- construction (scene_parse.cpp's material / sphere / quad / emit)
    def material(self, kind: int, rgb=(1.0, 1.0, 1.0), ior: float = 1.5, name: str = "") -> int:
        if kind not in (LAMBERTIAN, MIRROR, DIELECTRIC):
            raise ValueError(f"unsupported material kind {kind}")
        if kind == DIELECTRIC and not ior > 1.0:
            raise ValueError("ior must exceed 1")
        self.material_name.append(name or f"m{len(self.material_kind)}")
        self.material_kind.append(kind)
        self.material_rgb.append([float(x) for x in rgb])
        self.material_ior.append(float(ior))
        return len(self.material_kind) - 1

    def sphere(self, center, radius: float, material: int) -> int:
        if not radius > 0.0:
            raise ValueError("sphere radius must be positive")
        self.shape_kind.append(SPHERE)
        self.shape.append([*map(float, center), float(radius), 0.0, 0.0, 0.0, 0.0, 0.0])
        self.shape_material.append(material)
        return len(self.shape_kind) - 1

    def quad(self, corner, e1, e2, material: int, emit=None) -> int:
        self.shape_kind.append(QUAD)
        self.shape.append([*map(float, corner), *map(float, e1), *map(float, e2)])
        self.shape_material.append(material)
        idx = len(self.shape_kind) - 1
        if emit is not None:
            self.emitter_shape.append(idx)
            self.emitter_radiance.append([float(x) for x in emit])
        return idx

    def arrays(self) -> dict:
        return dict(
            material_kind=np.asarray(self.material_kind, np.int32),
            material_rgb=np.asarray(self.material_rgb, np.float64).reshape(-1, 3),
            material_ior=np.asarray(self.material_ior, np.float64),
            shape_kind=np.asarray(self.shape_kind, np.int32),
            shape=np.asarray(self.shape, np.float64).reshape(-1, 9),
            shape_material=np.asarray(self.shape_material, np.int32),
            emitter_shape=np.asarray(self.emitter_shape, np.int32),
            emitter_radiance=np.asarray(self.emitter_radiance, np.float64).reshape(-1, 3),
        )


def schedule_radius_host(base: float, alpha: float, i: int) -> float:
    """schedule_radius (gather.cpp:11-13) through the library's host table
    function (glibc pow, like the reference build)."""
    from .api import schedule_radius
    return schedule_radius(base, alpha, i)


def is_chromatic(c) -> bool:
    """integrator.cpp:77."""
    return c[0] != c[1] or c[1] != c[2]


def has_chromatic_emitter(scene: Scene) -> bool:
    """integrator.cpp:79-91 for the area emitters the device supports: the
    Renderer resolves TestChannels::auto_detect to rgb when this holds
    (integrator.cpp:128-130)."""
    return any(is_chromatic(r) for r in scene.emitter_radiance)


def _g17(x: float) -> str:
    return "%.17g" % float(x)


def _v3(v) -> str:
    return "(" + ",".join(_g17(x) for x in v) + ")"


def serialize_scene(scene: Scene, camera=None) -> str:
    """serialize_scene (scene_parse.cpp:441-548): the reference's text form,
    numbers printed %.17g, one line per camera / material / primitive (with
    its emitter inline), so parse_scene(serialize_scene(s)) rebuilds s."""
    out = []
    if camera is not None:
        out.append(f"camera pos={_v3(camera.position)} look={_v3(camera.look_at)} up={_v3(camera.up)} "
                   f"fov={_g17(camera.vfov_deg)} res={int(camera.width)}x{int(camera.height)}\n")
    names = scene.material_name or [f"m{i}" for i in range(len(scene.material_kind))]
    for name, kind, rgb, ior in zip(names, scene.material_kind, scene.material_rgb, scene.material_ior):
        if kind == LAMBERTIAN:
            out.append(f"material {name} lambertian albedo={_v3(rgb)}\n")
        elif kind == MIRROR:
            out.append(f"material {name} mirror refl={_v3(rgb)}\n")
        else:
            out.append(f"material {name} dielectric ior={_g17(ior)} tint={_v3(rgb)}\n")
    emit = dict(zip(scene.emitter_shape, scene.emitter_radiance))
    for i, (kind, sh, m) in enumerate(zip(scene.shape_kind, scene.shape, scene.shape_material)):
        if kind == SPHERE:
            line = f"sphere center={_v3(sh[0:3])} radius={_g17(sh[3])}"
        else:
            line = f"quad corner={_v3(sh[0:3])} e1={_v3(sh[3:6])} e2={_v3(sh[6:9])}"
        line += f" material={names[m]}"
        if i in emit:
            line += f" emit={_v3(emit[i])}"
        out.append(line + "\n")
    return "".join(out)


@dataclass
class Camera:
    """Pinhole camera (Camera, scene.hpp:75-82)."""
    position: tuple = (0.0, 0.0, 0.0)
    look_at: tuple = (0.0, 0.0, -1.0)
    up: tuple = (0.0, 1.0, 0.0)
    vfov_deg: float = 45.0
    width: int = 1
    height: int = 1


def caustic_box_camera(res: int = 1024) -> Camera:
    """BASELINE configs[2]: res x res pinhole at (0.5, 0.5, -1.4), FOV 40
    degrees, looking into the room (+z)."""
    return Camera((0.5, 0.5, -1.4), (0.5, 0.5, 0.0), (0.0, 1.0, 0.0), 40.0, res, res)


def bounding_radius(scene: Scene) -> float:
    """bounding_radius (scene_geometry.cpp:341-362): half the diagonal of the
    box of all non-emitter primitives (all primitives if there are none); the
    reference's initial radius is r0_frac (0.002) times this."""
    emitters = set(scene.emitter_shape)
    lo = np.full(3, np.inf)
    hi = np.full(3, -np.inf)
    for pass_ in range(2):
        any_ = False
        for i, (k, p) in enumerate(zip(scene.shape_kind, scene.shape)):
            if pass_ == 0 and i in emitters:
                continue
            any_ = True
            p = np.asarray(p, np.float64)
            if k == SPHERE:
                pts = [p[:3] - p[3], p[:3] + p[3]]
            else:
                c, e1, e2 = p[:3], p[3:6], p[6:9]
                pts = [c, c + e1, c + e2, c + e1 + e2]
            for q in pts:
                lo = np.minimum(lo, q)
                hi = np.maximum(hi, q)
        if any_:
            break
    d = hi - lo
    return 0.5 * float(np.sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]))


def caustic_box(light_radiance: float = 15.0) -> Scene:
    """BASELINE.json configs[2] / [3]: an axis-aligned unit room of five
    Lambertian walls (albedo 0.75, red/green side pair, open towards the camera
    at z < 0), a glass sphere (IOR 1.5, radius 0.2) at (0.5, 0.2, 0.5) and a
    0.2 x 0.2 area light of radiance 15 just below the ceiling, facing down."""
    s = Scene()
    white = s.material(LAMBERTIAN, (0.75, 0.75, 0.75))
    red = s.material(LAMBERTIAN, (0.75, 0.25, 0.25))
    green = s.material(LAMBERTIAN, (0.25, 0.75, 0.25))
    glass = s.material(DIELECTRIC, (1.0, 1.0, 1.0), 1.5)
    s.quad((0, 0, 0), (0, 0, 1), (1, 0, 0), white)        # floor, normal +y
    s.quad((0, 1, 0), (1, 0, 0), (0, 0, 1), white)        # ceiling, normal -y
    s.quad((0, 0, 1), (1, 0, 0), (0, 1, 0), white)        # back wall, normal -z
    s.quad((0, 0, 0), (0, 1, 0), (0, 0, 1), red)          # left wall, normal +x
    s.quad((1, 0, 0), (0, 0, 1), (0, 1, 0), green)        # right wall, normal -x
    s.sphere((0.5, 0.2, 0.5), 0.2, glass)
    L = light_radiance
    s.quad((0.4, 0.999, 0.4), (0.2, 0, 0), (0, 0, 0.2), white, emit=(L, L, L))  # e1 x e2 = -y
    return s


def mixed_box() -> Scene:
    """Closed box with a chromatic ceiling light, a mirror and a glass sphere:
    every material path of the tracer (delta chains, refraction, total
    internal reflection, roulette) in one scene.  Test fixture."""
    s = Scene()
    white = s.material(LAMBERTIAN, (0.72, 0.72, 0.72))
    red = s.material(LAMBERTIAN, (0.6, 0.1, 0.08))
    green = s.material(LAMBERTIAN, (0.12, 0.5, 0.1))
    chrome = s.material(MIRROR, (0.9, 0.9, 0.9))
    glass = s.material(DIELECTRIC, (0.98, 0.96, 0.94), 1.5)
    s.quad((-1, -1, -1), (0, 0, 2), (2, 0, 0), white)
    s.quad((-1, 1, -1), (2, 0, 0), (0, 0, 2), white)
    s.quad((-1, -1, -1), (2, 0, 0), (0, 2, 0), white)
    s.quad((-1, -1, 1), (0, 2, 0), (2, 0, 0), white)
    s.quad((-1, -1, -1), (0, 2, 0), (0, 0, 2), red)
    s.quad((1, -1, -1), (0, 0, 2), (0, 2, 0), green)
    s.quad((-0.3, 0.99, -0.3), (0.6, 0, 0), (0, 0, 0.6), white, emit=(12.0, 10.0, 7.0))
    s.sphere((-0.42, -0.62, 0.28), 0.33, chrome)
    s.sphere((0.44, -0.64, -0.12), 0.31, glass)
    return s


def two_lights_sphere_emitter() -> Scene:
    """Two emitters (a quad and a sphere light) over a diffuse floor: covers
    the emitter pick and sphere emission (path.cpp:180-195)."""
    s = Scene()
    floor = s.material(LAMBERTIAN, (0.6, 0.6, 0.6))
    wall = s.material(LAMBERTIAN, (0.3, 0.5, 0.7))
    s.quad((-2, 0, -2), (0, 0, 4), (4, 0, 0), floor)
    s.quad((-2, 0, 2), (0, 3, 0), (4, 0, 0), wall)
    s.quad((-0.25, 1.5, -0.25), (0.5, 0, 0), (0, 0, 0.5), floor, emit=(5.0, 5.0, 5.0))
    sid = s.sphere((0.8, 0.6, 0.3), 0.15, floor)
    s.emitter_shape.append(sid)
    s.emitter_radiance.append([3.0, 2.0, 1.0])
    return s


class _SceneStruct(C.Structure):
    _fields_ = [("n_materials", C.c_uint32), ("material_kind", C.c_void_p), ("material_rgb", C.c_void_p),
                ("material_ior", C.c_void_p), ("n_primitives", C.c_uint32), ("shape_kind", C.c_void_p),
                ("shape", C.c_void_p), ("shape_material", C.c_void_p), ("n_emitters", C.c_uint32),
                ("emitter_shape", C.c_void_p), ("emitter_radiance", C.c_void_p)]


def to_struct(scene: Scene):
    """(fppm_scene struct, arrays kept alive by the caller)."""
    a = {k: np.ascontiguousarray(v) for k, v in scene.arrays().items()}
    st = _SceneStruct(len(a["material_kind"]), a["material_kind"].ctypes.data, a["material_rgb"].ctypes.data,
                      a["material_ior"].ctypes.data, len(a["shape_kind"]), a["shape_kind"].ctypes.data,
                      a["shape"].ctypes.data, a["shape_material"].ctypes.data, len(a["emitter_shape"]),
                      a["emitter_shape"].ctypes.data, a["emitter_radiance"].ctypes.data)
    return st, a
