"""The reference's on-disk formats for the device path.

* ``parse_scene(text)`` reads the reference's line-oriented scene text
  (scene_parse.cpp:244-440: ``camera``, ``material NAME KIND k=v..``,
  ``sphere``, ``quad``, ``arealight``) into a :class:`scene.Scene` plus a
  :class:`scene.Camera`, with the reference's validation rules and
  ``file:line:col: message`` errors.  Meshes, point / spot lights and Phong
  materials parse but are rejected: the device tracer does not model them.
* ``write_pfm(path, image)`` writes a film the way film.cpp:95-115 does
  (little-endian fp32, bottom row first).
"""
from __future__ import annotations

import math
import re

import numpy as np

from .scene import DIELECTRIC, LAMBERTIAN, MIRROR, Camera, Scene

# std::from_chars(double) general format: optional '-', digits with an
# optional fraction, optional exponent (no leading '+', no hex)
_NUM = re.compile(r"-?(?:(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?|(?i:infinity|inf|nan))")
_IDENT = re.compile(r"[A-Za-z0-9_]+")


class ParseError(ValueError):
    """scene_parse.cpp's ParseError: '<file>:<line>:<col>: <message>'."""


class _Cursor:
    def __init__(self, label, line_no, line):
        self.label, self.line_no, self.line, self.pos = label, line_no, line, 0

    def fail(self, msg):
        raise ParseError(f"{self.label}:{self.line_no}:{self.pos + 1}: {msg}")

    def skip_ws(self):
        while self.pos < len(self.line) and self.line[self.pos] in " \t":
            self.pos += 1

    def at_end(self):
        self.skip_ws()
        return self.pos >= len(self.line) or self.line[self.pos] == "#"

    def ident(self):
        self.skip_ws()
        m = _IDENT.match(self.line, self.pos)
        if not m:
            self.fail("expected an identifier")
        self.pos = m.end()
        return m.group(0)

    def scalar(self):
        self.skip_ws()
        m = _NUM.match(self.line, self.pos)
        if not m:
            self.fail("expected a number")
        v = float(m.group(0))
        if not math.isfinite(v):
            self.fail("number is not finite")
        self.pos = m.end()
        return v

    def expect(self, c):
        self.skip_ws()
        if self.pos >= len(self.line) or self.line[self.pos] != c:
            self.fail(f"expected '{c}'")
        self.pos += 1

    def value(self):
        """('tuple', (x, y, z)) | ('scalar', v, text) | ('string', text)"""
        self.skip_ws()
        if self.pos < len(self.line) and self.line[self.pos] == "(":
            self.pos += 1
            x = self.scalar()
            self.expect(",")
            y = self.scalar()
            self.expect(",")
            z = self.scalar()
            self.expect(")")
            return ("tuple", (x, y, z))
        start = self.pos
        while self.pos < len(self.line) and not self.line[self.pos].isspace():
            self.pos += 1
        if self.pos == start:
            self.fail("expected a value")
        text = self.line[start:self.pos]
        m = _NUM.fullmatch(text)
        if m:
            v = float(text)
            if not math.isfinite(v):
                self.fail("number is not finite")
            return ("scalar", v, text)
        return ("string", text)


class _Kv:
    def __init__(self, cur):
        self.cur, self.kvs = cur, {}
        while not cur.at_end():
            key = cur.ident()
            cur.expect("=")
            val = cur.value()  # read before the duplicate check (the column the reference reports)
            if key in self.kvs:
                cur.fail(f"duplicate key '{key}'")
            self.kvs[key] = val

    def take(self, key):
        if key not in self.kvs:
            self.cur.fail(f"missing key '{key}'")
        return self.kvs.pop(key)

    def opt(self, key):
        return self.kvs.pop(key, None)

    def number(self, key):
        v = self.take(key)
        if v[0] != "scalar":
            self.cur.fail(f"'{key}' must be a number")
        return v[1]

    def tuple(self, key):
        v = self.take(key)
        if v[0] != "tuple":
            self.cur.fail(f"'{key}' must be a (x,y,z) tuple")
        return v[1]

    def string(self, key):
        v = self.take(key)
        if v[0] == "tuple":
            self.cur.fail(f"'{key}' must be a string")
        return v[2] if v[0] == "scalar" else v[1]

    def done(self):
        if self.kvs:
            self.cur.fail(f"unknown key '{sorted(self.kvs)[0]}'")


def _unit(cur, c, what):
    if any(x < 0.0 or x > 1.0 for x in c):
        cur.fail(f"{what} components must be in [0,1]")


def _nonneg(cur, c, what):
    if any(x < 0.0 for x in c):
        cur.fail(f"{what} must be non-negative")


def _cross(a, b):
    return (a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0])


def _len(v):
    return math.sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2])


def parse_scene(text: str, label: str = "<scene>"):
    """(Scene, Camera or None) from the reference's scene text."""
    scene, camera = Scene(), None
    materials, shapes = {}, {}
    counts = {"sphere": 0, "quad": 0, "mesh": 0}
    emits = set()

    def add_shape(kind, idx):
        shapes[f"{kind}{counts[kind]}"] = idx
        counts[kind] += 1

    def attach(cur, idx, radiance):
        if idx in emits:
            name = next(k for k, v in shapes.items() if v == idx)
            cur.fail(f"shape '{name}' already emits")
        emits.add(idx)
        scene.emitter_shape.append(idx)
        scene.emitter_radiance.append(list(radiance))

    for line_no, line in enumerate(text.split("\n"), 1):
        cur = _Cursor(label, line_no, line)
        if cur.at_end():
            continue
        kw = cur.ident()
        if kw == "camera":
            kv = _Kv(cur)
            pos, look, up, fov = kv.tuple("pos"), kv.tuple("look"), kv.tuple("up"), kv.number("fov")
            res = kv.string("res")
            kv.done()
            m = re.match(r"\s*([+-]?\d+)x([+-]?\d+)", res)
            if not m:
                cur.fail("res must look like 640x480")
            w, h = int(m.group(1)), int(m.group(2))
            if w < 1 or h < 1:
                cur.fail("resolution must be at least 1x1")
            if not 0.0 < fov < 180.0:
                cur.fail("fov must be in (0,180)")
            if _len(_cross(tuple(a - b for a, b in zip(look, pos)), up)) == 0.0:
                cur.fail("up is parallel to the view direction")
            camera = Camera(pos, look, up, fov, w, h)
        elif kw == "material":
            name = cur.ident()
            if name in materials:
                cur.fail(f"duplicate material '{name}'")
            kind = cur.ident()
            kv = _Kv(cur)
            if kind == "lambertian":
                c = kv.tuple("albedo")
                _unit(cur, c, "albedo")
                mk, ior = LAMBERTIAN, 1.5
            elif kind == "mirror":
                c = kv.tuple("refl")
                _unit(cur, c, "refl")
                mk, ior = MIRROR, 1.5
            elif kind == "dielectric":
                ior = kv.number("ior")
                if not ior > 1.0:
                    cur.fail("ior must exceed 1")
                t = kv.opt("tint")
                c = (1.0, 1.0, 1.0)
                if t is not None:
                    if t[0] != "tuple":
                        cur.fail("'tint' must be a (x,y,z) tuple")
                    c = t[1]
                    _unit(cur, c, "tint")
                mk = DIELECTRIC
            elif kind == "phong":
                cur.fail("phong materials are not supported by the device tracer")
            else:
                cur.fail(f"unknown material kind '{kind}'")
            kv.done()
            materials[name] = scene.material(mk, c, ior, name=name)
        elif kw in ("sphere", "quad"):
            kv = _Kv(cur)
            if kw == "sphere":
                center, radius = kv.tuple("center"), kv.number("radius")
                if not radius > 0.0:
                    cur.fail("radius must be positive")
            else:
                corner, e1, e2 = kv.tuple("corner"), kv.tuple("e1"), kv.tuple("e2")
                if _len(_cross(e1, e2)) <= 1e-12 * _len(e1) * _len(e2):
                    cur.fail("quad edges are parallel")
            mname = kv.string("material")
            if mname not in materials:
                cur.fail(f"unknown material '{mname}'")
            emit = kv.opt("emit")
            kv.done()
            if kw == "sphere":
                idx = scene.sphere(center, radius, materials[mname])
            else:
                idx = scene.quad(corner, e1, e2, materials[mname])
            add_shape(kw, idx)
            if emit is not None:
                if emit[0] != "tuple":
                    cur.fail("'emit' must be a (x,y,z) tuple")
                _nonneg(cur, emit[1], "emit")
                attach(cur, idx, emit[1])
        elif kw == "arealight":
            kv = _Kv(cur)
            shape, radiance = kv.string("shape"), kv.tuple("radiance")
            kv.done()
            _nonneg(cur, radiance, "radiance")
            if shape not in shapes:
                cur.fail(f"unknown shape '{shape}'")
            attach(cur, shapes[shape], radiance)
        elif kw in ("mesh", "pointlight", "spotlight"):
            cur.fail(f"'{kw}' is not supported by the device tracer (spheres, quads, area lights)")
        else:
            cur.fail(f"unknown keyword '{kw}'")
    return scene, camera


def load_scene(path: str):
    with open(path) as f:
        return parse_scene(f.read(), path)


# PFM film I/O lives in film.py (film.cpp:95-154); kept importable from here
from .film import read_pfm, write_pfm  # noqa: E402,F401
