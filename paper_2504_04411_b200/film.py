"""Film outputs and convergence files of the reference (proj/core/src/film.cpp),
on the host: the device accumulates the film sum and the per-pixel vc / vm
luminance splits (fppm_gpu_film_mean / fppm_gpu_film_splits); these helpers
turn them into the reference's auxiliary images and files with the same
arithmetic (fp64, same operation order) and the same error messages.

Images are numpy arrays [height, width, 3] (fp64), row 0 at the top, the
layout of Image::at(x, y).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Iterable, List, Sequence

import numpy as np

CSV_HEADER = "iteration,seconds,mse,mean_radius,vm_share"


def _gray(v: np.ndarray) -> np.ndarray:
    return np.repeat(np.asarray(v, np.float64)[..., None], 3, axis=-1)


def radius_image(radius, r_min: float, r_1: float) -> np.ndarray:
    """Film::radius_image (film.cpp:52-61): r_min -> 0, r_1 -> 1, linear."""
    r = np.asarray(radius, np.float64)
    span = r_1 - r_min
    return _gray((r - r_min) / span if span > 0 else np.zeros_like(r))


def vc_share_image(vc, vm) -> np.ndarray:
    """Film::vc_share_image (film.cpp:63-71): connection share of each pixel."""
    vc, vm = np.asarray(vc, np.float64), np.asarray(vm, np.float64)
    total = vc + vm
    with np.errstate(invalid="ignore", divide="ignore"):
        return _gray(np.where(total > 0, vc / np.where(total > 0, total, 1.0), 0.0))


def vm_share_image(vc, vm) -> np.ndarray:
    """Film::vm_share_image (film.cpp:73-81): merge share of each pixel."""
    vc, vm = np.asarray(vc, np.float64), np.asarray(vm, np.float64)
    total = vc + vm
    with np.errstate(invalid="ignore", divide="ignore"):
        return _gray(np.where(total > 0, vm / np.where(total > 0, total, 1.0), 0.0))


def squared_error_image(mean, reference) -> np.ndarray:
    """Film::squared_error_image (film.cpp:83-93)."""
    a, b = np.asarray(mean, np.float64), np.asarray(reference, np.float64)
    if a.shape != b.shape:
        raise ValueError("squared_error_image: size mismatch")
    d = a - b
    return d * d


def mse(a, b) -> float:
    """mse (film.cpp:156-166): 255^2 * mean over pixels and channels of the
    squared difference, summed in pixel order r + g + b."""
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    if a.shape != b.shape:
        raise ValueError("mse: image size mismatch")
    d = (a - b).reshape(-1, 3)
    s = 0.0
    for r, g, bb in d:  # sequential, as the reference
        s += r * r + g * g + bb * bb
    return 255.0 * 255.0 * s / (3.0 * float(len(d)))


def fit_convergence_slope(iterations: Sequence[int], mse_values: Sequence[float], lo: int, hi: int) -> float:
    """fit_convergence_slope (film.cpp:168-185): least-squares slope of
    log(mse) over log(iteration) for iterations in [lo, hi]."""
    if len(iterations) != len(mse_values):
        raise ValueError("fit_convergence_slope: size mismatch")
    sx = sy = sxx = sxy = 0.0
    n = 0
    for it, m in zip(iterations, mse_values):
        if it < lo or it > hi:
            continue
        if not (m > 0) or not math.isfinite(m):
            continue
        x, y = math.log(float(it)), math.log(m)
        sx += x
        sy += y
        sxx += x * x
        sxy += x * y
        n += 1
    if n < 2:
        raise ValueError("fit_convergence_slope: fewer than 2 usable points")
    denom = float(n) * sxx - sx * sx
    return (float(n) * sxy - sx * sy) / denom


@dataclass
class ConvergenceRow:
    """film.hpp:83-89."""
    iteration: int = 0
    seconds: float = 0.0
    mse: float = 0.0
    mean_radius: float = 0.0
    vm_share: float = 0.0


def _g9(x: float) -> str:
    return "%.9g" % x


def write_convergence_csv(path: str, rows: Iterable[ConvergenceRow]) -> None:
    """write_convergence_csv (film.cpp:187-200), byte for byte."""
    try:
        f = open(path, "w", newline="\n")
    except OSError:
        raise RuntimeError("cannot open for writing: " + path)
    with f:
        f.write(CSV_HEADER + "\n")
        for r in rows:
            f.write(f"{int(r.iteration)},{_g9(r.seconds)},{_g9(r.mse)},{_g9(r.mean_radius)},{_g9(r.vm_share)}\n")


def read_convergence_csv(path: str) -> List[ConvergenceRow]:
    """read_convergence_csv (film.cpp:202-226)."""
    try:
        f = open(path)
    except OSError:
        raise RuntimeError("cannot open for reading: " + path)
    with f:
        lines = f.read().split("\n")
    if not lines or lines[0] != CSV_HEADER:
        raise RuntimeError(path + ": unexpected CSV header")
    out = []
    for line in lines[1:]:
        if not line:
            continue
        parts = line.split(",")
        try:
            if len(parts) < 5:
                raise ValueError
            out.append(ConvergenceRow(int(parts[0]), float(parts[1]), float(parts[2]), float(parts[3]),
                                      float(parts[4])))
        except ValueError:
            raise RuntimeError(path + ": bad CSV row '" + line + "'")
    return out


def write_pfm(path: str, image) -> None:
    """write_pfm (film.cpp:95-115): 'PF', width height, -1.0 (little endian),
    rows from the bottom of the image up, RGB fp32."""
    img = np.asarray(image, dtype=np.float64)
    h, w = img.shape[:2]
    try:
        f = open(path, "wb")
    except OSError:
        raise RuntimeError("cannot open for writing: " + path)
    with f:
        f.write(f"PF\n{w} {h}\n-1.0\n".encode())
        f.write(img[::-1].astype("<f4").tobytes())


def read_pfm(path: str) -> np.ndarray:
    """read_pfm (film.cpp:117-154), with the reference's error messages."""
    try:
        f = open(path, "rb")
    except OSError:
        raise RuntimeError("cannot open for reading: " + path)
    with f:
        magic = f.readline().rstrip(b"\n").decode("latin-1")
        if magic != "PF":
            raise RuntimeError(f"{path}: not a color PFM (header '{magic}')")
        dims = f.readline().rstrip(b"\n").decode("latin-1")
        try:
            w, h = (int(x) for x in dims.split()[:2])
            if w <= 0 or h <= 0:
                raise ValueError
        except ValueError:
            raise RuntimeError(f"{path}: bad PFM dimensions '{dims}'")
        scale_line = f.readline().decode("latin-1")
        try:
            scale = float(scale_line.split()[0]) if scale_line.split() else 0.0
        except ValueError:
            scale = 0.0
        if scale >= 0:
            raise RuntimeError(f"{path}: big-endian PFM not supported")
        data = f.read(w * h * 12)
        if len(data) < w * h * 12:
            raise RuntimeError(f"{path}: truncated PFM payload")
    return np.frombuffer(data, dtype="<f4").reshape(h, w, 3)[::-1].astype(np.float64)
