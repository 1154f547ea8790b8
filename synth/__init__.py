"""Seeded synthetic inputs for the butterfly sparse Fourier transform.

This module is shared by the oracle (``oracle/``) and the CUDA path
(``paper_0801_1524_b200``) and by nothing else of the method: it holds
geometry sampling and random numbers only, none of the transform's
arithmetic.

Workloads follow BASELINE.json:7-11 (configs C0..C4); the paper's own
geometries ("Both X and K are ellipses", P:490-496 sphere
vs. F16/submarine meshes) are not available, so these analytic shapes stand
in for them.

Readings:
  * 2D: ``density`` points per unit arc length of the *scaled* curve N*X,
    equispaced in arc length starting at t=0, n = round(density*perimeter)
    (reading 17).
  * 3D: latitude/longitude rings.  n_r = round(density * meridian length)
    rings at meridian arc length (i+1/2)*L_m/n_r; ring i carries
    round(density * ring circumference) points at phi = 2*pi*(j+1/2)/n_i
    (reading 18).
  * charges f_j: re, im i.i.d. N(0,1) from numpy default_rng(seed), re drawn
    first (reading 14; BASELINE.json overrides the paper's "mean 0",
    P:371-372).
  * error sample: default_rng(1_000_000+seed).choice(n_x, 1024, replace=False)
    (reading 15).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

__all__ = [
    "Workload",
    "CONFIGS",
    "make_workload",
    "sample_ellipse_2d",
    "sample_ellipsoid_3d",
    "random_charges",
    "error_sample",
]


# --------------------------------------------------------------------------
# arc length helpers (geometry only)
# --------------------------------------------------------------------------
def _ellipse_speed(t, a, b):
    return np.sqrt((a * np.sin(t)) ** 2 + (b * np.cos(t)) ** 2)


def _ellipse_arclength_table(a, b, m=1 << 16):
    """Fourier representation of the arc length S(t) of (a cos t, b sin t).

    The speed is smooth and 2*pi periodic, so its FFT coefficients converge
    geometrically; S(t) = c0*t + sum_k (integrated harmonics).  Returns a
    callable S and the total perimeter.
    """
    t = 2.0 * np.pi * np.arange(m) / m
    v = _ellipse_speed(t, a, b)
    c = np.fft.rfft(v) / m
    c0 = c[0].real
    kk = np.arange(1, len(c))
    ck = c[1:]
    keep = np.abs(ck) > 1e-15 * abs(c0)
    kk = kk[keep]
    ck = ck[keep]

    def S(tt):
        tt = np.asarray(tt, dtype=np.float64)
        # integral of 2 Re(c_k e^{ikt}) from 0 to t
        ph = np.outer(tt, kk)
        re = (2.0 * (ck.real[None, :] * np.sin(ph) + ck.imag[None, :] * (np.cos(ph) - 1.0)) / kk[None, :])
        return c0 * tt + re.sum(axis=1)

    return S, 2.0 * np.pi * c0


def _invert_arclength(S, speed, targets, perimeter, chunk=1 << 14):
    """Solve S(t) = s for each s in targets (monotone S) by Newton."""
    out = np.empty_like(targets)
    for i0 in range(0, len(targets), chunk):
        s = targets[i0:i0 + chunk]
        t = 2.0 * np.pi * s / perimeter  # initial guess
        for _ in range(8):
            f = S(t) - s
            t = t - f / speed(t)
        out[i0:i0 + chunk] = t
    return out


# --------------------------------------------------------------------------
# 2D curves
# --------------------------------------------------------------------------
def sample_ellipse_2d(N: int, center, semi, density: float = 4.0) -> np.ndarray:
    """Points on the scaled ellipse N*(cx + a cos t, cy + b sin t), equispaced
    in arc length of the scaled curve at ``density`` points per unit length.

    Returns float64 array [n, 2] (row-major), n = round(density*perimeter).
    """
    cx, cy = center
    a, b = semi
    if a == b:
        perim = 2.0 * math.pi * a * N
        n = max(1, int(round(density * perim)))
        t = 2.0 * np.pi * np.arange(n) / n
    else:
        S, per_unit = _ellipse_arclength_table(a * N, b * N)
        perim = per_unit
        n = max(1, int(round(density * perim)))
        s = np.arange(n) * (perim / n)
        t = _invert_arclength(S, lambda tt: _ellipse_speed(tt, a * N, b * N), s, perim)
    pts = np.empty((n, 2), dtype=np.float64)
    pts[:, 0] = N * cx + (a * N) * np.cos(t)
    pts[:, 1] = N * cy + (b * N) * np.sin(t)
    return np.clip(pts, 0.0, float(N))


# --------------------------------------------------------------------------
# 3D surfaces
# --------------------------------------------------------------------------
def _ellipse_perimeter(a, b):
    if a == b:
        return 2.0 * math.pi * a
    _, per = _ellipse_arclength_table(a, b, m=1 << 12)
    return per


def sample_ellipsoid_3d(N: int, center, semi, density: float = 2.0) -> np.ndarray:
    """Lat-long sampling of the scaled ellipsoid
    N*(c + (a sin(th) cos(ph), b sin(th) sin(ph), c cos(th))).

    Rings are equispaced in arc length along the phi=0 meridian (the (a,c)
    ellipse, th in [0,pi]); ring i carries round(density*circumference_i)
    points at phi = 2 pi (j+1/2)/n_i.  Returns float64 [n, 3].
    """
    cx, cy, cz = center
    a, b, c = (s * N for s in semi)
    # meridian: (a sin th, c cos th), th in [0, pi] = half an ellipse
    if a == c:
        Lm = math.pi * a
        nr = max(1, int(round(density * Lm)))
        th = np.pi * (np.arange(nr) + 0.5) / nr
    else:
        # meridian m(th) = (a sin th, c cos th) has speed sqrt(c^2 sin^2 + a^2 cos^2),
        # which is the speed of the table curve (c cos t, a sin t) at t = th.
        S, per = _ellipse_arclength_table(c, a)
        Lm = per / 2.0
        nr = max(1, int(round(density * Lm)))
        targets = (np.arange(nr) + 0.5) * (Lm / nr)
        th = _invert_arclength(S, lambda tt: _ellipse_speed(tt, c, a), targets, per)
    pts = []
    for thi in th:
        st, ct = math.sin(thi), math.cos(thi)
        circ = _ellipse_perimeter(a * st, b * st)
        ni = max(1, int(round(density * circ)))
        ph = 2.0 * np.pi * (np.arange(ni) + 0.5) / ni
        ring = np.empty((ni, 3), dtype=np.float64)
        ring[:, 0] = N * cx + a * st * np.cos(ph)
        ring[:, 1] = N * cy + b * st * np.sin(ph)
        ring[:, 2] = N * cz + c * ct
        pts.append(ring)
    out = np.concatenate(pts, axis=0)
    return np.clip(out, 0.0, float(N))


# --------------------------------------------------------------------------
# charges / error sample
# --------------------------------------------------------------------------
def random_charges(n: int, seed: int) -> np.ndarray:
    """f_j = re + i im with re, im i.i.d. N(0,1); re drawn first (reading 14)."""
    rng = np.random.default_rng(seed)
    re = rng.standard_normal(n)
    im = rng.standard_normal(n)
    return (re + 1j * im).astype(np.complex128)


def error_sample(n_x: int, seed: int, m: int = 1024) -> np.ndarray:
    """Seeded target subset for the relative L2 error (reading 15)."""
    if n_x <= m:
        return np.arange(n_x, dtype=np.int64)
    rng = np.random.default_rng(1_000_000 + seed)
    return np.sort(rng.choice(n_x, m, replace=False)).astype(np.int64)


# --------------------------------------------------------------------------
# BASELINE.json configs
# --------------------------------------------------------------------------
@dataclasses.dataclass
class Workload:
    name: str
    dim: int
    N: int
    p: int
    seed: int
    x: np.ndarray  # targets  [nx, dim] float64
    k: np.ndarray  # sources  [nk, dim] float64
    f: np.ndarray  # charges  [nk] complex128
    sample: np.ndarray  # error-sample target indices
    all_targets_error: bool

    @property
    def P(self) -> int:
        """Paper's P = max(#targets, #sources)."""
        return max(len(self.x), len(self.k))


CONFIGS = {
    # name: (dim, N, p, seed, X shape, K shape, error on all targets?)
    "C0": (2, 64, 5, 0, ("circle",), ("circle",), True),
    "C1": (2, 1024, 7, 1, ("circle",), ("ellipse",), True),
    "C2": (2, 16384, 9, 2, ("circle",), ("ellipse",), False),
    "C3": (3, 128, 5, 3, ("sphere",), ("ellipsoid",), True),
    "C4": (3, 512, 7, 4, ("sphere",), ("ellipsoid",), False),
}


def _shape_points(kind: str, N: int) -> np.ndarray:
    if kind == "circle":
        return sample_ellipse_2d(N, (0.5, 0.5), (0.4, 0.4), 4.0)
    if kind == "ellipse":
        return sample_ellipse_2d(N, (0.5, 0.5), (0.35, 0.25), 4.0)
    if kind == "sphere":
        return sample_ellipsoid_3d(N, (0.5, 0.5, 0.5), (0.4, 0.4, 0.4), 2.0)
    if kind == "ellipsoid":
        return sample_ellipsoid_3d(N, (0.5, 0.5, 0.5), (0.4, 0.3, 0.25), 2.0)
    raise ValueError(kind)


def make_workload(name: str, N: int | None = None, p: int | None = None) -> Workload:
    """Build config ``name`` (C0..C4); N/p may be overridden for small tests
    (the shapes and densities stay those of the config)."""
    dim, N0, p0, seed, xs, ks, allerr = CONFIGS[name]
    N = N0 if N is None else N
    p = p0 if p is None else p
    x = _shape_points(xs[0], N)
    k = _shape_points(ks[0], N)
    f = random_charges(len(k), seed)
    sample = np.arange(len(x), dtype=np.int64) if allerr else error_sample(len(x), seed)
    return Workload(name, dim, N, p, seed, np.ascontiguousarray(x), np.ascontiguousarray(k), f, sample, allerr)
