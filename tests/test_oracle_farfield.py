"""Pins of the oracle's far-field sum (eq. far), independent of
its code: closed forms of the exponential kernel and of the scattering
integrals over a circle / sphere (Jacobi-Anger / Funk-Hecke), evaluated with
scipy's Bessel functions and exact quadratures."""
import numpy as np
import pytest
from scipy.special import j0

import oracle


def _dirs2(n):
    t = 2 * np.pi * (np.arange(n) + 0.25) / n
    return np.stack([np.cos(t), np.sin(t)], 1)


def test_single_source_closed_form():
    """One source y0 with charge F0: u(xhat) = F0 exp(-i kappa xhat.y0) (s = -1)
    and F0 exp(+i kappa xhat.y0) (s = +1)."""
    rng = np.random.default_rng(0)
    xh = _dirs2(37)
    y0 = np.array([[0.31, 0.72]])
    F0 = np.array([0.7 - 1.3j])
    for kappa in (3.0, 250.0):
        for sign in (-1, 1):
            u = oracle.farfield_direct(xh, y0, F0, kappa, sign=sign)
            ref = F0[0] * np.exp(sign * 1j * kappa * (xh @ y0[0]))
            assert np.max(np.abs(u - ref)) <= 1e-13 * kappa
    # y0 = 0 gives sum F for every direction
    y = np.zeros((5, 2))
    F = rng.normal(size=5) + 1j * rng.normal(size=5)
    assert np.allclose(oracle.farfield_direct(xh, y, F, 40.0), F.sum(), rtol=0, atol=1e-14)


def test_circle_jacobi_anger():
    """int over the circle |y - c| = rho of exp(-i kappa xhat.y) ds
    = 2 pi rho J0(kappa rho) exp(-i kappa xhat.c); the trapezoid rule with n
    equal weights is exact to rounding once n exceeds kappa rho by a margin."""
    c, rho, kappa = np.array([0.5, 0.5]), 0.3, 180.0
    n = 400
    t = 2 * np.pi * np.arange(n) / n
    y = c + rho * np.stack([np.cos(t), np.sin(t)], 1)
    F = np.full(n, 2 * np.pi * rho / n, dtype=np.complex128)
    xh = _dirs2(64)
    u = oracle.farfield_direct(xh, y, F, kappa)
    ref = 2 * np.pi * rho * j0(kappa * rho) * np.exp(-1j * kappa * (xh @ c))
    assert np.max(np.abs(u - ref)) <= 1e-12 * 2 * np.pi * rho


def test_sphere_funk_hecke():
    """int over the sphere |y - c| = rho of exp(-i kappa xhat.y) dS
    = 4 pi rho^2 sin(kappa rho)/(kappa rho) exp(-i kappa xhat.c), with a
    Gauss-Legendre (cos theta) x trapezoid (phi) product rule."""
    c, rho, kappa = np.array([0.5, 0.5, 0.5]), 0.25, 60.0
    nt, nph = 48, 96
    z, wz = np.polynomial.legendre.leggauss(nt)
    ph = 2 * np.pi * np.arange(nph) / nph
    Z, PH = np.meshgrid(z, ph, indexing="ij")
    S = np.sqrt(1 - Z ** 2)
    y = c + rho * np.stack([S * np.cos(PH), S * np.sin(PH), Z], -1).reshape(-1, 3)
    F = (np.repeat(wz, nph) * (2 * np.pi / nph) * rho ** 2).astype(np.complex128)
    rng = np.random.default_rng(1)
    xh = rng.normal(size=(40, 3))
    xh /= np.linalg.norm(xh, axis=1, keepdims=True)
    u = oracle.farfield_direct(xh, y, F, kappa)
    ref = 4 * np.pi * rho ** 2 * np.sin(kappa * rho) / (kappa * rho) * np.exp(-1j * kappa * (xh @ c))
    assert np.max(np.abs(u - ref)) <= 1e-11 * 4 * np.pi * rho ** 2


def test_linearity_and_adjoint_identity():
    """Linear in F; <A F, g> = <F, A^H g> with A^H the s = +1 sum over the
    swapped point sets."""
    rng = np.random.default_rng(2)
    xh = _dirs2(50)
    y = rng.uniform(0, 1, (70, 2))
    F = rng.normal(size=70) + 1j * rng.normal(size=70)
    G = rng.normal(size=70) + 1j * rng.normal(size=70)
    g = rng.normal(size=50) + 1j * rng.normal(size=50)
    kappa = 90.0
    uF, uG = oracle.farfield_direct(xh, y, F, kappa), oracle.farfield_direct(xh, y, G, kappa)
    uFG = oracle.farfield_direct(xh, y, 2 * F - 1j * G, kappa)
    assert np.max(np.abs(uFG - (2 * uF - 1j * uG))) <= 1e-13 * np.abs(uFG).max()
    v = oracle.farfield_direct(y, xh, g, kappa, sign=+1)
    assert abs(np.vdot(g, uF) - np.vdot(v, F)) <= 1e-12 * np.linalg.norm(g) * np.linalg.norm(uF)


def test_rejects_bad_arguments():
    with pytest.raises(ValueError):
        oracle.farfield_direct(_dirs2(3), np.zeros((2, 2)), np.ones(2), -1.0)
    with pytest.raises(ValueError):
        oracle.farfield_direct(_dirs2(3), np.zeros((2, 2)), np.ones(2), 1.0, sign=0)
