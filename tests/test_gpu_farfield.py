"""Far-field adapter (sft_farfield_plan, PAPER.md:82-96 eq. far) on the GPU:
u_inf(xhat_i) = sum_j exp(-i kappa xhat_i.y_j) F_j through the butterfly.

* parity: the oracle butterfly on the rescaled problem (x = N/2 - kappa
  xhat/(2 pi), k = N y, charges F_j exp(-i pi sum_a k_a), mapped here in numpy
  from the paper's statement) -- rel. L2 <= 1e-10;
* accuracy: the oracle's far-field sum (plain definition) within the BASELINE
  tolerance of p, and the Jacobi-Anger / Funk-Hecke closed forms.
"""
import numpy as np
import pytest
from scipy.special import j0

import oracle
import synth
from helpers import assert_close

pytestmark = pytest.mark.gpu

PARITY = 1e-10
DIRECT_TOL = {5: 5e-2, 7: 1e-3, 9: 1e-5}


def _dirs2(n):
    t = 2 * np.pi * (np.arange(n) + 0.25) / n
    return np.stack([np.cos(t), np.sin(t)], 1)


def _dirs3(n, seed):
    v = np.random.default_rng(seed).normal(size=(n, 3))
    return v / np.linalg.norm(v, axis=1, keepdims=True)


def _gpu(xh, y, F, kappa, p, adjoint=False, batch=False):
    import torch
    import paper_0801_1524_b200 as sft
    d = xh.shape[1]
    with sft.Plan.farfield(d, kappa, p, torch.from_numpy(xh).cuda(), torch.from_numpy(y).cuda(),
                           adjoint=adjoint) as plan:
        Ft = torch.from_numpy(np.ascontiguousarray(F)).cuda()
        u = plan.apply_batch(Ft) if batch else plan.apply(Ft)
        torch.cuda.synchronize()
        return u.cpu().numpy(), plan.N


def _mapped(xh, y, F, kappa, N):
    """eq. far -> eq. sfft, written out independently of the library."""
    x = N / 2 - kappa * xh / (2 * np.pi)
    k = N * y
    f = F * np.exp(-1j * np.pi * np.sum(k, axis=1))
    return x, k, f


def _circle(n, c, rho):
    t = 2 * np.pi * np.arange(n) / n
    return c + rho * np.stack([np.cos(t), np.sin(t)], 1)


@pytest.mark.parametrize("p,kappa", [(5, 200.0), (7, 700.0), (9, 2000.0)])
def test_farfield_2d(p, kappa):
    rng = np.random.default_rng(3)
    y = _circle(int(4 * 2 * np.pi * 0.35 * kappa / np.pi), np.array([0.5, 0.5]), 0.35)
    F = synth.random_charges(len(y), 5)
    xh = _dirs2(int(kappa))
    u, N = _gpu(xh, y, F, kappa, p)
    assert N >= kappa / np.pi and N < 2 * kappa / np.pi + 2
    x, k, f = _mapped(xh, y, F, kappa, N)
    assert_close(u, oracle.butterfly(x, k, f, N, p), PARITY)
    ud = oracle.farfield_direct(xh, y, F, kappa)
    assert_close(u, ud, DIRECT_TOL[p])
    del rng


def test_farfield_circle_closed_form():
    """Uniform density on a circle: 2 pi rho J0(kappa rho) exp(-i kappa xhat.c)."""
    kappa, rho, c = 1500.0, 0.3, np.array([0.45, 0.55])
    n = 2048
    y = _circle(n, c, rho)
    F = np.full(n, 2 * np.pi * rho / n, dtype=np.complex128)
    xh = _dirs2(3000)
    u, _ = _gpu(xh, y, F, kappa, 9)
    ref = 2 * np.pi * rho * j0(kappa * rho) * np.exp(-1j * kappa * (xh @ c))
    # the butterfly's error is relative to the charge mass sum |F| = 2 pi rho
    assert np.max(np.abs(u - ref)) <= DIRECT_TOL[9] * 2 * np.pi * rho


@pytest.mark.parametrize("p", [5, 7])
def test_farfield_3d_sphere(p):
    kappa, rho, c = 150.0, 0.3, np.array([0.5, 0.5, 0.5])
    nt, nph = 64, 128
    z, wz = np.polynomial.legendre.leggauss(nt)
    ph = 2 * np.pi * np.arange(nph) / nph
    Z, PH = np.meshgrid(z, ph, indexing="ij")
    S = np.sqrt(1 - Z ** 2)
    y = c + rho * np.stack([S * np.cos(PH), S * np.sin(PH), Z], -1).reshape(-1, 3)
    F = (np.repeat(wz, nph) * (2 * np.pi / nph) * rho ** 2).astype(np.complex128)
    xh = _dirs3(1500, 4)
    u, N = _gpu(xh, y, F, kappa, p)
    ref = 4 * np.pi * rho ** 2 * np.sin(kappa * rho) / (kappa * rho) * np.exp(-1j * kappa * (xh @ c))
    assert np.max(np.abs(u - ref)) <= 3 * DIRECT_TOL[p] * 4 * np.pi * rho ** 2
    x, k, f = _mapped(xh, y, F, kappa, N)
    assert_close(u, oracle.butterfly(x, k, f, N, p), PARITY)


def test_farfield_adjoint_and_batch():
    """adjoint: v_j = sum_i exp(+i kappa xhat_i.y_j) g_i; batch rows equal singles."""
    kappa, p = 400.0, 9
    y = _circle(900, np.array([0.5, 0.5]), 0.4)
    xh = _dirs2(500)
    g = synth.random_charges(len(xh), 6)
    v, N = _gpu(xh, y, g, kappa, p, adjoint=True)
    assert v.shape == (len(y),)
    vd = oracle.farfield_direct(y, xh, g, kappa, sign=+1)
    assert_close(v, vd, DIRECT_TOL[p])
    # parity: conj of the oracle butterfly from the directions to the scatterer points
    x, k, _ = _mapped(xh, y, np.zeros(len(y)), kappa, N)
    vb = np.conj(oracle.butterfly(k, x, np.conj(g), N, p)) * np.exp(1j * np.pi * np.sum(k, axis=1))
    assert_close(v, vb, PARITY)
    F = np.stack([synth.random_charges(len(y), 10 + r) for r in range(3)])
    U, _ = _gpu(xh, y, F, kappa, p, batch=True)
    for r in range(3):
        ur, _ = _gpu(xh, y, F[r], kappa, p)
        assert np.array_equal(U[r].view(np.uint64), ur.view(np.uint64))


def test_farfield_errors():
    import torch
    import paper_0801_1524_b200 as sft
    xh = torch.from_numpy(_dirs2(8)).cuda()
    y = torch.from_numpy(_circle(8, np.array([0.5, 0.5]), 0.3)).cuda()
    with pytest.raises(sft.SftError):
        sft.Plan.farfield(2, -1.0, 9, xh, y)
    with pytest.raises(sft.SftError):
        sft.Plan.farfield(2, 100.0, 9, xh, y + 1.0)  # y outside [0,1]^2
    with pytest.raises(sft.SftError):
        sft.Plan.farfield(2, 100.0, 9, 2 * xh, y)  # not unit directions
