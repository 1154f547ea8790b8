"""Multi-RHS apply (sft_apply_batch): several charge
vectors through one plan, one launch per step for the whole batch.

The per-vector arithmetic is unchanged, so every row of a batch must equal
sft_apply on that row bit for bit; rows are also checked against the oracle
butterfly (rel. L2 <= 1e-10, BASELINE.json:5) and the direct sum.
"""
import numpy as np
import pytest

import oracle
import synth
from helpers import assert_close

pytestmark = pytest.mark.gpu

PARITY = 1e-10
DIRECT_TOL = {5: 5e-2, 7: 1e-3, 9: 1e-5}


def _charges(nrhs, n, seed):
    return np.stack([synth.random_charges(n, seed + r) for r in range(nrhs)])


def _run(x, k, F, N, p, precision=0, adjoint=False, host=False):
    import torch
    import paper_0801_1524_b200 as sft
    d = x.shape[1]
    xt, kt = torch.from_numpy(x).cuda(), torch.from_numpy(k).cuda()
    with sft.Plan(d, N, p, xt, kt, precision=precision, adjoint=adjoint) as plan:
        Ft = torch.from_numpy(F) if host else torch.from_numpy(F).cuda()
        U = plan.apply_batch(Ft)
        torch.cuda.synchronize()
        U = U.cpu().numpy() if hasattr(U, "cpu") else np.asarray(U)
        singles = []
        for r in range(F.shape[0]):
            u = plan.apply(torch.from_numpy(np.ascontiguousarray(F[r])).cuda())
            singles.append(u.cpu().numpy())
        # a second batch call reuses the grown buffers
        U2 = plan.apply_batch(Ft)
        U2 = U2.cpu().numpy() if hasattr(U2, "cpu") else np.asarray(U2)
    return U, np.stack(singles), U2


@pytest.mark.parametrize("name,p,nrhs", [("C0", 5, 3), ("C0", 7, 2), ("C0", 9, 4), ("C1", 7, 3), ("C1", 9, 2)])
def test_batch_2d_bitwise_and_parity(name, p, nrhs):
    w = synth.make_workload(name, p=p)
    F = _charges(nrhs, len(w.k), 100)
    U, S, U2 = _run(w.x, w.k, F, w.N, p)
    assert U.shape == (nrhs, len(w.x))
    assert np.array_equal(U.view(np.uint64), S.view(np.uint64))
    assert np.array_equal(U.view(np.uint64), U2.view(np.uint64))
    for r in (0, nrhs - 1):
        assert_close(U[r], oracle.butterfly(w.x, w.k, F[r], w.N, p), PARITY)
    if name == "C0":
        assert_close(U[1], oracle.direct(w.x, w.k, F[1], w.N), DIRECT_TOL[p])


@pytest.mark.parametrize("N,p", [(16, 5), (16, 9), (32, 7)])
def test_batch_3d(N, p):
    w = synth.make_workload("C3", N=N, p=p)
    F = _charges(3, len(w.k), 200)
    U, S, _ = _run(w.x, w.k, F, w.N, p)
    assert np.array_equal(U.view(np.uint64), S.view(np.uint64))
    assert_close(U[2], oracle.butterfly(w.x, w.k, F[2], w.N, p), PARITY)


def test_batch_host_pointers_and_linearity():
    """Host (numpy) input and output: staged copies of every row inside the
    call; the batch of (f, g, f + 2g) is linear row-wise."""
    w = synth.make_workload("C1")
    f = synth.random_charges(len(w.k), 7)
    g = synth.random_charges(len(w.k), 8)
    F = np.stack([f, g, f + 2 * g])
    U, S, _ = _run(w.x, w.k, F, w.N, w.p, host=True)
    assert np.array_equal(U.view(np.uint64), S.view(np.uint64))
    assert_close(U[2], U[0] + 2 * U[1], 1e-13)


def test_batch_dense_leaves():
    """Leaves with more sources than a warp (chunked leaf path: partial sums of
    one RHS are re-read from the level buffer of that RHS)."""
    N = 64
    rng = np.random.default_rng(11)
    w = synth.make_workload("C0")
    k = np.concatenate([w.k, 17.0 + rng.uniform(0, 1, (200, 2))])
    x = np.concatenate([w.x, 33.0 + rng.uniform(0, 1, (150, 2))])
    F = _charges(3, len(k), 300)
    U, S, _ = _run(x, k, F, N, 9)
    assert np.array_equal(U.view(np.uint64), S.view(np.uint64))
    assert_close(U[1], oracle.butterfly(x, k, F[1], N, 9), PARITY)


def test_batch_fp32_and_adjoint():
    w = synth.make_workload("C0", p=9)
    F = _charges(3, len(w.k), 400)
    U, S, _ = _run(w.x, w.k, F, w.N, 9, precision=1)
    assert np.array_equal(U.view(np.uint64), S.view(np.uint64))
    assert_close(U[0], oracle.butterfly(w.x, w.k, F[0], w.N, 9), 1.3e-6)  # FP32_PARITY (test_gpu_parity.py)
    G = _charges(2, len(w.x), 500)
    V, S, _ = _run(w.x, w.k, G, w.N, 9, adjoint=True)
    assert V.shape == (2, len(w.k))
    assert np.array_equal(V.view(np.uint64), S.view(np.uint64))
    vb = np.conj(oracle.butterfly(w.k, w.x, np.conj(G[1]), w.N, 9))
    assert_close(V[1], vb, PARITY)


def test_batch_errors():
    import ctypes
    import torch
    import paper_0801_1524_b200 as sft
    w = synth.make_workload("C0")
    L = sft.lib()
    with sft.Plan(2, w.N, 5, torch.from_numpy(w.x).cuda(), torch.from_numpy(w.k).cuda()) as plan:
        F = torch.zeros(2, len(w.k), dtype=torch.complex128, device="cuda")
        U = torch.empty(2, len(w.x), dtype=torch.complex128, device="cuda")
        fp, up = ctypes.c_void_p(F.data_ptr()), ctypes.c_void_p(U.data_ptr())
        assert L.sft_apply_batch(plan._h, 0, fp, len(w.k), up, len(w.x)) == 1
        assert L.sft_apply_batch(plan._h, 2, fp, len(w.k) - 1, up, len(w.x)) == 1
        assert L.sft_apply_batch(plan._h, 2, fp, len(w.k), up, len(w.x) - 1) == 1
        assert L.sft_apply_batch(plan._h, 2, None, len(w.k), up, len(w.x)) == 1
        assert L.sft_apply_batch(plan._h, 2, fp, len(w.k), up, len(w.x)) == 0
        torch.cuda.synchronize()
        assert bool((U == 0).all())  # f == 0 gives u == 0 exactly
