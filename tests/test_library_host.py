"""Host-side tests of libsft (no GPU): the C ABI loads and exports every
symbol include/sft.h declares; the constant operator tables the kernels use
reproduce the oracle's paper-literal pair step at the field level; the host
partitioner of the multi-GPU path is consistent."""
import ctypes

import numpy as np
import pytest

import oracle
import synth

sft = pytest.importorskip("paper_0801_1524_b200")


def test_library_exports_header_symbols():
    L = sft.lib()
    assert len(sft.HEADER_SYMBOLS) >= 15
    for name in sft.HEADER_SYMBOLS:
        assert hasattr(L, name), name
    assert L.sft_strerror(0).decode() == "ok"
    assert "outside" in L.sft_strerror(2).decode()


def test_library_rejects_bad_args_without_gpu():
    L = sft.lib()
    h = ctypes.c_void_p()
    x = np.zeros((4, 2))
    # dim, N, p are validated before any device work
    assert L.sft_plan(4, 64, 5, x.ctypes.data, 4, x.ctypes.data, 4, None, ctypes.byref(h)) == 1
    assert L.sft_plan(2, 48, 5, x.ctypes.data, 4, x.ctypes.data, 4, None, ctypes.byref(h)) == 1
    assert L.sft_plan(2, 64, 6, x.ctypes.data, 4, x.ctypes.data, 4, None, ctypes.byref(h)) == 1
    assert L.sft_plan(2, 64, 5, x.ctypes.data, 0, x.ctypes.data, 4, None, ctypes.byref(h)) == 1
    assert L.sft_destroy(None) == 0
    assert L.sft_apply(None, None, None) == 1
    # multi-RHS and far-field entry points validate before any device work
    assert L.sft_apply_batch(None, 2, None, 4, None, 4) == 1
    xh = np.array([[1.0, 0.0], [0.0, 1.0]])
    assert L.sft_farfield_plan(2, -1.0, 9, xh.ctypes.data, 2, x.ctypes.data, 4, None, ctypes.byref(h)) == 1
    assert L.sft_farfield_plan(2, float("nan"), 9, xh.ctypes.data, 2, x.ctypes.data, 4, None, ctypes.byref(h)) == 1
    assert L.sft_farfield_plan(4, 10.0, 9, xh.ctypes.data, 2, x.ctypes.data, 4, None, ctypes.byref(h)) == 1
    assert L.sft_farfield_plan(2, 10.0, 9, None, 2, x.ctypes.data, 4, None, ctypes.byref(h)) == 1
    assert L.sft_farfield_plan(2, 10.0, 9, xh.ctypes.data, 0, x.ctypes.data, 4, None, ctypes.byref(h)) == 1


# ------------------------------------------------------------- operator tables
def _kernel(x, k, N):
    return np.exp(2j * np.pi * (np.asarray(x) @ np.asarray(k).T) / N)


def _grid(corner, width, p):
    d = len(corner)
    ax = [corner[a] + np.arange(p) * width / (p - 1) for a in range(d)]
    mesh = np.meshgrid(*ax, indexing="ij")
    return np.stack([m.reshape(-1) for m in mesh], axis=1)


def _axis_apply(T, X, a):
    return np.moveaxis(np.tensordot(T, X, axes=([1], [a])), 0, a)


@pytest.mark.parametrize("p", [5, 7, 9])
def test_real_form_equals_V(p):
    """T = c (RC + i s RS) equals V conjugated by diag(e^{i pi m/(p-1)})."""
    V, invD, RC, RS = sft.operator_tables(p, real=True)
    P1 = p - 1
    Eh = np.diag(np.exp(1j * np.pi * np.arange(p) / P1))
    for al in range(2):
        for be in range(2):
            c = [1, 1j, 1, -1j][al * 2 + be] if be else 1
            T = c * (RC[be] + 1j * (2 * al - 1) * RS[be])
            assert np.max(np.abs(T - Eh @ V[al, be] @ np.linalg.inv(Eh))) < 2e-14


@pytest.mark.parametrize("d,p", [(2, 5), (2, 7), (2, 9), (3, 5), (3, 7)])
def test_tables_reproduce_oracle_pair_step(d, p):
    """The kernels' child->parent operator (box-relative h charges, T from
    RC/RS) gives the same field in A as the oracle's paper-literal
    E-then-M^{-1} step -- checked at 100 random points of A."""
    rng = np.random.default_rng(3 + p + d)
    V, invD, RC, RS = sft.operator_tables(p, real=True)
    N, L, P1 = 256, 8, p - 1
    T = {}
    for al in range(2):
        for be in range(2):
            c = 1 if be == 0 else (1j if al == 0 else -1j)
            T[al, be] = c * (RC[be] + 1j * (2 * al - 1) * RS[be])
    lidx = np.arange(p)
    for _ in range(3):
        t = int(rng.integers(1, L - 1))
        wA, wB, wBc = N >> (L - t), N >> t, N >> (t + 1)
        ca = rng.integers(0, N // wA, d); cb = rng.integers(0, N // wB, d)
        cap = ca >> 1
        bits = np.sort(rng.choice(2 ** d, int(rng.integers(1, 2 ** d + 1)), replace=False))
        fch, hch = [], []
        for c in bits:
            cbit = np.array([(c >> (d - 1 - a)) & 1 for a in range(d)])
            cBc = (2 * cb + cbit) * wBc
            src = cBc + rng.uniform(0, wBc, (4, d))
            q = rng.normal(size=4) + 1j * rng.normal(size=4)
            u = _kernel(_grid(cap * 2 * wA, 2 * wA, p), src, N) @ q   # check potentials at x^{A'}
            f = oracle.solve_charges(d, N, p, cap * 2 * wA, 2 * wA, cBc, wBc, u)
            fch.append(f)
            h = f.reshape([p] * d)
            for a in range(d):  # h = e^{i pi l/P1} e^{2 pi i a' l/P1} f per axis
                ph = np.exp(1j * np.pi * lidx / P1) * np.exp(2j * np.pi * cap[a] * lidx / P1)
                h = h * ph.reshape([p if b == a else 1 for b in range(d)])
            hch.append(h)
        f_or = oracle.pair_charges(d, N, p, t, ca, cb, bits, np.array(fch))
        alpha = ca & 1
        h_ab = np.zeros([p] * d, complex)
        for i, c in enumerate(bits):
            y = hch[i]
            for a in range(d):
                y = _axis_apply(T[alpha[a], (c >> (d - 1 - a)) & 1], y, a)
            h_ab += y
        f_tab = h_ab
        for a in range(d):  # back to paper charges: f = e^{-2 pi i a l/P1} e^{-i pi l/P1} h
            ph = np.exp(-2j * np.pi * ca[a] * lidx / P1) * np.exp(-1j * np.pi * lidx / P1)
            f_tab = f_tab * ph.reshape([p if b == a else 1 for b in range(d)])
        xs = ca * wA + rng.uniform(0, wA, (100, d))
        KB = _kernel(xs, _grid(cb * wB, wB, p), N)
        u_or = KB @ f_or
        u_tab = KB @ f_tab.reshape(-1)
        assert np.linalg.norm(u_tab - u_or) / np.linalg.norm(u_or) < 1e-12


@pytest.mark.parametrize("d,p", [(2, 5), (2, 9), (3, 7)])
def test_leaf_weights_reproduce_oracle_leaf(d, p):
    """h-leaf weights e^{i pi s} invD_m prod_{q!=m} sin(pi (s P1 - q)/P1^2)
    (kernel K2) give the oracle's leaf charges at field level."""
    rng = np.random.default_rng(11)
    V, invD = sft.operator_tables(p)
    N, P1 = 64, p - 1
    for _ in range(3):
        cB = rng.integers(0, N, d)
        k = cB + rng.uniform(0, 1, (3, d))
        f = rng.normal(size=3) + 1j * rng.normal(size=3)
        h = np.zeros([p] * d, complex)
        for j in range(3):
            s = k[j] - cB
            w = np.ones([p] * d, complex) * f[j] * np.exp(1j * np.pi * s.sum())
            for a in range(d):
                r = np.array([invD[m] * np.prod([np.sin(np.pi * (s[a] * P1 - q) / P1 ** 2) for q in range(p) if q != m])
                              for m in range(p)])
                w = w * r.reshape([p if b == a else 1 for b in range(d)])
            h += w
        f_tab = h
        for a in range(d):
            f_tab = f_tab * np.exp(-1j * np.pi * np.arange(p) / P1).reshape([p if b == a else 1 for b in range(d)])
        f_or = oracle.leaf_charges(d, N, p, cB, k, f)
        xs = rng.uniform(0, N, (100, d))
        K = _kernel(xs, _grid(cB, 1, p), N)
        assert np.linalg.norm(K @ f_tab.reshape(-1) - K @ f_or) / np.linalg.norm(K @ f_or) < 1e-12


# ------------------------------------------------------------- partitioner
def tree_levels(pts, N, d):
    """Morton-ordered unique boxes per level and parent indices (numpy)."""
    L = N.bit_length() - 1
    leaf = np.minimum(np.floor(pts).astype(np.int64), N - 1)
    key = np.zeros(len(pts), np.int64)
    for b in range(L - 1, -1, -1):
        for a in range(d):
            key = (key << 1) | ((leaf[:, a] >> b) & 1)
    keys = [np.unique(key >> (d * (L - l))) for l in range(L + 1)]
    parents = [None] + [np.searchsorted(keys[l - 1], keys[l] >> d).astype(np.int32) for l in range(1, L + 1)]
    return keys, parents


@pytest.mark.parametrize("name,world", [("C1", 2), ("C1", 8), ("C2", 4), ("C2", 8), ("C3", 8)])
def test_partitioner_invariants(name, world):
    w = synth.make_workload(name)
    L = w.N.bit_length() - 1
    kx, px = tree_levels(w.x, w.N, w.dim)
    kk, pk = tree_levels(w.k, w.N, w.dim)
    cx = [len(v) for v in kx]; ck = [len(v) for v in kk]
    sk, sx, m, rng, cost = sft.choose_partition(L, world, cx, ck, px, pk)
    assert 0 <= sk <= m <= L - sx
    # contiguous ranges covering every subtree exactly once, in rank order
    assert rng[0, 0] == 0 and rng[-1, 1] == ck[sk] and rng[0, 2] == 0 and rng[-1, 3] == cx[sx]
    assert np.all(rng[1:, 0] == rng[:-1, 1]) and np.all(rng[1:, 2] == rng[:-1, 3])
    # balance: no rank has more than ~1.6x the ideal share of either phase
    pairs = [ck[t] * cx[L - t] for t in range(L + 1)]
    ph1 = sum(pairs[m:]); ph2 = sum(pairs[:m]) + cx[L]
    assert cost[0] <= 1.6 * ph1 / world + max(pairs) and cost[1] <= 1.6 * ph2 / world + max(pairs)


def test_partitioner_forced_and_infeasible():
    w = synth.make_workload("C1")
    L = 10
    kx, px = tree_levels(w.x, w.N, 2)
    kk, pk = tree_levels(w.k, w.N, 2)
    cx = [len(v) for v in kx]; ck = [len(v) for v in kk]
    sk, sx, m, rng, _ = sft.choose_partition(L, 2, cx, ck, px, pk, force=(2, 3, 5))
    assert (sk, sx, m) == (2, 3, 5)
    with pytest.raises(sft.SftError):
        sft.choose_partition(L, 2, cx, ck, px, pk, force=(6, 6, 5))  # m < s_K: infeasible


@pytest.mark.parametrize("p", [5, 7, 9])
def test_mirror_symmetry_of_tables(p):
    """The symmetric translation consumer relies on the child-1
    operators being the mirror images of the child-0 ones: RC_1 = J RS_0 J and
    RS_1 = J RC_0 J (J = index reversal) -- the child-1 grid is the mirror of
    the child-0 grid about the parent's centre and the Lagrange basis on the
    nodes e^{2 pi i m/(p-1)^2} maps to its conjugate under the mirror."""
    _, _, RC, RS = sft.operator_tables(p, real=True)
    J = np.eye(p)[::-1]
    assert np.max(np.abs(RC[1] - J @ RS[0] @ J)) <= 1e-15
    assert np.max(np.abs(RS[1] - J @ RC[0] @ J)) <= 1e-15


@pytest.mark.parametrize("p", [7, 9])
def test_symmetric_pass_equals_direct_pass(p):
    """The sum/difference form of one axis pass (s = x0 + J x1, t = x0 - J x1;
    SP, DP, SQ, DQ and the centre column) equals the direct form
    P = RC_0 x0 + RS_1 x1, Q = RS_0 x0 - RC_1 x1 on random complex fibers."""
    _, _, RC, RS = sft.operator_tables(p, real=True)
    H = (p - 1) // 2
    rng = np.random.default_rng(p)
    for _ in range(4):
        x0 = rng.normal(size=p) + 1j * rng.normal(size=p)
        x1 = rng.normal(size=p) + 1j * rng.normal(size=p)
        P = RC[0] @ x0 + RS[1] @ x1
        Q = RS[0] @ x0 - RC[1] @ x1
        s, t = x0 + x1[::-1], x0 - x1[::-1]
        P2 = np.zeros(p, complex)
        Q2 = np.zeros(p, complex)
        for m in range(H):
            mp = p - 1 - m
            SP = 0.5 * (RC[0][m] + RC[0][mp]) @ s
            DP = 0.5 * (RC[0][m] - RC[0][mp]) @ t
            SQ = 0.5 * (RS[0][m] + RS[0][mp]) @ t
            DQ = 0.5 * (RS[0][m] - RS[0][mp]) @ s
            P2[m], P2[mp], Q2[m], Q2[mp] = SP + DP, SP - DP, SQ + DQ, SQ - DQ
        P2[H], Q2[H] = RC[0][H] @ s, RS[0][H] @ t
        assert np.max(np.abs(P - P2)) <= 1e-14 and np.max(np.abs(Q - Q2)) <= 1e-14
