"""TEST INFRASTRUCTURE ONLY -- ctypes wrapper of the plain CPU oracle
(``oracle/sft_oracle.c``, long double, paper-literal).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module.  The
product path (``paper_0801_1524_b200``) never imports it and shares no code
with it.

Every function cites the PAPER.md passage it follows; see the C file header.
Parity of every function here is pinned by ``tests/test_oracle_pins.py``
against closed forms, invariants and independent brute force.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sft_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

_c_i64p = ctypes.POINTER(ctypes.c_int64)
_c_dp = ctypes.POINTER(ctypes.c_double)
_c_u8p = ctypes.POINTER(ctypes.c_uint8)
_c_ip = ctypes.POINTER(ctypes.c_int)


def build(force: bool = False) -> str:
    """Compile the oracle (plain gcc, OpenMP).  Building the checker is not using it."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp", "-Wall", "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        L.oracle_direct.argtypes = [ctypes.c_int, ctypes.c_double, _c_dp, ctypes.c_int64, _c_dp, ctypes.c_int64,
                                    _c_dp, _c_dp, _c_i64p, ctypes.c_int64, ctypes.c_int]
        L.oracle_farfield_direct.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_int, _c_dp, ctypes.c_int64, _c_dp,
                                             ctypes.c_int64, _c_dp, _c_dp, ctypes.c_int]
        L.oracle_G.argtypes = [ctypes.c_int, _c_dp]
        L.oracle_H.argtypes = [ctypes.c_int, _c_dp]
        for fn in (L.oracle_M1, L.oracle_E1):
            fn.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                           ctypes.c_int64, _c_dp]
        L.oracle_solve_charges.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int, _c_i64p, ctypes.c_int64,
                                           _c_i64p, ctypes.c_int64, _c_dp, _c_dp]
        L.oracle_leaf_charges.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int, _c_i64p, _c_dp, _c_dp,
                                          ctypes.c_int64, _c_dp]
        L.oracle_pair_charges.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int, ctypes.c_int, _c_i64p, _c_i64p,
                                          ctypes.c_int, _c_ip, _c_dp, _c_dp]
        L.oracle_eval_charges.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int, _c_i64p, ctypes.c_int64, _c_dp,
                                          _c_dp, ctypes.c_int64, _c_dp]
        L.oracle_tree_counts.argtypes = [ctypes.c_int, ctypes.c_int64, _c_dp, ctypes.c_int64, _c_i64p]
        L.oracle_butterfly.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int, _c_dp, ctypes.c_int64, _c_dp,
                                       ctypes.c_int64, _c_dp, _c_dp, _c_i64p, ctypes.c_int64, _c_u8p, ctypes.c_int]
        L.oracle_max_threads.argtypes = []
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(_c_dp)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _cplx_view(a):
    a = np.ascontiguousarray(a, dtype=np.complex128)
    return a.view(np.float64)


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def direct(x, k, f, N, targets=None, nthreads=0) -> np.ndarray:
    """u_i = sum_j exp(2 pi i x_i.k_j/N) f_j (eq. sfft), long double."""
    x = _f64(x); k = _f64(k)
    d = x.shape[1]
    fv = _cplx_view(f)
    if targets is None:
        n_out, tp, nt = len(x), None, 0
    else:
        targets = np.ascontiguousarray(targets, dtype=np.int64)
        n_out, tp, nt = len(targets), targets.ctypes.data_as(_c_i64p), len(targets)
    u = np.zeros(n_out, dtype=np.complex128)
    rc = lib().oracle_direct(d, float(N), _dp(x), len(x), _dp(k), len(k), _dp(fv), _dp(u.view(np.float64)),
                             tp, nt, int(nthreads))
    if rc:
        raise ValueError(f"oracle_direct rc={rc}")
    return u


def farfield_direct(xhat, y, F, kappa, sign=-1, nthreads=0) -> np.ndarray:
    """u_i = sum_j exp(sign * i kappa xhat_i.y_j) F_j: the far-field pattern of
    eq. (far), with the quadrature F_j = f(y_j) ds_j (sign -1);
    sign +1 is the adjoint sum.  Long double, plain definition."""
    xhat = _f64(xhat); y = _f64(y)
    Fv = _cplx_view(F)
    u = np.zeros(len(xhat), dtype=np.complex128)
    rc = lib().oracle_farfield_direct(xhat.shape[1], float(kappa), int(sign), _dp(xhat), len(xhat), _dp(y), len(y),
                                      _dp(Fv), _dp(u.view(np.float64)), int(nthreads))
    if rc:
        raise ValueError(f"oracle_farfield_direct rc={rc}")
    return u


def G(p) -> np.ndarray:
    """(G)_{ll'} = exp(2 pi i l l'/(p-1)^2)."""
    out = np.zeros((p, p), dtype=np.complex128)
    lib().oracle_G(p, _dp(out.view(np.float64)))
    return out


def H(p) -> np.ndarray:
    """(H)_{ll'} = exp(pi i l l'/(p-1)^2)."""
    out = np.zeros((p, p), dtype=np.complex128)
    lib().oracle_H(p, _dp(out.view(np.float64)))
    return out


def M1(p, N, cA, wA, cB, wB) -> np.ndarray:
    """M1 = M11 G M12 (eq. M1), one axis."""
    out = np.zeros((p, p), dtype=np.complex128)
    lib().oracle_M1(p, N, cA, wA, cB, wB, _dp(out.view(np.float64)))
    return out


def E1(p, N, cA, wA, cBc, wBc) -> np.ndarray:
    """E1 = E11 H E12 (eq. E1), one axis."""
    out = np.zeros((p, p), dtype=np.complex128)
    lib().oracle_E1(p, N, cA, wA, cBc, wBc, _dp(out.view(np.float64)))
    return out


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def solve_charges(d, N, p, cA, wA, cB, wB, u) -> np.ndarray:
    """f = M^{-1} u on the pair (A,B); u is p^d complex (row-major)."""
    cA = _i64(cA); cB = _i64(cB)
    uv = _cplx_view(u.reshape(-1))
    f = np.zeros(p ** d, dtype=np.complex128)
    rc = lib().oracle_solve_charges(d, N, p, cA.ctypes.data_as(_c_i64p), wA, cB.ctypes.data_as(_c_i64p), wB,
                                    _dp(uv), _dp(f.view(np.float64)))
    if rc:
        raise ValueError("oracle_solve_charges")
    return f


def leaf_charges(d, N, p, cB, k, f) -> np.ndarray:
    """f^{A0 B} for leaf B at corner cB (width 1), A0 root of T_X."""
    cB = _i64(cB); k = _f64(k).reshape(-1, d)
    fv = _cplx_view(f)
    out = np.zeros(p ** d, dtype=np.complex128)
    rc = lib().oracle_leaf_charges(d, N, p, cB.ctypes.data_as(_c_i64p), _dp(k), _dp(fv), len(k),
                                   _dp(out.view(np.float64)))
    if rc:
        raise ValueError("oracle_leaf_charges")
    return out


def pair_charges(d, N, p, t, ca, cb, child_bits, fchild) -> np.ndarray:
    """f^{AB} from children's f^{A'B_c} (step 3 P:300-305).

    ca: coords of A at level L-t; cb: coords of B at level t; child_bits[i]
    gives the child index c of B_c (axis a <-> bit d-1-a); fchild[i] is the
    p^d array f^{A' B_c}.
    """
    ca = _i64(ca); cb = _i64(cb)
    bits = np.ascontiguousarray(child_bits, dtype=np.int32)
    fc = _cplx_view(np.asarray(fchild, dtype=np.complex128).reshape(-1))
    out = np.zeros(p ** d, dtype=np.complex128)
    rc = lib().oracle_pair_charges(d, N, p, t, ca.ctypes.data_as(_c_i64p), cb.ctypes.data_as(_c_i64p), len(bits),
                                   bits.ctypes.data_as(_c_ip), _dp(fc), _dp(out.view(np.float64)))
    if rc:
        raise ValueError("oracle_pair_charges")
    return out


def eval_charges(d, N, p, cB, wB, f, x) -> np.ndarray:
    """sum_l exp(2 pi i x.k^B_l/N) f_l on the grid of box B."""
    cB = _i64(cB); x = _f64(x).reshape(-1, d)
    fv = _cplx_view(f)
    u = np.zeros(len(x), dtype=np.complex128)
    rc = lib().oracle_eval_charges(d, N, p, cB.ctypes.data_as(_c_i64p), wB, _dp(fv), _dp(x), len(x),
                                   _dp(u.view(np.float64)))
    if rc:
        raise ValueError("oracle_eval_charges")
    return u


def tree_counts(pts, N) -> np.ndarray:
    """Number of non-empty boxes per level 0..L."""
    pts = _f64(pts)
    L = int(N).bit_length() - 1
    out = np.zeros(L + 1, dtype=np.int64)
    rc = lib().oracle_tree_counts(pts.shape[1], N, _dp(pts), len(pts), out.ctypes.data_as(_c_i64p))
    if rc:
        raise ValueError("oracle_tree_counts")
    return out


def butterfly(x, k, f, N, p, targets=None, src_active=None, nthreads=0) -> np.ndarray:
    """Paper-literal butterfly, §2.2 steps 1-4, long double.

    ``targets``: evaluate only these target indices (restricts A to their
    ancestors).  ``src_active``: boolean mask; inactive sources carry no
    charge (restricts B to boxes holding active sources).  Both restrictions
    skip only pairs that are zero or never reach a sampled target.
    """
    x = _f64(x); k = _f64(k)
    d = x.shape[1]
    fv = _cplx_view(f)
    if targets is None:
        n_out, tp, nt = len(x), None, 0
    else:
        targets = np.ascontiguousarray(targets, dtype=np.int64)
        n_out, tp, nt = len(targets), targets.ctypes.data_as(_c_i64p), len(targets)
    if src_active is None:
        sp = None
    else:
        src_active = np.ascontiguousarray(src_active, dtype=np.uint8)
        sp = src_active.ctypes.data_as(_c_u8p)
    u = np.zeros(n_out, dtype=np.complex128)
    rc = lib().oracle_butterfly(d, int(N), int(p), _dp(x), len(x), _dp(k), len(k), _dp(fv),
                                _dp(u.view(np.float64)), tp, nt, sp, int(nthreads))
    if rc:
        raise ValueError(f"oracle_butterfly rc={rc}")
    return u


def rel_l2(approx, exact) -> float:
    """sqrt(sum |u - u^a|^2 / sum |u|^2)."""
    approx = np.asarray(approx); exact = np.asarray(exact)
    return float(np.sqrt(np.sum(np.abs(approx - exact) ** 2) / np.sum(np.abs(exact) ** 2)))
