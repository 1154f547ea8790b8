"""B200-native butterfly sparse Fourier transform (Ying, arXiv 0801.1524).

Thin ctypes binding of ``libsft.so`` (C ABI in ``include/sft.h``).  This
module only marshals arguments: every step of the transform -- tree build,
leaf charges, per-level translations, final evaluation -- runs in the
library's sm_100a kernels.  There is no CPU fallback: if the library is
missing or no CUDA device is present, calls raise.

    plan = Plan(dim, N, p, x, k)        # sft_plan
    u = plan.apply(f)                   # sft_apply
    plan.close()                        # sft_destroy

x [nx, dim] float64, k [nk, dim] float64, f [nk] complex128: torch tensors
(CUDA or pinned/pageable CPU) or numpy arrays.  Host buffers are staged by the
library (the end-to-end path).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

__all__ = ["Plan", "lib", "LIB_PATH", "SftError", "operator_tables", "choose_partition", "HEADER_SYMBOLS", "launch_count",
           "nccl_unique_id", "nccl_release"]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SFT_LIB", os.path.join(_HERE, "libsft.so"))
HEADER = os.path.join(os.path.dirname(_HERE), "include", "sft.h")

_c_i64p = ctypes.POINTER(ctypes.c_int64)
_c_dp = ctypes.POINTER(ctypes.c_double)


class SftError(RuntimeError):
    pass


class _Opts(ctypes.Structure):
    _fields_ = [("precision", ctypes.c_int), ("stream", ctypes.c_void_p), ("rank", ctypes.c_int),
                ("world", ctypes.c_int), ("exchange_level", ctypes.c_int), ("split_k", ctypes.c_int),
                ("split_x", ctypes.c_int), ("adjoint", ctypes.c_int), ("nccl_id", ctypes.c_void_p)]


_lib = None


def _header_symbols():
    import re
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(sft_\w+)\s*\(", txt, re.M)))


HEADER_SYMBOLS = _header_symbols() if os.path.exists(HEADER) else []


def lib():
    """Load libsft.so (built by ``paper_0801_1524_b200/build.py`` / ``__graft_entry__.build``)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise SftError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(LIB_PATH)
    vp = ctypes.c_void_p
    L.sft_default_opts.argtypes = [ctypes.POINTER(_Opts)]
    L.sft_default_opts.restype = None
    L.sft_plan.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int, vp, ctypes.c_int64, vp, ctypes.c_int64,
                           ctypes.POINTER(_Opts), ctypes.POINTER(vp)]
    L.sft_apply.argtypes = [vp, vp, vp]
    L.sft_farfield_plan.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_int, vp, ctypes.c_int64, vp,
                                    ctypes.c_int64, ctypes.POINTER(_Opts), ctypes.POINTER(vp)]
    L.sft_apply_batch.argtypes = [vp, ctypes.c_int, vp, ctypes.c_int64, vp, ctypes.c_int64]
    L.sft_destroy.argtypes = [vp]
    L.sft_strerror.argtypes = [ctypes.c_int]
    L.sft_strerror.restype = ctypes.c_char_p
    L.sft_last_error.argtypes = []
    L.sft_last_error.restype = ctypes.c_char_p
    L.sft_plan_stats.argtypes = [vp, _c_i64p, _c_i64p, _c_i64p, _c_dp]
    L.sft_set_timing.argtypes = [vp, ctypes.c_int]
    L.sft_translation_launches.argtypes = [vp, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                           ctypes.POINTER(ctypes.c_int)]
    L.sft_last_timing.argtypes = [vp, _c_dp, _c_dp]
    L.sft_exchange_counts.argtypes = [vp, _c_i64p, _c_i64p]
    L.sft_apply_phase1.argtypes = [vp, vp, vp]
    L.sft_apply_phase2.argtypes = [vp, vp, vp]
    L.sft_partition_info.argtypes = [vp, _c_i64p]
    L.sft_set_peer_buffers.argtypes = [vp, ctypes.POINTER(vp)]
    L.sft_peer_offsets.argtypes = [vp, _c_i64p]
    L.sft_device_alloc.argtypes = [ctypes.c_int64, ctypes.POINTER(vp)]
    L.sft_device_free.argtypes = [vp]
    L.sft_ipc_handle.argtypes = [vp, ctypes.c_char_p]
    L.sft_ipc_open.argtypes = [ctypes.c_char_p, ctypes.POINTER(vp)]
    L.sft_ipc_close.argtypes = [vp]
    L.sft_choose_partition.argtypes = [ctypes.c_int, ctypes.c_int, _c_i64p, _c_i64p,
                                       ctypes.POINTER(ctypes.POINTER(ctypes.c_int32)),
                                       ctypes.POINTER(ctypes.POINTER(ctypes.c_int32)), ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int, _c_i64p, _c_i64p]
    L.sft_operator_tables.argtypes = [ctypes.c_int, _c_dp, _c_dp, _c_dp, _c_dp]
    L.sft_launch_count.argtypes = [_c_i64p]
    L.sft_nccl_unique_id.argtypes = [ctypes.c_char_p]
    L.sft_plan_work.argtypes = [vp, _c_dp]
    L.sft_nccl_release.argtypes = [ctypes.c_char_p]
    _lib = L
    return L


def _check(rc):
    if rc != 0:
        L = lib()
        raise SftError(f"{L.sft_strerror(rc).decode()} ({rc}): {L.sft_last_error().decode()}")


def _ptr(a, dtype_np, out=False):
    """Return (pointer, keepalive) for a torch tensor or numpy array, contiguous, right dtype.
    Inputs are converted if needed; an output buffer (out=True) must already be
    contiguous with the right dtype -- the library writes into it, so a converted
    temporary would silently drop the result."""
    try:
        import torch
        if isinstance(a, torch.Tensor):
            want = {np.float64: torch.float64, np.complex128: torch.complex128}[dtype_np]
            if a.dtype != want or not a.is_contiguous():
                if out:
                    raise ValueError(f"output buffer must be a contiguous {want} tensor (got {a.dtype}, "
                                     f"contiguous={a.is_contiguous()})")
                a = a.to(want).contiguous()
            return ctypes.c_void_p(a.data_ptr()), a
    except ImportError:  # pragma: no cover
        pass
    if out:
        if not (isinstance(a, np.ndarray) and a.dtype == dtype_np and a.flags.c_contiguous and a.flags.writeable):
            raise ValueError(f"output buffer must be a writeable C-contiguous {np.dtype(dtype_np)} array")
        return ctypes.c_void_p(a.ctypes.data), a
    a = np.ascontiguousarray(a, dtype=dtype_np)
    return ctypes.c_void_p(a.ctypes.data), a


def _stream_handle(stream):
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        except ImportError:  # pragma: no cover
            pass
        return ctypes.c_void_p(0)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


class Plan:
    """sft_plan / sft_apply / sft_destroy (include/sft.h)."""

    def __init__(self, dim, N, p, x, k, stream=None, rank=0, world=1, exchange_level=-1, split_k=-1, split_x=-1,
                 precision=0, adjoint=False, nccl_id=None):
        """precision 0: FP64 charges (default); 1: the FP32 variant (single GPU;
        f and u stay complex128 at the boundary, the level charges are complex64).
        adjoint=True: apply() computes v_j = sum_i exp(-2 pi i x_i.k_j/N) g_i
        (g on the x points, v on the k points).  nccl_id (128 bytes, from
        nccl_unique_id() on one rank, shared by all): apply() runs the whole
        sharded transform with the library's own NCCL collectives."""
        L = lib()
        o = _Opts()
        L.sft_default_opts(ctypes.byref(o))
        o.precision = int(precision)
        o.adjoint = 1 if adjoint else 0
        o.stream = _stream_handle(stream)
        o.rank, o.world = int(rank), int(world)
        o.exchange_level, o.split_k, o.split_x = int(exchange_level), int(split_k), int(split_x)
        self._nid = None
        if nccl_id is not None:
            if len(nccl_id) != 128:
                raise ValueError("nccl_id must be 128 bytes")
            self._nid = ctypes.create_string_buffer(bytes(nccl_id), 128)
            o.nccl_id = ctypes.cast(self._nid, ctypes.c_void_p)
        xp, self._x = _ptr(x, np.float64)
        kp, self._k = _ptr(k, np.float64)
        self.dim, self.N, self.p = int(dim), int(N), int(p)
        self.nx = int(self._x.shape[0]) if len(self._x.shape) else 0
        self.nk = int(self._k.shape[0]) if len(self._k.shape) else 0
        self.adjoint = bool(adjoint)
        self.world, self.rank = int(world), int(rank)
        self.L = int(N).bit_length() - 1
        h = ctypes.c_void_p()
        _check(L.sft_plan(self.dim, self.N, self.p, xp, self.nx, kp, self.nk, ctypes.byref(o), ctypes.byref(h)))
        self._h = h
        self._x = self._k = None  # the plan copied what it needs

    @classmethod
    def farfield(cls, dim, kappa, p, xhat, y, stream=None, precision=0, adjoint=False):
        """sft_farfield_plan: apply(F) = u_inf(xhat_i) = sum_j exp(-i kappa xhat_i.y_j) F_j
        (PAPER.md:82-96), xhat [nx, dim] unit directions, y [ny, dim] in [0,1]^dim.
        adjoint=True: apply(g) = sum_i exp(+i kappa xhat_i.y_j) g_i on the y points."""
        L = lib()
        o = _Opts()
        L.sft_default_opts(ctypes.byref(o))
        o.precision = int(precision)
        o.adjoint = 1 if adjoint else 0
        o.stream = _stream_handle(stream)
        xp, xk = _ptr(xhat, np.float64)
        yp, yk = _ptr(y, np.float64)
        nx, ny = int(xk.shape[0]), int(yk.shape[0])
        h = ctypes.c_void_p()
        _check(L.sft_farfield_plan(int(dim), float(kappa), int(p), xp, nx, yp, ny, ctypes.byref(o), ctypes.byref(h)))
        self = cls.__new__(cls)
        self._h = h
        self._x = self._k = None
        self.dim, self.p = int(dim), int(p)
        self.nx, self.nk = nx, ny
        self.adjoint = bool(adjoint)
        self.world, self.rank = 1, 0
        info = np.zeros(8)
        _check(L.sft_plan_stats(h, None, None, None, info.ctypes.data_as(_c_dp)))
        self.L = int(info[0])
        self.N = 1 << self.L
        self.kappa = float(kappa)
        return self

    # -- single GPU ---------------------------------------------------------
    def apply(self, f, u=None):
        """u = butterfly(f).  If ``u`` is None a buffer like ``f`` (device or host) is allocated."""
        fp, fk = _ptr(f, np.complex128)
        if u is None:
            u = self._like(fk, self.nk if self.adjoint else self.nx)
        up, uk = _ptr(u, np.complex128, out=True)
        _check(lib().sft_apply(self._h, fp, up))
        return uk

    def apply_batch(self, f, u=None):
        """sft_apply_batch: f [nrhs, n_in] complex128 (row r = one charge vector,
        rows contiguous), u [nrhs, n_out]; one launch per step for all rows."""
        fp, fk = _ptr(f, np.complex128)
        if len(fk.shape) != 2:
            raise ValueError("apply_batch: f must be 2-D [nrhs, n]")
        nrhs, ldf = int(fk.shape[0]), int(fk.shape[1])
        nout = self.nk if self.adjoint else self.nx
        if u is None:
            u = self._like(fk, nrhs * nout).reshape(nrhs, nout)
        up, uk = _ptr(u, np.complex128, out=True)
        if tuple(uk.shape) != (nrhs, nout):
            raise ValueError("apply_batch: u must be [nrhs, n_out]")
        _check(lib().sft_apply_batch(self._h, nrhs, fp, ldf, up, nout))
        return uk

    @staticmethod
    def _like(ref, n):
        try:
            import torch
            if isinstance(ref, torch.Tensor):
                return torch.empty(n, dtype=torch.complex128, device=ref.device,
                                   pin_memory=(ref.device.type == "cpu" and ref.is_pinned()))
        except ImportError:  # pragma: no cover
            pass
        return np.empty(n, dtype=np.complex128)

    # -- multi GPU (see paper_0801_1524_b200.dist) ---------------------------
    def exchange_counts(self):
        s = np.zeros(self.world, np.int64)
        r = np.zeros(self.world, np.int64)
        _check(lib().sft_exchange_counts(self._h, s.ctypes.data_as(_c_i64p), r.ctypes.data_as(_c_i64p)))
        return s, r

    def partition(self):
        out = np.zeros(3 + 4 * self.world, np.int64)
        _check(lib().sft_partition_info(self._h, out.ctypes.data_as(_c_i64p)))
        return out

    def apply_phase1(self, f, sendbuf=None):
        """sendbuf None: fused exchange (set_peer_buffers first)."""
        fp, fk = _ptr(f, np.complex128)
        if sendbuf is None or isinstance(sendbuf, int):
            sp = ctypes.c_void_p(sendbuf or 0)
        else:
            sp, _ = _ptr(sendbuf, np.complex128, out=True)
        _check(lib().sft_apply_phase1(self._h, fp, sp))

    def apply_phase2(self, recvbuf, u):
        if isinstance(recvbuf, int):
            rp = ctypes.c_void_p(recvbuf)
        else:
            rp, _ = _ptr(recvbuf, np.complex128)
        up, _ = _ptr(u, np.complex128, out=True)
        _check(lib().sft_apply_phase2(self._h, rp, up))

    def set_peer_buffers(self, ptrs):
        """Fused exchange: ptrs[world] = device addresses (ints) of every rank's
        receive buffer as mapped in this process; None switches it off."""
        if ptrs is None:
            _check(lib().sft_set_peer_buffers(self._h, None))
            return
        arr = (ctypes.c_void_p * self.world)(*[int(q) for q in ptrs])
        _check(lib().sft_set_peer_buffers(self._h, arr))

    def peer_offsets(self):
        out = np.zeros(self.world, np.int64)
        _check(lib().sft_peer_offsets(self._h, out.ctypes.data_as(_c_i64p)))
        return out

    # -- stats / timing -------------------------------------------------------
    def stats(self):
        n = self.L + 1
        cx = np.zeros(n, np.int64); ck = np.zeros(n, np.int64); pr = np.zeros(n, np.int64)
        info = np.zeros(8)
        _check(lib().sft_plan_stats(self._h, cx.ctypes.data_as(_c_i64p), ck.ctypes.data_as(_c_i64p),
                                    pr.ctypes.data_as(_c_i64p), info.ctypes.data_as(_c_dp)))
        keys = ["L", "pd", "nx", "nk", "level_buffer_bytes", "plan_ms", "groups", "trans_alg_bytes"]
        d = dict(zip(keys, info.tolist()))
        d.update(counts_x=cx, counts_k=ck, pairs=pr)
        nl = ctypes.c_int(0)
        lv = (ctypes.c_int * max(1, self.L))()
        f2 = (ctypes.c_int * max(1, self.L))()
        _check(lib().sft_translation_launches(self._h, ctypes.byref(nl), lv, f2))
        d.update(launches=[(int(lv[i]), bool(f2[i])) for i in range(nl.value)])
        return d

    def work(self):
        """sft_plan_work: work model of one apply's translation step."""
        w = np.zeros(6)
        _check(lib().sft_plan_work(self._h, w.ctypes.data_as(_c_dp)))
        return dict(alg_bytes=w[0], fp64_flops=w[1], supertiles=w[2], tasks=w[3], groups=w[4], pairs=w[5])

    def set_timing(self, on=True):
        """on: False / True (events around every launch) / 2 (events around the
        translation chain only: per-level times not recorded)."""
        _check(lib().sft_set_timing(self._h, int(on) if on in (0, 1, 2) else 1))

    def last_timing(self):
        t = np.zeros(4); lv = np.zeros(max(self.L, 1))
        _check(lib().sft_last_timing(self._h, t.ctypes.data_as(_c_dp), lv.ctypes.data_as(_c_dp)))
        return dict(leaf_ms=t[0], trans_ms=t[1], final_ms=t[2], apply_ms=t[3], level_ms=lv[: self.L])

    def close(self):
        if getattr(self, "_h", None):
            lib().sft_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def device_alloc(nbytes: int) -> int:
    """cudaMalloc'd device memory (IPC-shareable, unlike the stream-ordered pool)."""
    p = ctypes.c_void_p()
    _check(lib().sft_device_alloc(int(nbytes), ctypes.byref(p)))
    return int(p.value)


def device_free(ptr: int) -> None:
    _check(lib().sft_device_free(ctypes.c_void_p(ptr)))


def ipc_handle(ptr: int) -> bytes:
    buf = ctypes.create_string_buffer(64)
    _check(lib().sft_ipc_handle(ctypes.c_void_p(ptr), buf))
    return buf.raw


def ipc_open(handle: bytes) -> int:
    p = ctypes.c_void_p()
    _check(lib().sft_ipc_open(ctypes.c_char_p(handle), ctypes.byref(p)))
    return int(p.value)


def ipc_close(ptr: int) -> None:
    _check(lib().sft_ipc_close(ctypes.c_void_p(ptr)))


def nccl_unique_id() -> bytes:
    """sft_nccl_unique_id: a fresh 128-byte ncclUniqueId (call on one rank, share with all)."""
    buf = ctypes.create_string_buffer(128)
    _check(lib().sft_nccl_unique_id(buf))
    return buf.raw


def nccl_release(nccl_id: bytes) -> None:
    """sft_nccl_release: destroy this process's communicators of that id."""
    _check(lib().sft_nccl_release(ctypes.create_string_buffer(bytes(nccl_id), 128)))


def launch_count() -> int:
    """Kernels launched by libsft so far (own kernels, CUB sort/scan excluded)."""
    v = np.zeros(1, np.int64)
    _check(lib().sft_launch_count(v.ctypes.data_as(_c_i64p)))
    return int(v[0])


def operator_tables(p, real=False):
    """Host-only: (V [2,2,p,p] complex128, invD [p]) -- and with real=True also
    (RC, RS) [2,p,p] float64, exactly as uploaded to the GPU's constant bank."""
    V = np.zeros(2 * 4 * p * p)
    invD = np.zeros(p)
    RC = np.zeros(2 * p * p)
    RS = np.zeros(2 * p * p)
    _check(lib().sft_operator_tables(p, V.ctypes.data_as(_c_dp), invD.ctypes.data_as(_c_dp),
                                     RC.ctypes.data_as(_c_dp), RS.ctypes.data_as(_c_dp)))
    V = V.view(np.complex128).reshape(2, 2, p, p)
    if real:
        return V, invD, RC.reshape(2, p, p), RS.reshape(2, p, p)
    return V, invD


def choose_partition(L, world, counts_x, counts_k, parents_x, parents_k, force=(-1, -1, -1)):
    """Host-only partitioner (sft_choose_partition).  parents_*[l] int32 arrays for l=1..L
    (index 0 ignored).  Returns (s_K, s_X, m, ranges [world,4], cost [3])."""
    cx = np.ascontiguousarray(counts_x, np.int64)
    ck = np.ascontiguousarray(counts_k, np.int64)
    keep = []

    def parr(ps):
        arr = (ctypes.POINTER(ctypes.c_int32) * (L + 1))()
        for l in range(1, L + 1):
            a = np.ascontiguousarray(ps[l], np.int32)
            keep.append(a)
            arr[l] = a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        return arr

    out = np.zeros(3 + 4 * world, np.int64)
    cost = np.zeros(3, np.int64)
    _check(lib().sft_choose_partition(L, world, cx.ctypes.data_as(_c_i64p), ck.ctypes.data_as(_c_i64p),
                                      parr(parents_x), parr(parents_k), force[0], force[1], force[2],
                                      out.ctypes.data_as(_c_i64p), cost.ctypes.data_as(_c_i64p)))
    return int(out[0]), int(out[1]), int(out[2]), out[3:].reshape(world, 4), cost
