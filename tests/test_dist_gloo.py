"""World-size-2 test of the multi-GPU orchestration (paper_0801_1524_b200.dist)
on CPU with the gloo backend.

The CUDA phases are replaced by a host stand-in that follows the documented
exchange layout (include/sft.h) with the partition chosen by the
library's own host partitioner: phase 1 tags every level-m pair (A, B) it owns
with (iB, iA); the real all_to_all_single + all_reduce of DistPlan run over
gloo; phase 2 checks that it received exactly the pairs of its T_X subtrees
in global [iB][iA_local] order.  The kernels' side of the same layout is
covered bit for bit on the GPU by tests/test_gpu_multirank.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth

sft = pytest.importorskip("paper_0801_1524_b200")
from paper_0801_1524_b200.dist import DistPlan, exchange_layout  # noqa: E402

PD = 3  # complex elements per pair in the stand-in


def tree_levels(pts, N, d):
    L = N.bit_length() - 1
    leaf = np.minimum(np.floor(pts).astype(np.int64), N - 1)
    key = np.zeros(len(pts), np.int64)
    for b in range(L - 1, -1, -1):
        for a in range(d):
            key = (key << 1) | ((leaf[:, a] >> b) & 1)
    keys = [np.unique(key >> (d * (L - l))) for l in range(L + 1)]
    parents = [None] + [np.searchsorted(keys[l - 1], keys[l] >> d).astype(np.int32) for l in range(1, L + 1)]
    return keys, parents, key


class HostPhases:
    """Stand-in for the CUDA phases, driven by the library's partitioner."""

    def __init__(self, w, rank, world, force):
        self.rank, self.world = rank, world
        self.nx = len(w.x)
        self.L = L = w.N.bit_length() - 1
        kx, px, self.xleafkey = tree_levels(w.x, w.N, w.dim)
        kk, pk, _ = tree_levels(w.k, w.N, w.dim)
        cx = [len(v) for v in kx]; ck = [len(v) for v in kk]
        self.lay = exchange_layout(cx, ck, px, pk, world, PD, force)
        self.kx, self.d = kx, w.dim
        self.nA = cx[L - self.lay["m"]]

    def exchange_counts(self):
        c = self.lay["counts"]
        return c[self.rank, :].copy(), c[:, self.rank].copy()

    def partition(self):
        return np.array([self.lay["sk"], self.lay["sx"], self.lay["m"]])

    def apply_phase1(self, f, sendbuf):
        b0, b1 = self.lay["b_rng"][self.rank]
        out = []
        for q in range(self.world):
            a0, a1 = self.lay["a_rng"][q]
            for iB in range(b0, b1):
                for iA in range(a0, a1):
                    out += [complex(iB, iA)] * PD
        if out:
            sendbuf[: len(out)] = torch.tensor(out, dtype=torch.complex128)

    def apply_phase2(self, recvbuf, u):
        a0, a1 = self.lay["a_rng"][self.rank]
        nB = sum(b1 - b0 for b0, b1 in self.lay["b_rng"])
        exp = [complex(iB, iA) for iB in range(nB) for iA in range(a0, a1) for _ in range(PD)]
        got = recvbuf[: len(exp)].numpy()
        assert np.array_equal(got, np.array(exp, dtype=np.complex128)), "exchange layout mismatch"
        # targets owned: leaf ancestor at level L-m inside [a0, a1)
        m, L, d = self.lay["m"], self.L, self.d
        anc = np.searchsorted(self.kx[L - m], self.xleafkey >> (d * m))
        own = (anc >= a0) & (anc < a1)
        u.zero_()
        u[torch.from_numpy(own)] = torch.from_numpy((np.arange(self.nx) + 0.5j)[own])

    def close(self):
        pass


def _worker(rank, world, port, name, force, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = synth.make_workload(name)
        plan = HostPhases(w, rank, world, force)
        dp = DistPlan(w.dim, w.N, w.p, None, None, plan=plan, device="cpu")
        u = dp.apply(torch.zeros(len(w.k), dtype=torch.complex128))
        ok = np.array_equal(u.numpy(), np.arange(len(w.x)) + 0.5j)
        q.put((rank, ok, tuple(int(v) for v in plan.partition())))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e), None))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("name,force", [("C1", (-1, -1, -1)), ("C1", (1, 2, 4)), ("C0", (0, 0, 6)), ("C0", (0, 1, 0))])
def test_dist_world2_gloo(name, force):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, force, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, part in res:
        assert ok is True, (rank, ok)
    parts = {r[2] for r in res}
    assert len(parts) == 1  # both ranks chose the same (s_K, s_X, m)


def _id_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_0801_1524_b200.dist import nccl_id_for
        a = nccl_id_for()
        b = nccl_id_for()  # cached: one communicator id per process group
        q.put((rank, a, a is b))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e), False))
    finally:
        dist.destroy_process_group()


def test_nccl_id_broadcast_gloo():
    """DistPlan(exchange="nccl") plumbing: rank 0 makes the ncclUniqueId with
    sft_nccl_unique_id (host call, no GPU needed) and torch.distributed
    broadcasts it once per process group; every rank holds the same 128 bytes."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_id_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(isinstance(r[1], bytes) and len(r[1]) == 128 for r in res), res
    assert res[0][1] == res[1][1]
    assert all(r[2] for r in res)
