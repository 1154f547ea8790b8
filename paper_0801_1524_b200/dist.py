"""Multi-GPU butterfly: one process per GPU.

Phase 1 runs levels t = L..m over this rank's T_K subtrees (level s_K), the
level-m equivalent charges are redistributed to the owners of the T_X subtrees
(level s_X), phase 2 runs levels t = m-1..0 and the final evaluation for this
rank's targets, and every rank ends with the full u.  The per-pair arithmetic
does not depend on the partition, so u is bitwise equal to the 1-GPU result.

``exchange`` selects who moves the bytes:

* ``"nccl"`` (default): everything inside libsft -- the plan joins an NCCL
  communicator (``opts.nccl_id``; the id is made once per process group by
  rank 0 and broadcast over torch.distributed), and ``sft_apply`` runs phase 1,
  grouped ncclSend/ncclRecv, phase 2, ncclAllGather of u and the scatter to
  user order on the plan stream.
* ``"fused"``: the exchange level's kernel stores its outputs straight into
  the receivers' buffers (CUDA IPC mappings over NVLink); one stream-ordered
  all-reduce of a flag is the barrier before phase 2.
* ``"torch"``: the phase calls with torch.distributed collectives
  (all_to_all_single, then a sum all-reduce of u: every entry has exactly one
  non-zero contributor) -- used by the gloo tests with a host stand-in plan.

torch.distributed is plumbing only (process group, id broadcast); every
arithmetic step runs in libsft's kernels.
"""
from __future__ import annotations

import numpy as np

from . import Plan

_NCCL_IDS = {}  # process group -> ncclUniqueId bytes (one communicator per group)


def nccl_id_for(group=None) -> bytes:
    """The NCCL id of this process group: made by rank 0 with
    sft_nccl_unique_id and broadcast once; later plans reuse the library's
    cached communicator of that id."""
    import torch.distributed as dist
    key = id(group) if group is not None else None
    if key not in _NCCL_IDS:
        from . import nccl_unique_id
        obj = [nccl_unique_id() if dist.get_rank(group) == 0 else None]
        src = 0 if group is None else dist.get_global_rank(group, 0)
        dist.broadcast_object_list(obj, src=src, group=group)
        _NCCL_IDS[key] = obj[0]
    return _NCCL_IDS[key]


class DistPlan:
    """One rank of the sharded transform.  ``plan`` may be injected (tests use
    a host-side stand-in with a gloo group; that implies exchange="torch");
    by default it is a libsft plan with rank/world taken from the process
    group."""

    def __init__(self, dim, N, p, x, k, group=None, stream=None, exchange_level=-1, split_k=-1, split_x=-1,
                 plan=None, device=None, fused=False, exchange=None):
        import torch
        import torch.distributed as dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if exchange is None:
            exchange = "fused" if fused else ("torch" if plan is not None else "nccl")
        if exchange not in ("nccl", "fused", "torch"):
            raise ValueError(f"exchange must be nccl, fused or torch, not {exchange!r}")
        self.exchange = exchange
        if plan is None:
            nid = nccl_id_for(group) if exchange == "nccl" else None
            plan = Plan(dim, N, p, x, k, stream=stream, rank=self.rank, world=self.world,
                        exchange_level=exchange_level, split_k=split_k, split_x=split_x, nccl_id=nid)
        self.plan = plan
        self.nx = plan.nx
        if device is None:
            device = x.device if isinstance(x, torch.Tensor) and x.is_cuda else torch.device(
                "cuda", torch.cuda.current_device())
        self.device = torch.device(device)
        if exchange == "nccl":
            return
        s, r = plan.exchange_counts()
        self.send_counts = [int(v) for v in s]
        self.recv_counts = [int(v) for v in r]
        if exchange == "torch":
            self.sendbuf = torch.empty(max(1, sum(self.send_counts)), dtype=torch.complex128, device=self.device)
            self.recvbuf = torch.empty(max(1, sum(self.recv_counts)), dtype=torch.complex128, device=self.device)
        else:
            # fused exchange: every rank's receive buffer is mapped into every
            # process (CUDA IPC over NVLink); the exchange level's kernel stores
            # its outputs straight into the receivers' buffers
            from . import device_alloc, ipc_handle, ipc_open
            self._own = device_alloc(16 * max(1, sum(self.recv_counts)))
            handles = [None] * self.world
            dist.all_gather_object(handles, ipc_handle(self._own), group=group)
            self._peers = [self._own if q == self.rank else ipc_open(handles[q]) for q in range(self.world)]
            self.plan.set_peer_buffers(self._peers)
            self._flag = torch.zeros(1, dtype=torch.float32, device=self.device)

    def partition(self):
        return self.plan.partition()

    def apply(self, f, u=None):
        import torch
        import torch.distributed as dist
        if u is None:
            u = torch.empty(self.nx, dtype=torch.complex128, device=self.device)
        if self.exchange == "nccl":
            self.plan.apply(f, u)  # exchange and all-gather inside the library
            return u
        if self.exchange == "fused":
            self.plan.apply_phase1(f, None)
            # stream-ordered barrier: every rank's exchange-level kernel (and so
            # its peer stores into our buffer) precedes this collective
            dist.all_reduce(self._flag, group=self.group)
            self.plan.apply_phase2(self._own, u)
        else:
            self.plan.apply_phase1(f, self.sendbuf)
            # the level-m charge exchange; complex128 moved as (re, im) float64 pairs
            ns, nr = sum(self.send_counts), sum(self.recv_counts)
            dist.all_to_all_single(torch.view_as_real(self.recvbuf[:nr]).reshape(-1),
                                   torch.view_as_real(self.sendbuf[:ns]).reshape(-1),
                                   output_split_sizes=[2 * c for c in self.recv_counts],
                                   input_split_sizes=[2 * c for c in self.send_counts], group=self.group)
            self.plan.apply_phase2(self.recvbuf, u)
        # every target has exactly one non-zero contributor: the sum is exact
        dist.all_reduce(torch.view_as_real(u), op=dist.ReduceOp.SUM, group=self.group)
        return u

    def close(self):
        self.plan.close()
        if self.exchange == "fused" and getattr(self, "_peers", None):
            from . import device_free, ipc_close
            import torch
            torch.cuda.synchronize(self.device)
            for q, ptr in enumerate(self._peers):
                if q != self.rank:
                    ipc_close(ptr)
            device_free(self._own)
            self._peers = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def exchange_layout(counts_x, counts_k, parents_x, parents_k, world, pd, force=(-1, -1, -1)):
    """Host-side description of the level-m exchange that DistPlan performs,
    computed from the same partitioner the library uses (sft_choose_partition):
    returns dict with s_K, s_X, m, per-rank B ranges at level m, A ranges at
    level L-m, and send/recv element counts per (src, dst)."""
    from . import choose_partition
    L = len(counts_x) - 1
    sk, sx, m, rng, cost = choose_partition(L, world, counts_x, counts_k, parents_x, parents_k, force)

    def desc_range(parents, s, lo, hi, lev):
        """boxes at level `lev` whose ancestor at level s lies in [lo, hi)"""
        if lev == s:
            return int(lo), int(hi)
        a = np.asarray(parents[lev])          # ancestors at lev-1
        for l in range(lev - 1, s, -1):
            a = np.asarray(parents[l])[a]     # ... up to level s
        return int(np.searchsorted(a, lo)), int(np.searchsorted(a, hi))

    b_rng = [desc_range(parents_k, sk, rng[r, 0], rng[r, 1], m) for r in range(world)]
    a_rng = [desc_range(parents_x, sx, rng[r, 2], rng[r, 3], L - m) for r in range(world)]
    counts = np.zeros((world, world), np.int64)
    for src in range(world):
        for dst in range(world):
            counts[src, dst] = (b_rng[src][1] - b_rng[src][0]) * (a_rng[dst][1] - a_rng[dst][0]) * pd
    return dict(sk=sk, sx=sx, m=m, b_rng=b_rng, a_rng=a_rng, counts=counts, cost=cost)
