"""Multi-rank path emulated on ONE GPU: every rank is an
independent plan (world=W, rank=r); phase 1 of all ranks runs, the
all-to-all is done with plain device copies in rank order, then phase 2 of
all ranks runs and the per-rank outputs are summed.  No kernel waits on
another rank, so this is safe on a single device.  The result must equal the
1-GPU sft_apply bit for bit (per-pair arithmetic is partition-independent)."""
import numpy as np
import pytest

import oracle
import synth
from helpers import assert_close

pytestmark = pytest.mark.gpu


def emulate(w, world, force=(-1, -1, -1), timing=False):
    import torch
    import paper_0801_1524_b200 as sft
    x = torch.from_numpy(w.x).cuda(); k = torch.from_numpy(w.k).cuda(); f = torch.from_numpy(w.f).cuda()
    plans = [sft.Plan(w.dim, w.N, w.p, x, k, rank=r, world=world, split_k=force[0], split_x=force[1],
                      exchange_level=force[2]) for r in range(world)]
    counts = [pl.exchange_counts() for pl in plans]
    parts = [pl.partition() for pl in plans]
    for pp in parts[1:]:
        assert np.array_equal(pp, parts[0])  # every rank derives the same partition
    if timing:
        for pl in plans:
            pl.set_timing(True)
    send = [torch.empty(max(1, int(c[0].sum())), dtype=torch.complex128, device="cuda") for c in counts]
    for r, pl in enumerate(plans):
        pl.apply_phase1(f, send[r])
    # all-to-all: recv[q] = concat_r send[r][segment q]
    recv = []
    for q in range(world):
        chunks = []
        for r in range(world):
            s = counts[r][0]
            off = int(s[:q].sum())
            chunks.append(send[r][off: off + int(s[q])])
            assert int(s[q]) == int(counts[q][1][r])  # sender/receiver agree on sizes
        recv.append(torch.cat(chunks) if chunks else torch.empty(1, dtype=torch.complex128, device="cuda"))
    u = torch.zeros(len(w.x), dtype=torch.complex128, device="cuda")
    for q, pl in enumerate(plans):
        uq = torch.empty(len(w.x), dtype=torch.complex128, device="cuda")
        pl.apply_phase2(recv[q] if recv[q].numel() else torch.empty(1, dtype=torch.complex128, device="cuda"), uq)
        u += uq
    torch.cuda.synchronize()
    if timing:  # per-rank translation time of both phases (bench.py's multi-GPU roofline)
        tms = [pl.last_timing()["trans_ms"] for pl in plans]
        assert all(t > 0 for t in tms), tms
    for pl in plans:
        pl.close()
    return u.cpu().numpy(), parts[0]


def single(w):
    import torch
    import paper_0801_1524_b200 as sft
    with sft.Plan(w.dim, w.N, w.p, torch.from_numpy(w.x).cuda(), torch.from_numpy(w.k).cuda()) as pl:
        u = pl.apply(torch.from_numpy(w.f).cuda())
    return u.cpu().numpy()


@pytest.mark.parametrize("name,world", [("C1", 2), ("C1", 4), ("C1", 8), ("C0", 2)])
def test_multirank_bitwise_2d(name, world):
    w = synth.make_workload(name)
    if world == 4:  # also exercise the phase timing (sft_set_timing on multi-rank plans)
        u, _ = emulate(w, world, timing=True)
        assert np.array_equal(u.view(np.uint64), single(w).view(np.uint64))
        return
    u1 = single(w)
    uw, part = emulate(w, world)
    assert np.array_equal(uw, u1), f"partition {part[:3]}"


@pytest.mark.parametrize("world", [2, 8])
def test_multirank_bitwise_3d(world):
    w = synth.make_workload("C3", N=32, p=5)
    u1 = single(w)
    uw, _ = emulate(w, world)
    assert np.array_equal(uw, u1)


@pytest.mark.parametrize("force", [(1, 1, 5), (2, 2, 2), (0, 0, 10), (1, 0, 10), (0, 3, 0)])
def test_multirank_forced_levels(force):
    """Every admissible (s_K, s_X, m), including the exchange at the leaf level
    (m = L) and at the root level (m = 0)."""
    w = synth.make_workload("C1")
    L = w.N.bit_length() - 1
    sk, sx, m = force
    if m == 10:
        m = L
    u1 = single(w)
    uw, part = emulate(w, 2, (sk, sx, m))
    assert tuple(part[:3]) == (sk, sx, m)
    assert np.array_equal(uw, u1)


def test_multirank_C2_vs_oracle():
    """C2 at full size sharded over 4 emulated ranks: bitwise equal to the
    single-GPU result on every target, and within parity of the oracle
    butterfly on every 4th of the 1024 seeded targets (spread over the whole
    circle, so every rank's T_X range is covered)."""
    w = synth.make_workload("C2")
    uw, part = emulate(w, 4)
    u1 = single(w)
    assert np.array_equal(uw.view(np.uint64), u1.view(np.uint64)), f"partition {part[:3]}"
    tg = w.sample[::4]
    ub = oracle.butterfly(w.x, w.k, w.f, w.N, w.p, targets=tg)
    assert_close(uw[tg], ub, 1e-10)


@pytest.mark.parametrize("name,force", [("C1", (1, 1, 5)), ("C1", (0, 0, 10)), ("C1", (0, 0, 0)), ("C3s", (1, 1, 2))])
def test_nccl_sharded_one_rank(name, force):
    """The in-library NCCL path (opts.nccl_id) on one GPU: world = 1 with an
    explicit exchange level runs phase 1, the grouped ncclSend/ncclRecv (to
    itself), phase 2 into the all-gather layout, ncclAllGather and the scatter
    to user order inside sft_apply -- bitwise equal to the plain apply."""
    import torch
    import paper_0801_1524_b200 as sft
    w = synth.make_workload("C3", N=32, p=5) if name == "C3s" else synth.make_workload(name)
    L = w.N.bit_length() - 1
    force = tuple(L if v == 10 else v for v in force)
    nid = sft.nccl_unique_id()
    x = torch.from_numpy(w.x).cuda(); k = torch.from_numpy(w.k).cuda(); f = torch.from_numpy(w.f).cuda()
    try:
        with sft.Plan(w.dim, w.N, w.p, x, k, rank=0, world=1, split_k=force[0], split_x=force[1],
                      exchange_level=force[2], nccl_id=nid) as pl:
            assert tuple(pl.partition()[:3]) == force
            u = pl.apply(f).cpu().numpy()
            uh = pl.apply(w.f)  # host in / host out through the same path
    finally:
        sft.nccl_release(nid)
    u1 = single(w)
    assert np.array_equal(u.view(np.uint64), u1.view(np.uint64))
    assert np.array_equal(uh.view(np.uint64), u1.view(np.uint64))


def emulate_fused(w, world, force=(-1, -1, -1)):
    """Fused exchange: each emulated rank's exchange-level kernel stores its
    level-m charges straight into the other ranks' receive buffers (here all on
    one device, standing in for the IPC-mapped peer buffers of a multi-GPU run);
    no send buffer and no all-to-all."""
    import torch
    import paper_0801_1524_b200 as sft
    x = torch.from_numpy(w.x).cuda(); k = torch.from_numpy(w.k).cuda(); f = torch.from_numpy(w.f).cuda()
    plans = [sft.Plan(w.dim, w.N, w.p, x, k, rank=r, world=world, split_k=force[0], split_x=force[1],
                      exchange_level=force[2]) for r in range(world)]
    counts = [pl.exchange_counts() for pl in plans]
    recv = [torch.full((max(1, int(c[1].sum())),), complex("nan"), dtype=torch.complex128, device="cuda")
            for c in counts]
    ptrs = [t.data_ptr() for t in recv]
    for r, pl in enumerate(plans):
        pl.set_peer_buffers(ptrs)
        offs = pl.peer_offsets()
        for q in range(world):  # this rank's segment in q's buffer starts after the lower ranks' segments
            assert int(offs[q]) == int(sum(counts[q][1][:r]))
    for pl in plans:
        pl.apply_phase1(f, None)
    torch.cuda.synchronize()
    u = torch.zeros(len(w.x), dtype=torch.complex128, device="cuda")
    for q, pl in enumerate(plans):
        uq = torch.empty(len(w.x), dtype=torch.complex128, device="cuda")
        pl.apply_phase2(recv[q], uq)
        u += uq
    torch.cuda.synchronize()
    for pl in plans:
        pl.close()
    return u.cpu().numpy()


@pytest.mark.parametrize("name,world,force", [("C1", 2, (-1, -1, -1)), ("C1", 4, (-1, -1, -1)),
                                              ("C0", 8, (-1, -1, -1)), ("C1", 2, (1, 0, 10)), ("C1", 2, (0, 3, 0))])
def test_fused_exchange_bitwise(name, world, force):
    w = synth.make_workload(name)
    L = w.N.bit_length() - 1
    force = tuple(L if v == 10 else v for v in force)
    u1 = single(w)
    uw = emulate_fused(w, world, force)
    assert np.array_equal(uw, u1)
