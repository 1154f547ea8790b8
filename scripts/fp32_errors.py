"""Measured error of the FP32 variant (opts.precision = 1) against the FP64
oracle butterfly and the direct sum on the FP32 test cases (tests/test_gpu_parity.py),
to set FP32_PARITY from data."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_0801_1524_b200 as sft  # noqa: E402
import synth  # noqa: E402

cases = [("C0", None, 5), ("C0", None, 7), ("C0", None, 9), ("C1", None, 7), ("C1", None, 9), ("C1", None, 5),
         ("C3", 16, 5), ("C3", 16, 7), ("C3", 16, 9), ("C3", 32, 7)]
worst = 0.0
for name, N, p in cases:
    w = synth.make_workload(name, N=N, p=p)
    x = torch.from_numpy(w.x).cuda(); k = torch.from_numpy(w.k).cuda(); f = torch.from_numpy(w.f).cuda()
    with sft.Plan(w.dim, w.N, p, x, k, precision=1) as pl:
        u = pl.apply(f).cpu().numpy()
    ub = oracle.butterfly(w.x, w.k, w.f, w.N, p)
    e = oracle.rel_l2(u, ub)
    m = float(np.max(np.abs(u - ub)) / np.sqrt(np.mean(np.abs(ub) ** 2)))
    worst = max(worst, e)
    print(f"{name} N={w.N} p={p}: rel_l2 vs FP64 oracle butterfly {e:.3e}, max_rel {m:.3e}", flush=True)
print(f"worst rel_l2 {worst:.3e}")
