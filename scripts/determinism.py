"""Run plan+apply several times on one config and report bitwise differences."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0801_1524_b200 as sft  # noqa: E402
import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
w = synth.make_workload(name)
x = torch.from_numpy(w.x).cuda(); k = torch.from_numpy(w.k).cuda(); f = torch.from_numpy(w.f).cuda()
ref = None
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 5):
    with sft.Plan(w.dim, w.N, w.p, x, k) as pl:
        u = pl.apply(f).cpu().numpy()
        u2 = pl.apply(f).cpu().numpy()
    if ref is None:
        ref = u
    print(i, "plan-vs-first diff:", int(np.sum(u != ref)), "apply-vs-apply diff:", int(np.sum(u != u2)),
          "max |d|:", float(np.max(np.abs(u - ref))))
