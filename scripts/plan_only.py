"""Build a plan (and one apply) for one config: profiling driver for the plan stage."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0801_1524_b200 as sft  # noqa: E402
import synth  # noqa: E402

w = synth.make_workload(sys.argv[1] if len(sys.argv) > 1 else "C2")
x = torch.from_numpy(w.x).cuda(); k = torch.from_numpy(w.k).cuda(); f = torch.from_numpy(w.f).cuda()
for _ in range(3):
    with sft.Plan(w.dim, w.N, w.p, x, k) as pl:
        u = pl.apply(f)
torch.cuda.synchronize()
print("ok")
