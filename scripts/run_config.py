"""Run plan+apply on one BASELINE config a few times (profiling driver)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0801_1524_b200 as sft  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
w = synth.make_workload(a.config)
x = torch.from_numpy(w.x).cuda(); k = torch.from_numpy(w.k).cuda(); f = torch.from_numpy(w.f).cuda()
with sft.Plan(w.dim, w.N, w.p, x, k) as plan:
    for _ in range(a.reps):
        u = plan.apply(f)
torch.cuda.synchronize()
print("ok", a.config, float(u.abs().sum()))
