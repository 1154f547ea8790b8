"""Timeline of one bench step (plan + apply + destroy) on a config: CUDA events
at the Python-level boundaries, host perf_counter, and SFT_PLAN_TRACE host
milestones inside sft_plan.  usage: SFT_PLAN_TRACE=1 python scripts/step_timeline.py C2"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0801_1524_b200 as sft  # noqa: E402
import synth  # noqa: E402

w = synth.make_workload(sys.argv[1] if len(sys.argv) > 1 else "C2")
x = torch.from_numpy(w.x).cuda(); k = torch.from_numpy(w.k).cuda(); f = torch.from_numpy(w.f).cuda()
u = torch.empty(len(w.x), dtype=torch.complex128, device="cuda")
s = torch.cuda.current_stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rows = []
for i in range(12):
    flush.zero_()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    h = [time.perf_counter()]
    ev[0].record(s)
    pl = sft.Plan(w.dim, w.N, w.p, x, k, stream=s)
    h.append(time.perf_counter()); ev[1].record(s)
    pl.apply(f, u)
    h.append(time.perf_counter()); ev[2].record(s)
    pl.close()
    h.append(time.perf_counter()); ev[3].record(s)
    torch.cuda.synchronize()
    if i >= 2:
        rows.append([ev[0].elapsed_time(ev[j]) for j in (1, 2, 3)] + [(h[j] - h[0]) * 1e3 for j in (1, 2, 3)])
r = np.median(np.array(rows), axis=0)
print(f"{w.name}: device ms at plan-return {r[0]:.4f} apply-return {r[1]:.4f} end {r[2]:.4f}; "
      f"host ms plan {r[3]:.4f} apply {r[4]:.4f} destroy {r[5]:.4f}", flush=True)
