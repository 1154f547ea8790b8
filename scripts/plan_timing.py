"""Plan-stage timing on one config: device time (events) and host wall time of sft_plan, over reps."""
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
s = torch.cuda.current_stream()
dev, host = [], []
for i in range(12):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(s)
    pl = sft.Plan(w.dim, w.N, w.p, x, k, stream=s)
    e1.record(s)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    pl.close()
    if i >= 2:
        dev.append(e0.elapsed_time(e1)); host.append((t1 - t0) * 1e3)
print(f"plan device ms median {np.median(dev):.4f}  host wall ms median {np.median(host):.4f}  stats plan_ms {pl.stats()['plan_ms'] if False else ''}")
