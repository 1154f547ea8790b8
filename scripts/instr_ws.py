"""Cycle accounting of the warp-specialised translation kernel (build with -DSFT_INSTR; SFT_LIB).

Sums clock64 intervals per CTA over all translation launches of one apply and
prints the mean per CTA (cycles) of: producer total / wait(empty) / build+issue,
consumer total / wait(full) / pass 1 / barrier / last pass (per consumer warp).
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0801_1524_b200 as sft  # noqa: E402
import synth  # noqa: E402

w = synth.make_workload(sys.argv[1] if len(sys.argv) > 1 else "C2")
x = torch.from_numpy(w.x).cuda(); k = torch.from_numpy(w.k).cuda(); f = torch.from_numpy(w.f).cuda()
L = sft.lib()
L.sft_instr_set.argtypes = [ctypes.c_void_p]
buf = torch.zeros(4096 * 8, dtype=torch.int64, device="cuda")
with sft.Plan(w.dim, w.N, w.p, x, k) as pl:
    pl.apply(f)
    torch.cuda.synchronize()
    L.sft_instr_set(buf.data_ptr())
    pl.set_timing(True)
    pl.apply(f)
    torch.cuda.synchronize()
    t = pl.last_timing()
    L.sft_instr_set(0)
b = buf.view(-1, 8).cpu().numpy().astype(np.float64)
b = b[b[:, 3] > 0]
nc = int(os.environ.get("NC", "4"))
names = ["prod total", "prod wait empty", "prod build+issue", "cons total", "cons wait full", "cons pass1",
         "cons barrier", "cons last pass"]
print(f"CTAs {len(b)}; translate ms {t['trans_ms']:.4f} ({t['trans_ms'] * 1.965e6:.0f} cycles at 1.965 GHz)")
for i, n in enumerate(names):
    div = nc if i >= 3 else 1
    print(f"  {n:18s} {b[:, i].mean() / div:12.0f} cycles per CTA{' (per consumer warp)' if i >= 3 else ''}")
