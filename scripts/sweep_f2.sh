#!/bin/bash
for f in sweep_libs/lib_*.so; do SFT_F2=1 SFT_LIB=$PWD/$f timeout 300 python scripts/sweep_cfg.py C2 2>&1 | tail -1 | cut -c1-120; done
SFT_F2=1 python scripts/sweep_cfg.py C2 | cut -c1-120
python - <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np, synth, paper_0801_1524_b200 as sft
w = synth.make_workload("C2")
x = torch.from_numpy(w.x).cuda(); k = torch.from_numpy(w.k).cuda(); f = torch.from_numpy(w.f).cuda()
for env in ("0", "1"):
    os.environ["SFT_F2"] = env
with sft.Plan(2, w.N, w.p, x, k) as pl:
    pl.set_timing(True)
    for _ in range(5): pl.apply(f)
    torch.cuda.synchronize()
    t = pl.last_timing()
    print("launches", pl.stats()["launches"])
    print("level_ms", [round(v, 4) for v in t["level_ms"]])
PY
SFT_F2=0 python - <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np, synth, paper_0801_1524_b200 as sft
w = synth.make_workload("C2")
x = torch.from_numpy(w.x).cuda(); k = torch.from_numpy(w.k).cuda(); f = torch.from_numpy(w.f).cuda()
with sft.Plan(2, w.N, w.p, x, k) as pl:
    pl.set_timing(True)
    for _ in range(5): pl.apply(f)
    torch.cuda.synchronize()
    print("single level_ms", [round(v, 4) for v in pl.last_timing()["level_ms"]])
PY
