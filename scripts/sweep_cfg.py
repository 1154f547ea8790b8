"""Time the translation kernels of one config with a given libsft build (SFT_LIB env)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0801_1524_b200 as sft  # noqa: E402
import synth  # noqa: E402

name = sys.argv[1]
w = synth.make_workload(name, p=int(os.environ['SWEEP_P']) if os.environ.get('SWEEP_P') else None)
x = torch.from_numpy(w.x).cuda(); k = torch.from_numpy(w.k).cuda(); f = torch.from_numpy(w.f).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
with sft.Plan(w.dim, w.N, w.p, x, k, precision=int(os.environ.get('SWEEP_PREC', '0'))) as pl:
    pl.set_timing(True)
    ts = []
    for i in range(8):
        flush.zero_()
        u = pl.apply(f)
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(pl.last_timing())
    st = pl.stats()
tr = float(np.median([t["trans_ms"] for t in ts]))
ap = float(np.median([t["apply_ms"] for t in ts]))
lf = float(np.median([t["leaf_ms"] for t in ts]))
fi = float(np.median([t["final_ms"] for t in ts]))
print(json.dumps({"lib": os.path.basename(os.environ.get("SFT_LIB", "default")), "cfg": name, "trans_ms": round(tr, 4),
                  "apply_ms": round(ap, 4), "leaf_ms": round(lf, 4), "final_ms": round(fi, 4), "GBps": round(st["trans_alg_bytes"] / tr / 1e6, 1),
                  "checksum": float(u.abs().sum())}))
