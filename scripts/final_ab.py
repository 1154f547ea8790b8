"""A/B of the final kernel variants (SFT_FINAL_STAGE in a subprocess each): final ms and bitwise equality."""
import os, subprocess, sys, json
code = r'''
import sys, os, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch, synth, paper_0801_1524_b200 as sft
w = synth.make_workload(sys.argv[1])
x = torch.from_numpy(w.x).cuda(); k = torch.from_numpy(w.k).cuda(); f = torch.from_numpy(w.f).cuda()
with sft.Plan(w.dim, w.N, w.p, x, k) as pl:
    pl.set_timing(True); ts = []
    for i in range(8):
        u = pl.apply(f); torch.cuda.synchronize()
        if i >= 3: ts.append(pl.last_timing()["final_ms"])
    np.save(sys.argv[2], u.cpu().numpy())
print(json.dumps({"final_ms": float(np.median(ts))}))
'''
for cfg in sys.argv[1:]:
    out = {}
    for m in ("0", "1"):
        path = f"/tmp/final_{cfg}_{m}.npy"
        r = subprocess.run([sys.executable, "-c", code, cfg, path], env=dict(os.environ, SFT_FINAL_STAGE=m),
                           capture_output=True, text=True)
        out[m] = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-500:]
    import numpy as np
    same = np.array_equal(np.load(f"/tmp/final_{cfg}_0.npy").view(np.uint64), np.load(f"/tmp/final_{cfg}_1.npy").view(np.uint64))
    print(cfg, out, "bitwise equal:", same)
