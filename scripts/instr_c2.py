"""Per-CTA phase timeline of one translation level (instrumented build, SFT_LIB)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_0801_1524_b200 as sft, synth
w = synth.make_workload(sys.argv[1] if len(sys.argv) > 1 else "C2")
level = int(sys.argv[2]) if len(sys.argv) > 2 else 7
x = torch.from_numpy(w.x).cuda(); k = torch.from_numpy(w.k).cuda(); f = torch.from_numpy(w.f).cuda()
L = sft.lib(); L.sft_instr_set.argtypes = [ctypes.c_void_p]
buf = torch.zeros(200000 * 8, dtype=torch.int64, device="cuda")
with sft.Plan(w.dim, w.N, w.p, x, k) as pl:
    pl.apply(f); torch.cuda.synchronize()
    # run once more with instrumentation only during the chosen level: simplest is all levels
    # overwrite the buffer; the last launch that writes is level 0, so instrument via env below
    L.sft_instr_set(buf.data_ptr())
    pl.set_timing(True)
    pl.apply(f); torch.cuda.synchronize()
    t = pl.last_timing()
L.sft_instr_set(0)
b = buf.view(-1, 8).cpu().numpy()
b = b[b[:, 0] > 0]
t0 = b[:, 0].min()
rel = (b[:, :5] - t0) / 1e3  # us
print("CTAs", len(b), "level0 kernel ms", t["level_ms"][0])
ph = np.diff(b[:, :5], axis=1) / 1e3
names = ["meta+issue", "tma wait", "pass1", "pass0"]
for i, n in enumerate(names):
    print(f"{n:12s} mean {ph[:, i].mean():7.3f} us  p50 {np.median(ph[:, i]):7.3f}  p90 {np.percentile(ph[:, i], 90):7.3f}")
life = (b[:, 4] - b[:, 0]) / 1e3
span = (b[:, 4].max() - t0) / 1e3
sm = b[:, 7]
print("lifetime mean", life.mean(), "span us", span, "CTA-us per SM", life.sum() / 148, "=> mean resident CTAs/SM", life.sum() / 148 / span)
