"""Dump the tile schedules of a multi-rank emulation (world W) to an .npz (for diffing libs)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_0801_1524_b200 as sft, synth
w = synth.make_workload(sys.argv[1]); world = int(sys.argv[2]); out = sys.argv[3]
L = sft.lib(); L.sft_schedule_bytes.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_int64), ctypes.c_void_p]
x = torch.from_numpy(w.x).cuda(); k = torch.from_numpy(w.k).cuda()
res = {}
for r in range(world):
    pl = sft.Plan(w.dim, w.N, w.p, x, k, rank=r, world=world) if world > 1 else sft.Plan(w.dim, w.N, w.p, x, k)
    for t in range(w.N.bit_length() - 1):
        n = ctypes.c_int64(0)
        L.sft_schedule_bytes(pl._h, t, ctypes.byref(n), None)
        buf = np.zeros(n.value, dtype=np.uint8)
        if n.value:
            L.sft_schedule_bytes(pl._h, t, ctypes.byref(n), buf.ctypes.data)
        res[f"r{r}_t{t}"] = buf
    pl.close()
np.savez(out, **res)
print("saved", out, len(res))
