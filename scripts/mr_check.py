"""Multi-rank emulation vs single plan, repeated: prints mismatch counts."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402

import synth  # noqa: E402
from test_gpu_multirank import emulate, single  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
world = int(sys.argv[2]) if len(sys.argv) > 2 else 2
w = synth.make_workload(name)
u1 = single(w)
for i in range(3):
    uw, part = emulate(w, world)
    bad = np.nonzero(uw != u1)[0]
    print(i, "part", part[:3].tolist(), "mismatch", len(bad), "max", float(np.max(np.abs(uw - u1))) if len(bad) else 0.0,
          "first", bad[:5].tolist())
