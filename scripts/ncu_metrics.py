"""Print selected raw metrics of an ncu report: python scripts/ncu_metrics.py REP [substr ...]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
keys = sys.argv[2:] or ["dmma", "pipe_fp64_cycles", "pipe_tensor_cycles", "inst_executed_pipe_xu", "issue_active",
                        "warps_active.avg.pct", "dram__throughput.avg.pct", "gpu__time_duration.sum",
                        "smsp__inst_executed.sum ", "achieved_occupancy", "sm__cycles_elapsed.avg "]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, u = rows[0], rows[1]
for v in rows[2:]:
    print("#", v[h.index("Kernel Name")][:80])
    for i, name in enumerate(h):
        if any(k in name + " " for k in keys):
            print(f"  {name:90s} {u[i]:8s} {v[i]}")
