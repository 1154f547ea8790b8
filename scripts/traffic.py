"""From an ncu CSV of dram bytes per translate launch, write profiles/traffic_<cfg>.json.

usage: python scripts/traffic.py ncu_traffic.csv C2 [alg_bytes_per_launch]
"""
import csv
import json
import sys

path, cfg = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(path)))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi, ui, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("ID")
per = {}
for r in rows[hdr + 1:]:
    if len(r) <= vi or "k_translate" not in r[ki]:
        continue
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r[ui], 1)
    per.setdefault(r[idi], 0.0)
    per[r[idi]] += float(r[vi].replace(",", "")) * scale
vals = list(per.values())
out = {"config": cfg, "launches": len(vals), "dram_bytes_per_launch": sum(vals) / max(1, len(vals)),
       "dram_bytes_total": sum(vals), "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum ({path})"}
if len(sys.argv) > 3:
    out["alg_bytes_per_launch"] = float(sys.argv[3])
json.dump(out, open(f"profiles/traffic_{cfg}.json", "w"), indent=1)
print(json.dumps(out))
