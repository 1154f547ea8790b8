"""Summarise gpurun_out/ab.txt (scripts/gpu_ab.sh): per (config, lib) translate / apply ms of each rep."""
import collections
import json
import sys

r = collections.defaultdict(list)
for line in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ab.txt"):
    try:
        d = json.loads(line)
    except ValueError:
        continue
    r[(d["cfg"], d["lib"])].append((d["trans_ms"], d["apply_ms"], d["checksum"]))
for k in sorted(r):
    print(k, r[k])
