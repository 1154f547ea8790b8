#!/bin/bash
# Build libsft variants from -D flag sets and time C2 (or $CFG) translate with each.
# usage: VARIANTS="name1:-DA=1 -DB=2;name2:-DC=3" bash scripts/variants.sh
mkdir -p gpurun_out
python - <<'PY'
import os
from concurrent.futures import ThreadPoolExecutor
from paper_0801_1524_b200 import build as b
vs = [v for v in os.environ["VARIANTS"].split(";") if v.strip()]
def one(v):
    name, flags = v.split(":", 1)
    b.build(extra=flags.split(), out=os.path.join(b.HERE, f"libsft_v_{name}.so"))
with ThreadPoolExecutor(4) as ex:
    list(ex.map(one, vs))
PY
IFS=';' read -ra VS <<< "$VARIANTS"
for v in "${VS[@]}"; do
  name=${v%%:*}
  SFT_LIB=$(pwd)/paper_0801_1524_b200/libsft_v_$name.so timeout 300 python scripts/sweep_cfg.py ${CFG:-C2} | sed "s/^/$name /"
done
