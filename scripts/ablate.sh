#!/bin/bash
# Build ablation variants of libsft and time the translation of C2 with each.
mkdir -p gpurun_out
python - <<'PY'
from paper_0801_1524_b200 import build as b
import os
for tag, flags in [("noload", ["-DSFT_ABL_NOLOAD"]), ("nocompute", ["-DSFT_ABL_NOCOMPUTE"]), ("noboth", ["-DSFT_ABL_NOLOAD", "-DSFT_ABL_NOCOMPUTE"]), ("nostore", ["-DSFT_ABL_NOSTORE"]), ("none", ["-DSFT_ABL_NOLOAD", "-DSFT_ABL_NOCOMPUTE", "-DSFT_ABL_NOSTORE"])]:
    b.build(extra=flags, out=os.path.join(b.HERE, f"libsft_{tag}.so"))
PY
for mode in ${MODES:-mma1}; do
for tag in ${TAGS:-base noload nocompute noboth nostore none}; do
  lib=paper_0801_1524_b200/libsft_$tag.so; [ $tag = base ] && lib=paper_0801_1524_b200/libsft.so
  SFT_LIB=$(pwd)/$lib SFT_TRANSLATE=$mode timeout 300 python bench.py --no-cpu-baseline --steps 5 ${BENCH_ARGS} > gpurun_out/abl_$tag.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/abl_$tag.json'));r=d['roofline'];print('$mode $tag',r['kernel_ms']['translate_total'],r['level_ms'])"
done; done
