#!/bin/bash
# A/B: build/ab_old (a git worktree of an older commit, built locally) vs the working tree, same box
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 11; }
for i in 1 2; do
  for side in old new; do
    if [ $side = old ]; then d=build/ab_old; a=""; else d=.; a="--nrhs 1"; fi
    (cd $d && timeout 300 python bench.py --no-cpu-baseline --steps 20 ${AB_ARGS} $a 2>/dev/null) | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];print('$side',d['value'],'step',d['ms_per_step'],'apply',d['apply_ms'],'plan',d['plan_ms'],'trans',r['kernel_ms']['translate_total'])"
  done
done
