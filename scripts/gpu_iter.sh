#!/bin/bash
# build, gpu tests, bench (mma + fma), one ncu --set full capture of a mid-level translate launch
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 11; }
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log; cat gpurun_out/pytest_gpu.log
for mode in ${MODES:-mma fma}; do
  SFT_TRANSLATE=$mode timeout 600 python bench.py --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_$mode.json 2> gpurun_out/bench_$mode.err; tail -2 gpurun_out/bench_$mode.err
  python -c "import json;d=json.load(open('gpurun_out/bench_$mode.json'));r=d['roofline'];print('$mode',d['value'],d['ms_per_step'],d['apply_ms'],d['plan_ms'],r['frac'],r['kernel_ms'],r['level_ms'])"
done
KREGEX=${KREGEX:-k_translate_mma}
timeout 600 ncu --set full --import-source on --clock-control none -k regex:$KREGEX --launch-skip ${NCU_SKIP:-10} --launch-count 1 -f -o gpurun_out/trans python scripts/run_config.py --config ${NCU_CONFIG:-C2} > gpurun_out/ncu_full.log 2>&1; tail -2 gpurun_out/ncu_full.log
