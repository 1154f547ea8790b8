#!/bin/bash
# bench lines for every config + ncu --set full of one C2 translation level (t=7)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 11; }
for c in C0 C1 C2 C3 C4; do
  timeout 900 python bench.py --no-cpu-baseline --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python -c "import json;d=json.load(open('gpurun_out/bench_$c.json'));r=d['roofline'];print('$c',d['value'],d['ms_per_step'],d['apply_ms'],d['plan_ms'],r['frac'],r['kernel_ms']['translate_total'],d.get('batch',{}).get('apply_ms_per_rhs'))" || tail -3 gpurun_out/bench_$c.err
done
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name regex:k_translate_ws --launch-skip 6 --launch-count 1 -o gpurun_out/trans_c2 -f python scripts/run_config.py --config C2 --reps 1 > gpurun_out/ncu_full.log 2>&1; tail -2 gpurun_out/ncu_full.log
