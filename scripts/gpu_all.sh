#!/bin/bash
# build, gpu tests, smoke, bench lines for every config (C2 with cpu_baseline), C2 launch list
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 11; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
for c in C0 C1 C3 C4; do timeout 900 python bench.py --no-cpu-baseline --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 600 python bench.py --no-cpu-baseline --precision f32 > gpurun_out/bench_C2_f32.json 2> gpurun_out/bench_f32.err
for c in C0 C1 C2 C3 C4 C2_f32; do python -c "import json;d=json.load(open('gpurun_out/bench_$c.json'));r=d['roofline'];print('$c',d['value'],d['ms_per_step'],d['apply_ms'],d['plan_ms'],d['e2e']['value'],r['frac'],r['kernel_ms']['translate_total'],d['clocks']['sm_mhz'],d.get('batch',{}).get('apply_ms_per_rhs'))"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --nrhs 1 > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?"
