#!/bin/bash
# build, full gpu tests, bench (C2 default + batch)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 11; }
timeout 300 python -m pytest tests/test_gpu_batch.py -x -q > gpurun_out/pytest_batch.log 2>&1; tail -15 gpurun_out/pytest_batch.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --nrhs 8 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
python -c "import json;d=json.load(open('gpurun_out/bench.json'));r=d['roofline'];print(d['value'],d['ms_per_step'],d['apply_ms'],d['plan_ms'],r['frac'],r['kernel_ms']);print(d.get('batch'))"
for c in C1 C3; do timeout 600 python bench.py --no-cpu-baseline --config $c --nrhs 8 > gpurun_out/bench_$c.json 2>>gpurun_out/bench.err; python -c "import json;d=json.load(open('gpurun_out/bench_$c.json'));print('$c',d['value'],d['apply_ms'],d.get('batch'))"; done
