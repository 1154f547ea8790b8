#!/bin/bash
# Summaries of a gpu_r2*_evidence run into profiles/ (tag = run dir name, e.g. r2d)
T=${1:-r2d}; O=gpurun_out/$T
for c in C0 C1 C3 C4; do cp $O/bench_$c.json profiles/${T}_bench_$c.json; done
cp $O/bench.json profiles/${T}_bench_C2.json
cp $O/bench_C2_f32.json profiles/${T}_bench_C2_f32.json
cp $O/bench_ref.json profiles/${T}_bench_reference_C2.json
python scripts/launch_summary.py $O/launches_C2.csv "$T: ncu launch list of python bench.py --steps 2 --warmup 3 --no-cpu-baseline --nrhs 1 (C2)" > profiles/${T}_launches_C2.txt
for c in c2 c3 c4; do python scripts/ncu_summary.py $O/trans_$c.ncu-rep profiles/${T}_${c}_translate.txt "$T: k_translate_ws, ${c^^} (one level), ncu --set full"; done
for c in C2 C3 C4; do python scripts/traffic.py $O/traffic_$c.csv $c > /dev/null; done
python scripts/sass_hist.py profiles/${T}_sass_hist.txt > /dev/null 2>&1
tail -3 $O/pytest_gpu.log > profiles/${T}_gputest_tail.txt
