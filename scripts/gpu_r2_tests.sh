cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
nproc > gpurun_out/nproc.txt; lscpu | grep "Model name" >> gpurun_out/nproc.txt
timeout 2400 python -m pytest tests -x -q -m "gpu" -p no:cacheprovider --durations=25 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
for c in C3 C4; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --nrhs 1 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:k_translate_ws --launch-skip 3 --launch-count 1 -o gpurun_out/trans_c3 -f python scripts/run_config.py --config C3 --reps 1 > gpurun_out/ncu_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:k_translate_ws --launch-skip 4 --launch-count 1 -o gpurun_out/trans_c4 -f python scripts/run_config.py --config C4 --reps 1 > gpurun_out/ncu_c4.log 2>&1
