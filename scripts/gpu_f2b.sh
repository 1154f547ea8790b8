cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m "gpu and not slow" -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in C0 C1 C2; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --nrhs 1 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
