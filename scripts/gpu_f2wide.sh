cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py -x -q -k "C0 or two_level or small or adjoint or single" -p no:cacheprovider > gpurun_out/pytest_f2w.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_f2w.log
for c in C0 C1; do timeout 600 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --no-configs --nrhs 1 > gpurun_out/bench_${c}_w.json 2> gpurun_out/bench_${c}_w.err; done
