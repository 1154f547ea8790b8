cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -p no:cacheprovider -k "two_level" > gpurun_out/pytest_f2.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_f2.log
for c in C0 C1 C2; do for m in 0 first all; do SFT_F2=$m timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --nrhs 1 > gpurun_out/bench_f2${m}_$c.json 2> gpurun_out/bench_f2${m}_$c.err; done; done
