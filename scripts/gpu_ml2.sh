cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SFT_ML=1 timeout 1200 python -m pytest tests -x -q -m "gpu and not slow" -p no:cacheprovider -k "parity_2d or parity_3d or uniform" > gpurun_out/pytest_ml.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_ml.log
for c in C0 C1 C2 C3; do for m in 0 1; do SFT_ML=$m timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --nrhs 1 > gpurun_out/bench_ml${m}_$c.json 2> gpurun_out/bench_ml${m}_$c.err; done; done
