cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SFT_ML=1 timeout 1200 python -m pytest tests -x -q -m "gpu and not slow" -p no:cacheprovider -k "parity or batch or farfield" > gpurun_out/pytest_ml.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_ml.log
: > gpurun_out/ml.txt
for rep in 1 2; do for c in C0 C1 C2 C3; do for m in 0 1; do echo "ML=$m $(SFT_ML=$m timeout 300 python scripts/sweep_cfg.py $c 2>&1 | tail -1)" >> gpurun_out/ml.txt; done; done; done
for c in C0 C1 C2 C3; do for m in 0 1; do SFT_ML=$m timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --nrhs 1 > gpurun_out/bench_ml${m}_$c.json 2> gpurun_out/bench_ml${m}_$c.err; done; done
