# chain-timed roofline: new tests, bench lines C2 (default) and C3/C4
cd $GRAFT_REPO_ROOT
O=gpurun_out/chain; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -p no:cacheprovider -k "dynamic or errors" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err
for c in C3 C4; do timeout 900 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
