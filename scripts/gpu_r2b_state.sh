# Re-entry check of the current head: GPU tests, default bench line, per-config lines.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2b
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=15 > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err
for c in C0 C1 C3 C4; do timeout 900 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
