# compute-sanitizer over the hot path: memcheck on C0-C3 (plan + apply), smoke, the batch / farfield /
# multirank test files; synccheck and initcheck on C0, C1, C3.  Tails go to gpurun_out/san/.
cd $GRAFT_REPO_ROOT
O=gpurun_out/san; mkdir -p $O
CS="compute-sanitizer --error-exitcode 99 --print-limit 20"
for c in C0 C1 C3 C2; do
  timeout 400 $CS --tool memcheck python scripts/run_config.py --config $c --reps 1 > $O/memcheck_$c.log 2>&1; echo "rc=$?" >> $O/memcheck_$c.log
done
timeout 300 $CS --tool memcheck python -c "import __graft_entry__ as g; g.smoke()" > $O/memcheck_smoke.log 2>&1; echo "rc=$?" >> $O/memcheck_smoke.log
for c in C0 C1 C3; do
  timeout 300 $CS --tool synccheck python scripts/run_config.py --config $c --reps 1 > $O/synccheck_$c.log 2>&1; echo "rc=$?" >> $O/synccheck_$c.log
  timeout 300 $CS --tool initcheck python scripts/run_config.py --config $c --reps 1 > $O/initcheck_$c.log 2>&1; echo "rc=$?" >> $O/initcheck_$c.log
done
timeout 600 $CS --tool memcheck python -m pytest tests/test_gpu_batch.py tests/test_gpu_farfield.py -q -m gpu -x -p no:cacheprovider > $O/memcheck_pytest_batch_ff.log 2>&1; echo "rc=$?" >> $O/memcheck_pytest_batch_ff.log
timeout 600 $CS --tool memcheck python -m pytest tests/test_gpu_multirank.py -q -m gpu -x -p no:cacheprovider -k "not C2" > $O/memcheck_pytest_mr.log 2>&1; echo "rc=$?" >> $O/memcheck_pytest_mr.log
for f in $O/*.log; do echo "== $f"; tail -4 $f; done
