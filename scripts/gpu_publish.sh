# plan header published by a kernel into pinned memory vs D2H copy + sync: tests + A/B
cd $GRAFT_REPO_ROOT
O=gpurun_out/pub; mkdir -p $O
timeout 1200 python -m pytest tests -q -x -m gpu -p no:cacheprovider -k "errors or tree or sort or small or extreme or dynamic or multirank or nccl or farfield" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for rep in 1 2; do for c in C0 C1 C2; do
  timeout 300 python scripts/plan_timing.py $c | sed "s/^/default $c /" >> $O/ab.txt 2>&1
  SFT_LIB=$PWD/sweep_libs/lib_PUBLISH0.so timeout 300 python scripts/plan_timing.py $c | sed "s/^/PUBLISH0 $c /" >> $O/ab.txt 2>&1
done; done
for c in C0 C1; do timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2>/dev/null; SFT_LIB=$PWD/sweep_libs/lib_PUBLISH0.so timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_${c}_old.json 2>/dev/null; done
