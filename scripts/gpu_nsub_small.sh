# NSUB = 2 for 2D p = 5 / 7 (latency-bound small configs): parity subset + A/B
cd $GRAFT_REPO_ROOT
O=gpurun_out/nsub; mkdir -p $O
SFT_LIB=$PWD/sweep_libs/lib_NSUB272.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -p no:cacheprovider -k "small or two_level or C1" > $O/pytest7.log 2>&1; echo "rc=$?" >> $O/pytest7.log
for rep in 1 2; do for c in C0 C1; do
  timeout 300 python scripts/sweep_cfg.py $c >> $O/ab.txt 2>&1
  for f in sweep_libs/lib_*.so; do SFT_LIB=$PWD/$f timeout 300 python scripts/sweep_cfg.py $c >> $O/ab.txt 2>&1; done
done; done
for c in C0 C1; do timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2>/dev/null; SFT_LIB=$PWD/sweep_libs/lib_NSUB272.so timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_${c}_n2.json 2>/dev/null; done
