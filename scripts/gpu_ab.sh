# A/B of sweep_libs variants against the default build on one box, interleaved
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
out=gpurun_out/ab.txt; : > $out
for rep in 1 2; do
  for c in ${AB_CONFIGS:-C2 C3 C4}; do
    timeout 300 python scripts/sweep_cfg.py $c >> $out 2>&1
    for f in sweep_libs/lib_*.so; do SFT_LIB=$PWD/$f timeout 300 python scripts/sweep_cfg.py $c >> $out 2>&1; done
  done
done
