cd $GRAFT_REPO_ROOT
O=gpurun_out/ab_c3b; mkdir -p $O
for rep in 1 2; do
  timeout 300 python scripts/sweep_cfg.py C3 >> $O/ab.txt 2>&1
  for f in sweep_libs/lib_*.so; do SFT_LIB=$PWD/$f timeout 300 python scripts/sweep_cfg.py C3 >> $O/ab.txt 2>&1; done
done
