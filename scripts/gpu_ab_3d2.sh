# A/B: 3D p = 5 (C3) and p = 7 (C4) configurations
cd $GRAFT_REPO_ROOT
O=gpurun_out/ab3d2; mkdir -p $O
for rep in 1 2; do
  timeout 300 python scripts/sweep_cfg.py C3 >> $O/ab.txt 2>&1
  for f in sweep_libs/lib_*35*.so; do SFT_LIB=$PWD/$f timeout 300 python scripts/sweep_cfg.py C3 >> $O/ab.txt 2>&1; done
  timeout 300 python scripts/sweep_cfg.py C4 >> $O/ab.txt 2>&1
  for f in sweep_libs/lib_*37*.so; do SFT_LIB=$PWD/$f timeout 300 python scripts/sweep_cfg.py C4 >> $O/ab.txt 2>&1; done
done
