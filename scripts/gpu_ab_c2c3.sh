# A/B: p = 9 centre on DMMA (C2), 3D p = 5 configs (C3)
cd $GRAFT_REPO_ROOT
O=gpurun_out/ab23; mkdir -p $O
for rep in 1 2; do
  timeout 300 python scripts/sweep_cfg.py C2 >> $O/ab.txt 2>&1
  SFT_LIB=$PWD/sweep_libs/lib_CENTRE_DMMA1.so timeout 300 python scripts/sweep_cfg.py C2 >> $O/ab.txt 2>&1
  timeout 300 python scripts/sweep_cfg.py C3 >> $O/ab.txt 2>&1
  for f in sweep_libs/lib_*35*.so; do SFT_LIB=$PWD/$f timeout 300 python scripts/sweep_cfg.py C3 >> $O/ab.txt 2>&1; done
done
