# 3D skewed round pipeline (NST >= 3 configs): parity on one variant per p, A/B timing
cd $GRAFT_REPO_ROOT
O=gpurun_out/skew3; mkdir -p $O
SFT_LIB=$PWD/sweep_libs/lib_G351_NST353_MINB354.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -p no:cacheprovider -k "3d or C3_full or dynamic" > $O/pytest5.log 2>&1; echo "rc=$?" >> $O/pytest5.log
SFT_LIB=$PWD/sweep_libs/lib_NST373_NC3716.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -p no:cacheprovider -k "3d or C4_one" > $O/pytest7.log 2>&1; echo "rc=$?" >> $O/pytest7.log
for rep in 1 2; do
  timeout 300 python scripts/sweep_cfg.py C3 >> $O/ab.txt 2>&1
  for f in sweep_libs/lib_*35*.so; do SFT_LIB=$PWD/$f timeout 300 python scripts/sweep_cfg.py C3 >> $O/ab.txt 2>&1; done
  timeout 300 python scripts/sweep_cfg.py C4 >> $O/ab.txt 2>&1
  for f in sweep_libs/lib_*37*.so; do SFT_LIB=$PWD/$f timeout 300 python scripts/sweep_cfg.py C4 >> $O/ab.txt 2>&1; done
done
