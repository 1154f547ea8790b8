# p = 5 tail on a second DMMA tile (SFT_TAIL5_DMMA=1): parity for p = 5 and timing
cd $GRAFT_REPO_ROOT
O=gpurun_out/tail5; mkdir -p $O
export SFT_LIB_V=$PWD/sweep_libs/lib_TAIL5_DMMA1.so
SFT_LIB=$SFT_LIB_V timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -p no:cacheprovider -k "(small and 5) or C3_full or C0 or uniform or extreme" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for rep in 1 2; do for c in C0 C3; do
  timeout 300 python scripts/sweep_cfg.py $c >> $O/ab.txt 2>&1
  SFT_LIB=$SFT_LIB_V timeout 300 python scripts/sweep_cfg.py $c >> $O/ab.txt 2>&1
done; done
SWEEP_P=5 timeout 300 python scripts/sweep_cfg.py C2 >> $O/ab.txt 2>&1
SWEEP_P=5 SFT_LIB=$SFT_LIB_V timeout 300 python scripts/sweep_cfg.py C2 >> $O/ab.txt 2>&1
