# p = 5 in the symmetric form (SFT_SYM5=1) vs the direct form: parity (small 2D/3D p=5) and timing
cd $GRAFT_REPO_ROOT
O=gpurun_out/sym5; mkdir -p $O
SFT_LIB=$PWD/sweep_libs/lib_SYM51.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -p no:cacheprovider -k "small and 5" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for rep in 1 2; do for c in C0 C3; do
  timeout 300 python scripts/sweep_cfg.py $c >> $O/ab.txt 2>&1
  SFT_LIB=$PWD/sweep_libs/lib_SYM51.so timeout 300 python scripts/sweep_cfg.py $c >> $O/ab.txt 2>&1
done; done
SWEEP_P=5 timeout 300 python scripts/sweep_cfg.py C2 >> $O/ab.txt 2>&1
SWEEP_P=5 SFT_LIB=$PWD/sweep_libs/lib_SYM51.so timeout 300 python scripts/sweep_cfg.py C2 >> $O/ab.txt 2>&1
