# producer-less translation kernel: quick parity subset, then A/B vs SFT_PL=0
cd $GRAFT_REPO_ROOT
O=gpurun_out/pl; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -p no:cacheprovider -k "small or C2_full or C3_full or C4_one or batch or two_level or uniform" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for rep in 1 2; do for c in C0 C1 C2 C3 C4; do
  timeout 300 python scripts/sweep_cfg.py $c >> $O/ab.txt 2>&1
  SFT_LIB=$PWD/sweep_libs/lib_PL0.so timeout 300 python scripts/sweep_cfg.py $c >> $O/ab.txt 2>&1
done; done
