# p = 5 direct form: tail delta merged into lane 0's child-1 load (+ axis-0 row map): parity + A/B
cd $GRAFT_REPO_ROOT
O=gpurun_out/tl; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -p no:cacheprovider -k "(small and 5) or C3_full or C0 or uniform or extreme or dynamic" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for rep in 1 2; do for c in C0 C3; do
  timeout 300 python scripts/sweep_cfg.py $c >> $O/ab.txt 2>&1
  SFT_LIB=$PWD/sweep_libs/lib_prevtail.so timeout 300 python scripts/sweep_cfg.py $c >> $O/ab.txt 2>&1
done; done
