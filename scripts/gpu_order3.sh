# 3D per-group axis order: A/B of the translation time (default vs SFT_ORDER3=0), then the GPU tests
cd $GRAFT_REPO_ROOT
O=gpurun_out/o3; mkdir -p $O
for rep in 1 2; do for c in C3 C4; do
  timeout 300 python scripts/sweep_cfg.py $c >> $O/ab.txt 2>&1
  SFT_LIB=$PWD/sweep_libs/lib_ORDER30.so timeout 300 python scripts/sweep_cfg.py $c >> $O/ab.txt 2>&1
done; done
timeout 2400 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
