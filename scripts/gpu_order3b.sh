# 3D rounds: unroll variant timing; ncu of one C3 level, default vs fixed order
cd $GRAFT_REPO_ROOT
O=gpurun_out/o3b; mkdir -p $O
for rep in 1 2; do for c in C3 C4; do
  timeout 300 python scripts/sweep_cfg.py $c >> $O/ab.txt 2>&1
  SFT_LIB=$PWD/sweep_libs/lib_ROUND_UNROLL1.so timeout 300 python scripts/sweep_cfg.py $c >> $O/ab.txt 2>&1
done; done
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name regex:k_translate_ws --launch-skip 3 --launch-count 1 -o $O/c3_new -f python scripts/run_config.py --config C3 --reps 1 > $O/ncu1.log 2>&1
SFT_LIB=$PWD/sweep_libs/lib_ORDER30.so timeout 600 ncu --set full --clock-control none --import-source on --kernel-name regex:k_translate_ws --launch-skip 3 --launch-count 1 -o $O/c3_fixed -f python scripts/run_config.py --config C3 --reps 1 > $O/ncu2.log 2>&1
