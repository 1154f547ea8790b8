cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:k_translate_ws --launch-skip 4 --launch-count 1 -o gpurun_out/c4_def -f python scripts/run_config.py --config C4 --reps 1 > gpurun_out/ncu_a.log 2>&1
SFT_LIB=$PWD/sweep_libs/lib_ABL_NOSSTORE1.so timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:k_translate_ws --launch-skip 4 --launch-count 1 -o gpurun_out/c4_noss -f python scripts/run_config.py --config C4 --reps 1 > gpurun_out/ncu_b.log 2>&1
