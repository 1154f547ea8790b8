cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SFT_PLAN_TRACE=1 timeout 120 python scripts/step_timeline.py C2 > gpurun_out/trace_c2.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name regex:"k_final|k_leaf" --launch-count 2 -o gpurun_out/leaf_final_c2 -f python scripts/run_config.py --config C2 --reps 1 > gpurun_out/ncu_lf.log 2>&1
