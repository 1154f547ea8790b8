cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name regex:k_translate_ws --launch-skip 6 --launch-count 1 -o gpurun_out/trans_c2_z -f python scripts/run_config.py --config C2 --reps 1 > gpurun_out/ncu_c2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name regex:"k_leaf|k_final|k_schedule|k_fill|k_count" --launch-count 5 -o gpurun_out/aux_c2 -f python scripts/run_config.py --config C2 --reps 1 > gpurun_out/ncu_aux.log 2>&1
