# ncu --set full of one C2 and one C4 translation level (current head)
cd $GRAFT_REPO_ROOT
O=gpurun_out/ncu3; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name regex:k_translate_ws --launch-skip 6 --launch-count 1 -o $O/c2 -f python scripts/run_config.py --config C2 --reps 1 > $O/ncu_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:k_translate_ws --launch-skip 4 --launch-count 1 -o $O/c4 -f python scripts/run_config.py --config C4 --reps 1 > $O/ncu_c4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name regex:k_translate_ws --launch-skip 3 --launch-count 1 -o $O/c3 -f python scripts/run_config.py --config C3 --reps 1 > $O/ncu_c3.log 2>&1
