cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
out=gpurun_out/sweep.txt; : > $out
for c in C2 C3 C4; do timeout 300 python scripts/sweep_cfg.py $c >> $out 2>&1; done
for f in sweep_libs/lib_*37*.so sweep_libs/lib_G372*.so; do SFT_LIB=$PWD/$f timeout 300 python scripts/sweep_cfg.py C4 >> $out 2>&1; done
for f in sweep_libs/lib_*29*.so; do SFT_LIB=$PWD/$f timeout 300 python scripts/sweep_cfg.py C2 >> $out 2>&1; done
for f in sweep_libs/lib_*35*.so; do SFT_LIB=$PWD/$f timeout 300 python scripts/sweep_cfg.py C3 >> $out 2>&1; done
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name regex:k_translate_ws --launch-skip 6 --launch-count 1 -o gpurun_out/trans_c2_sym -f python scripts/run_config.py --config C2 --reps 1 > gpurun_out/ncu_c2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name regex:k_translate_ws --launch-skip 3 --launch-count 1 -o gpurun_out/trans_c3_sym -f python scripts/run_config.py --config C3 --reps 1 > gpurun_out/ncu_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:k_translate_ws --launch-skip 4 --launch-count 1 -o gpurun_out/trans_c4_sym -f python scripts/run_config.py --config C4 --reps 1 > gpurun_out/ncu_c4.log 2>&1
timeout 2400 python -m pytest tests -x -q -m "gpu and slow" -p no:cacheprovider -s --durations=5 > gpurun_out/pytest_slow.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_slow.log
