cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m "gpu and not slow" -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
out=gpurun_out/sweep.txt; : > $out
for c in C2 C3 C4 C1 C0; do timeout 300 python scripts/sweep_cfg.py $c >> $out 2>&1; done
for f in sweep_libs/lib_*.so; do for c in C2 C4; do SFT_LIB=$PWD/$f timeout 300 python scripts/sweep_cfg.py $c >> $out 2>&1; done; done
SFT_PLAN_TRACE=1 timeout 120 python scripts/step_timeline.py C2 > gpurun_out/trace_c2.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name regex:k_translate_ws --launch-skip 6 --launch-count 1 -o gpurun_out/trans_c2_m -f python scripts/run_config.py --config C2 --reps 1 > gpurun_out/ncu_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:k_translate_ws --launch-skip 4 --launch-count 1 -o gpurun_out/trans_c4_m -f python scripts/run_config.py --config C4 --reps 1 > gpurun_out/ncu_c4.log 2>&1
