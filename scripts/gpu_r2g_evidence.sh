# Round-2 (session 3, final head) evidence: default bench line, per-config lines, FP32 line,
# reference arm, ncu launch list, ncu --set full of C2/C3/C4 levels, DRAM traffic
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2g; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=10 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err
for c in C0 C1 C3 C4; do timeout 900 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 600 python bench.py --precision f32 --no-cpu-baseline > $O/bench_C2_f32.json 2> $O/bench_f32.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_C2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --nrhs 1 > $O/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name regex:k_translate_ws --launch-skip 6 --launch-count 1 -o $O/trans_c2 -f python scripts/run_config.py --config C2 --reps 1 > $O/ncu_c2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name regex:k_translate_ws --launch-skip 3 --launch-count 1 -o $O/trans_c3 -f python scripts/run_config.py --config C3 --reps 1 > $O/ncu_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:k_translate_ws --launch-skip 4 --launch-count 1 -o $O/trans_c4 -f python scripts/run_config.py --config C4 --reps 1 > $O/ncu_c4.log 2>&1
for c in C2 C3 C4; do timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --kernel-name regex:k_translate_ws --csv --log-file $O/traffic_$c.csv python scripts/run_config.py --config $c --reps 1 > $O/ncu_traffic_$c.log 2>&1; done
