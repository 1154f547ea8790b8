cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SFT_PLAN_TRACE=1 timeout 300 python bench.py --config C1 --steps 5 --warmup 3 --no-cpu-baseline --no-configs --nrhs 1 > gpurun_out/c1_trace.json 2> gpurun_out/c1_trace.err
SFT_PLAN_TRACE=1 timeout 300 python bench.py --config C0 --steps 5 --warmup 3 --no-cpu-baseline --no-configs --nrhs 1 > gpurun_out/c0_trace.json 2> gpurun_out/c0_trace.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_C1.csv python bench.py --config C1 --steps 2 --warmup 3 --no-cpu-baseline --no-configs --nrhs 1 > gpurun_out/ncu_c1.log 2>&1
