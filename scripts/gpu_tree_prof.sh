cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in C1 C0; do timeout 600 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --no-configs --nrhs 1 > gpurun_out/bench_${c}_ct.json 2> gpurun_out/bench_${c}_ct.err; done
SFT_CLUSTER_TREE=0 timeout 600 python bench.py --config C1 --steps 50 --warmup 5 --no-cpu-baseline --no-configs --nrhs 1 > gpurun_out/bench_C1_ct0.json 2> gpurun_out/bench_C1_ct0.err
for c in C1 C0; do SFT_LIB=$PWD/sweep_libs/lib_TREE_PROF1.so timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-configs --nrhs 1 > gpurun_out/prof_$c.out 2>&1; done
SFT_SMALL_FULL=16384 SFT_LIB=$PWD/sweep_libs/lib_TREE_PROF1.so timeout 300 python bench.py --config C1 --steps 3 --warmup 3 --no-cpu-baseline --no-configs --nrhs 1 > gpurun_out/prof_C1full.out 2>&1
