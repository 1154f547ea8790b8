cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "small_tree or errors or extreme or C1 or single or domain or sort_graph" -p no:cacheprovider > gpurun_out/pytest_st.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_st.log
for c in C1 C0 C2; do for v in 1 0; do SFT_CLUSTER_TREE=$v timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-configs --nrhs 1 > gpurun_out/bench_${c}_ct$v.json 2> gpurun_out/bench_${c}_ct$v.err; done; done
