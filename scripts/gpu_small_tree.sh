cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "small_tree or errors or extreme or C1 or single or domain" -p no:cacheprovider > gpurun_out/pytest_st.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_st.log
for c in C0 C1; do for v in "1 2048" "1 16384" "1 0" "0 0"; do set -- $v; SFT_SMALL_TREE=$1 SFT_SMALL_FULL=$2 timeout 600 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --no-configs --nrhs 1 > gpurun_out/bench_${c}_st$1_$2.json 2> gpurun_out/bench_${c}_st$1_$2.err; done; done
