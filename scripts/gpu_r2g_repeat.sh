# Box-to-box / run-to-run variance of the r2g head: C2, C3, C4 bench lines three times each
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2g_rep; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $O/smi.txt 2>&1
for i in 1 2 3; do
  for c in C2 C3 C4; do timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_${c}_$i.json 2> $O/bench_${c}_$i.err; done
done
