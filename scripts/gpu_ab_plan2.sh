cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
out=gpurun_out/ab_plan.txt; : > $out
for rep in 1 2; do for c in C0 C1; do
  echo "$c default $(timeout 300 python scripts/plan_timing.py $c 2>&1 | tail -1)" >> $out
  for f in sweep_libs/lib_*.so; do echo "$c $(basename $f) $(SFT_LIB=$PWD/$f timeout 300 python scripts/plan_timing.py $c 2>&1 | tail -1)" >> $out; done
done; done
