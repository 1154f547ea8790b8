cd $GRAFT_REPO_ROOT
O=gpurun_out/trs; mkdir -p $O
for c in C0 C1; do SFT_PLAN_TRACE=1 timeout 300 python scripts/step_timeline.py $c > $O/trace_$c.txt 2>&1; done
