cd $GRAFT_REPO_ROOT
./sweep_libs/malloc_probe
SFT_PLAN_TRACE=1 timeout 120 python scripts/step_timeline.py C2 2>&1 | tail -3
SFT_PLAN_TRACE=1 timeout 120 python scripts/step_timeline.py C1 2>&1 | tail -3
