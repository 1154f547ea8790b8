cd $GRAFT_REPO_ROOT
for c in C0 C1; do SFT_PLAN_TRACE=1 timeout 120 python scripts/step_timeline.py $c 2>&1 | tail -3; done
for c in C0 C1; do timeout 120 python scripts/step_timeline.py $c 2>&1 | tail -1; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_C1.csv python scripts/step_timeline.py C1 > /dev/null 2>&1
