# tree build with the per-block count scan: tree tests + plan timing
cd $GRAFT_REPO_ROOT
O=gpurun_out/ts; mkdir -p $O
timeout 1200 python -m pytest tests -q -x -m gpu -p no:cacheprovider -k "tree or sort or extreme or uniform or C2_full or C4_full or C3_full or multirank or small" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for c in C2 C3 C4; do timeout 300 python scripts/plan_timing.py $c > $O/plan_$c.txt 2>&1; done
SFT_PLAN_TRACE=1 timeout 300 python scripts/step_timeline.py C4 2>&1 | tail -3 > $O/trace_C4.txt
