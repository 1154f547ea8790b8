# full GPU suite on the current defaults + plan traces of C2 / C4
cd $GRAFT_REPO_ROOT
O=gpurun_out/st; mkdir -p $O
for c in C2 C4; do SFT_PLAN_TRACE=1 timeout 300 python scripts/step_timeline.py $c > $O/trace_$c.txt 2>&1; timeout 300 python scripts/plan_timing.py $c > $O/plan_$c.txt 2>&1; done
timeout 2400 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
