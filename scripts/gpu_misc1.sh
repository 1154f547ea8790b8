cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/fp32_errors.py > gpurun_out/fp32_errors.txt 2>&1
for m in 0 first all; do SFT_F2=$m timeout 300 python scripts/sweep_cfg.py C2 >> gpurun_out/f2.txt 2>&1; SFT_F2=$m timeout 300 python scripts/sweep_cfg.py C1 >> gpurun_out/f2.txt 2>&1; done
for c in C2 C3 C4; do timeout 300 python scripts/sweep_cfg.py $c >> gpurun_out/f2.txt 2>&1; done
