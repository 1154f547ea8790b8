# dynamic tile scheduling: parity subset, then A/B vs SFT_DYN=0 (static grid-stride)
cd $GRAFT_REPO_ROOT
O=gpurun_out/dyn; mkdir -p $O
timeout 1500 python -m pytest tests -q -x -m gpu -p no:cacheprovider -k "small or C2_full or C3_full or C4_one or batch or two_level or multirank or nccl or fp32 or determin or zero" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for rep in 1 2; do for c in C1 C2 C3 C4; do
  timeout 300 python scripts/sweep_cfg.py $c >> $O/ab.txt 2>&1
  SFT_DYN=0 timeout 300 python scripts/sweep_cfg.py $c | sed 's/"default"/"DYN0"/' >> $O/ab.txt 2>&1
done; done
