# PDL on leaf/final + early triggers: A/B (SFT_PDL=0 disables the attribute), bench C0/C1, GPU suite
cd $GRAFT_REPO_ROOT
O=gpurun_out/pdl; mkdir -p $O
for rep in 1 2; do for c in C0 C1 C2; do
  timeout 300 python scripts/sweep_cfg.py $c >> $O/ab.txt 2>&1
  SFT_PDL=0 timeout 300 python scripts/sweep_cfg.py $c | sed 's/"default"/"PDL0"/' >> $O/ab.txt 2>&1
done; done
for c in C0 C1; do timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 2400 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
