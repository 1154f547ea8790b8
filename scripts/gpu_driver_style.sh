# The driver's own commands on one GPU: bench under torchrun with N = 1, and the two arms with defaults
cd $GRAFT_REPO_ROOT
O=gpurun_out/drv; mkdir -p $O
S=$(date +%s)
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 10 --warmup 3 > $O/bench_torchrun_n1.json 2> $O/bench_torchrun_n1.err; echo "rc=$? $(( $(date +%s) - S )) s" >> $O/bench_torchrun_n1.err
S=$(date +%s)
timeout 900 python bench.py --impl reference --gpus 1 --steps 10 --warmup 3 > $O/bench_ref_default.json 2> $O/bench_ref_default.err; echo "rc=$? $(( $(date +%s) - S )) s" >> $O/bench_ref_default.err
for f in $O/*.err; do tail -n 2 $f; done; cut -c1-300 $O/*.json
