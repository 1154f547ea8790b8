# A/B of sweep_libs variants vs the default build on C3 / C4 translation time
cd $GRAFT_REPO_ROOT
O=gpurun_out/ab3d; mkdir -p $O
for rep in 1 2; do
  for c in ${AB_CONFIGS:-C3 C4}; do
    timeout 300 python scripts/sweep_cfg.py $c >> $O/ab.txt 2>&1
    for f in sweep_libs/lib_*.so; do
      case "$c:$f" in C3:*NC37*) continue;; C4:*35*) continue;; esac
      SFT_LIB=$PWD/$f timeout 300 python scripts/sweep_cfg.py $c >> $O/ab.txt 2>&1
    done
  done
done
