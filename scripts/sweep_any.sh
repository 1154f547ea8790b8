# time the default build and every sweep_libs variant on the given configs (args), twice
for rep in 1 2; do for c in "$@"; do
  python scripts/sweep_cfg.py $c | cut -c1-100
  for f in sweep_libs/lib_*.so; do SFT_LIB=$PWD/$f python scripts/sweep_cfg.py $c | cut -c1-100; done
done; done
