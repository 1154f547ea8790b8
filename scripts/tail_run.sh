for c in C2 C3 C2 C3; do
  python scripts/sweep_cfg.py $c | cut -c1-100
  for f in sweep_libs/lib_TAIL*.so; do SFT_LIB=$PWD/$f python scripts/sweep_cfg.py $c | cut -c1-100; done
done
