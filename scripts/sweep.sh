for f in sweep_libs/lib_*.so; do SFT_LIB=$PWD/$f python scripts/sweep_cfg.py C2; done
for f in sweep_libs/lib_*.so; do SFT_LIB=$PWD/$f python scripts/sweep_cfg.py C4; done
