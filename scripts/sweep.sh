for f in build/sweep/lib_29_*.so; do SFT_LIB=$PWD/$f python scripts/sweep_cfg.py C2; done
for f in build/sweep/lib_37_*.so; do SFT_LIB=$PWD/$f python scripts/sweep_cfg.py C4; done
