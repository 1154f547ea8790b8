for rep in 1; do
SWEEP_P=7 python scripts/sweep_cfg.py C2 | cut -c1-100; for f in sweep_libs/lib_G27*.so; do SWEEP_P=7 SFT_LIB=$PWD/$f python scripts/sweep_cfg.py C2 | cut -c1-100; done
SWEEP_P=5 python scripts/sweep_cfg.py C2 | cut -c1-100; for f in sweep_libs/lib_G25*.so; do SWEEP_P=5 SFT_LIB=$PWD/$f python scripts/sweep_cfg.py C2 | cut -c1-100; done
done
