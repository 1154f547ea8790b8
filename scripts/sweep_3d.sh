for rep in 1 2; do
python scripts/sweep_cfg.py C4 | cut -c1-100
for f in sweep_libs/lib_NC37*.so; do SFT_LIB=$PWD/$f python scripts/sweep_cfg.py C4 | cut -c1-100; done
python scripts/sweep_cfg.py C3 | cut -c1-100
for f in sweep_libs/lib_G35*.so; do SFT_LIB=$PWD/$f python scripts/sweep_cfg.py C3 | cut -c1-100; done
done
