for rep in 1 2; do python scripts/step_timeline.py C1 | tail -1; for f in sweep_libs/lib_BS*.so; do echo $f; SFT_LIB=$PWD/$f python scripts/step_timeline.py C1 | tail -1; done; done
