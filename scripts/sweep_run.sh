#!/bin/bash
# run the translation timing of every variant lib on the configs its name targets
for f in sweep_libs/lib_*.so; do
  n=$(basename $f)
  cfgs=""
  case $n in *29*|*OTHER*) cfgs="$cfgs C2";; esac
  case $n in *37*|*OTHER*) cfgs="$cfgs C4";; esac
  case $n in *35*) cfgs="$cfgs C3";; esac
  case $n in lib_G294_NC294_NST292_MINB294.so) cfgs="C2 C3 C4";; esac
  for c in $cfgs; do SFT_LIB=$PWD/$f timeout 300 python scripts/sweep_cfg.py $c 2>&1 | tail -1; done
done
