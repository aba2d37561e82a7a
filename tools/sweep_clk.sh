#!/bin/bash
# Dev: per-variant effective SM clock + per-cycle MMA efficiency (libs built with -DGF2E_INSTR=2) and config 3 timing.
for lib in build/variants/lib_*.so; do
  v=$(basename $lib .so)
  echo "== $v $(GF2E_LIB_PATH=$PWD/$lib timeout 300 python tools/instr.py 8 16384 16384 16384 2>&1 | tail -2 | tr '\n' ' ')"
done
