#!/bin/bash
# Dev: per-variant wait-cycle counters (libs built with -DGF2E_INSTR=1) + config 3 timing.
for lib in build/variants/lib_*.so; do
  v=$(basename $lib .so)
  echo "== $v"
  GF2E_LIB_PATH=$PWD/$lib timeout 300 python tools/instr.py 8 16384 16384 16384 2>&1 | grep -E "exp_empty|exp_bfull|mma_full|mma_tempty"
  GF2E_LIB_PATH=$PWD/$lib timeout 300 python bench.py --config 3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', d['ms_per_step'], d['roofline']['frac'])"
done
