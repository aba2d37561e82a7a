#!/bin/bash
# Dev: config-4 (k = 256) device time per build variant in build/variants/lib_*.so.
for lib in build/variants/lib_*.so; do
  v=$(basename $lib .so)
  for e in 2 8; do
    c4=$(GF2E_LIB_PATH=$PWD/$lib timeout 300 python bench.py --config 4 --e $e --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'])")
    echo "$v | c4 e=$e ms,frac: $c4"
  done
done
