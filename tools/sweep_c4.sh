#!/bin/bash
# Dev: config 4 (e=8) per backend + config 3 for each variant lib.
for lib in build/variants/lib_*.so; do
  v=$(basename $lib .so)
  for be in tc_fp4 tc_i8; do
    r=$(GF2E_LIB_PATH=$PWD/$lib timeout 300 python bench.py --config 4 --e 8 --backend $be --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['kernel'])")
    echo "$v c4e8 $be: $r"
  done
  r=$(GF2E_LIB_PATH=$PWD/$lib timeout 300 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'])")
  echo "$v c3: $r"
done
