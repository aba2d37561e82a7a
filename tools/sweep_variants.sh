#!/bin/bash
# A/B timing of kernel build variants in build/variants/lib_*.so (dev tool).
for lib in build/variants/lib_*.so; do
  v=$(basename $lib .so)
  ok=$(GF2E_LIB_PATH=$PWD/$lib timeout 300 python tools/debug_mismatch.py 8 1024 4096 1024 2 2>&1 | tail -1)
  c3=$(GF2E_LIB_PATH=$PWD/$lib timeout 300 python bench.py --config 3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'])")
  c4=$(GF2E_LIB_PATH=$PWD/$lib timeout 300 python bench.py --config 4 --e 8 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'])")
  echo "$v | check: $ok | c3 ms,frac: $c3 | c4e8 ms,frac: $c4"
done
