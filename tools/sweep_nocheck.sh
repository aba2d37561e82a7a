for lib in build/variants/lib_*.so; do
  v=$(basename $lib .so)
  c3=$(GF2E_LIB_PATH=$PWD/$lib timeout 300 python bench.py --config 3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'])")
  echo "$v | c3 ms,frac: $c3"
done
