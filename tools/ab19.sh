O=gpurun_out/ab19; mkdir -p $O
for r in 1 2 3; do for V in s8 s48; do for e in 2 3 4 5 6; do
  GF2E_LIB_PATH=build/variants/lib_$V.so timeout 300 python bench.py --config 4 --e $e --no-e2e --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$V', d['config']['e'], d['ms_per_step'], d['value'])"
done; done; done 2>&1 | tee $O/ab.txt
