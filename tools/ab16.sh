O=gpurun_out/ab16; mkdir -p $O
for V in gm8 gm16 gm24 gm32 gm48; do for e in 2 3 4 5 6 7 8 9 10; do
  GF2E_LIB_PATH=build/variants/lib_$V.so timeout 300 python bench.py --config 4 --e $e --no-e2e --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$V', d['config']['e'], d['ms_per_step'], d['value'], d['roofline']['frac'])"
done; done 2>&1 | tee $O/ab.txt
