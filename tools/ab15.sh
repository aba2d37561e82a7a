O=gpurun_out/ab15; mkdir -p $O
for r in 1 2; do for V in gm8 gm32 gm128; do for e in 2 8 10; do
  GF2E_LIB_PATH=build/variants/lib_$V.so timeout 300 python bench.py --config 4 --e $e --no-e2e --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$V', d['config']['workload'][:20], d['ms_per_step'], d['value'], d['roofline']['frac'], d.get('parity',{}).get('device'))"
done; done; done 2>&1 | tee $O/ab.txt
