O=gpurun_out/ab20; mkdir -p $O
for r in 1 2; do for V in t8 t4 t12 t16; do
 GF2E_LIB_PATH=build/variants/lib_$V.so timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$V c3', d['ms_per_step'], d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
 GF2E_LIB_PATH=build/variants/lib_$V.so timeout 300 python bench.py --config 2 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$V c2', d['ms_per_step'], d['value'], d['roofline']['frac'])"
done; done 2>&1 | tee $O/ab.txt
