O=gpurun_out/ab9; mkdir -p $O
GF2E_LIB_PATH=build/variants/lib_noreinit.so timeout 900 python -m pytest tests -m gpu -x -q -k "run or config4 or fuzz or selfcheck or fp4 or paired" 2>&1 | tail -2 > $O/pytest.txt; cat $O/pytest.txt
for V in noreinit reinit1; do for e in 2 3 4 5 6 7 8 9 10; do
 GF2E_LIB_PATH=build/variants/lib_$V.so timeout 300 python bench.py --config 4 --e $e --no-e2e --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$V', d['config']['workload'][:20], d['ms_per_step'], d['value'], d['roofline']['frac'], d.get('parity',{}).get('device'))"
done; done 2>&1 | tee $O/ab.txt
