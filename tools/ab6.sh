O=gpurun_out/ab6; mkdir -p $O
L=build/variants/lib_pair.so
GF2E_LIB_PATH=$L timeout 900 python -m pytest tests -m gpu -x -q -k "run or config4 or fuzz or selfcheck or fp4" 2>&1 | tail -3 > $O/pytest.txt
cat $O/pytest.txt
for P in 1 0; do for e in 2 3 4 5 6 7 8; do
 GF2E_RUN_PAIR=$P GF2E_LIB_PATH=$L timeout 300 python bench.py --config 4 --e $e --no-e2e --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('pair$P', d['config']['workload'][:20], d['ms_per_step'], d['value'], d['roofline']['frac'], d.get('parity',{}).get('device'))"
done; done 2>&1 | tee $O/ab.txt
