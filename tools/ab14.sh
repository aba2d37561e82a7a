O=gpurun_out/ab14; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q -k "run or config4 or fuzz or paired or selfcheck" 2>&1 | tail -2 > $O/pytest.txt; cat $O/pytest.txt
for r in 1 2; do for V in rt1 default; do
  L=paper_1111_6900_b200/libgf2e_b200.so; [ $V = rt1 ] && L=build/variants/lib_rt1.so
  for e in 3 4 5 6; do
  GF2E_LIB_PATH=$L timeout 300 python bench.py --config 4 --e $e --no-e2e --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$V', d['config']['workload'][:20], d['ms_per_step'], d['value'], d['roofline']['frac'], d.get('parity',{}).get('device'))"
  done
done; done 2>&1 | tee $O/ab.txt
