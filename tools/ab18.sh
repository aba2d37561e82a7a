O=gpurun_out/ab18; mkdir -p $O
for r in 1 2; do for B in tc tc_run; do
 timeout 300 python bench.py --config 2 --backend $B --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$B', d['ms_per_step'], d['value'], d['roofline']['frac'], d['roofline']['kernel'], d['roofline']['kernel_ms'], d.get('parity',{}).get('device'))"
done; done 2>&1 | tee $O/ab.txt
timeout 600 python tools/form_cross.py 4 4096 4096 1024,2048,3072,4096,6144,8192 2>&1 | tee -a $O/ab.txt
timeout 600 python tools/form_cross.py 8 8192 8192 1024,2048,3072,4096 2>&1 | tee -a $O/ab.txt
