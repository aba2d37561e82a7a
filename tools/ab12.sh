O=gpurun_out/ab12; mkdir -p $O
for F in 0 4194304; do for c in 1 2; do
 GF2E_FORK_MIN_BITS=$F timeout 300 python bench.py --config $c --no-e2e --steps 50 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('fork_min=$F', d['config']['workload'][:24], d['ms_per_step'], d['value'], d['roofline']['kernel_ms'], d.get('parity',{}).get('device'))"
done; GF2E_FORK_MIN_BITS=$F python tools/host_overhead.py 2>&1 | head -1 | sed "s/^/fork_min=$F /"; done 2>&1 | tee $O/ab.txt
timeout 300 python tools/prof_ple.py 8 1024 4 2>&1 | tail -1 | tee -a $O/ab.txt
