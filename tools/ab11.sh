O=gpurun_out/ab11; mkdir -p $O
GF2E_LIB_PATH=build/variants/lib_ad4.so timeout 1200 python -m pytest tests -m gpu -x -q -k "config3 or long or fuzz or smoke or selfcheck or fp4 or golden" 2>&1 | tail -2 > $O/pytest.txt; cat $O/pytest.txt
for r in 1 2; do for V in ad0 ad4 ad6 ad2; do
 GF2E_LIB_PATH=build/variants/lib_$V.so timeout 300 python bench.py --no-e2e --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$V', d['ms_per_step'], d['value'], d['roofline']['frac'], d['roofline']['kernel_ms'], d.get('parity',{}).get('device'), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done 2>&1 | tee $O/ab.txt
