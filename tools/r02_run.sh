#!/bin/bash
# run-form iteration: parity of the run form, config-4 lines (run vs i8), role counters, optional ncu
O=gpurun_out/${1:-r2d}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "run_form" > $O/pytest_run.log 2>&1; tail -2 $O/pytest_run.log
if grep -q failed $O/pytest_run.log; then grep -E "Error|assert" $O/pytest_run.log | head -20; exit 0; fi
for e in 2 8 10; do
  for b in tc_run tc_i8; do
    if [ "$b" = tc_i8 ] && [ -z "$3" ]; then continue; fi
    timeout 300 python bench.py --config 4 --e $e --backend $b --no-e2e --no-cpu-baseline > $O/c4_e${e}_$b.json 2>&1
    python -c "import json;d=json.loads(open('$O/c4_e${e}_$b.json').read().strip().splitlines()[-1]);r=d['roofline'];print('e=$e $b',d['value'],d['ms_per_step'],r['kernel'],r['kernel_ms'],r['frac'])" 2>&1 | tail -1
  done
done
GF2E_LIB_PATH=build/variants/lib_instr_run.so timeout 300 python tools/instr_run.py 8 65536 256 65536 --acc > $O/instr_e8.txt 2>&1; cat $O/instr_e8.txt
if [ -n "$2" ] && [ "$2" != "-" ]; then
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name k_product_run --launch-skip 1 --launch-count 1 -o $O/run_c4e8 -f python tools/prof_case.py 8 65536 256 65536 --acc --reps 2 --backend tc_run > $O/ncu_run.log 2>&1; tail -1 $O/ncu_run.log
fi
echo done
