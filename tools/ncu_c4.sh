# ncu --set full of the running-sum product kernel at config 4 (e given), after a clean run
O=gpurun_out/ncu_c4; mkdir -p $O
E=${1:-8}
timeout 300 python bench.py --config 4 --e $E --no-e2e --no-cpu-baseline --steps 2 --warmup 3 > $O/plain_e$E.json 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:k_product_run<.int.$E," -c 1 \
  -o $O/run_c4e$E python bench.py --config 4 --e $E --no-e2e --no-cpu-baseline --steps 1 --warmup 3 > $O/ncu_e$E.log 2>&1
tail -3 $O/ncu_e$E.log
