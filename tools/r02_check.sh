#!/bin/bash
# re-entry check of HEAD on a B200: GPU tests, smoke, headline bench, config 4 at e = 8
O=gpurun_out/${1:-r2check}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; tail -c 400 $O/bench_default.json
timeout 300 python bench.py --config 4 --e 8 > $O/bench_config4_e8.json 2>&1; tail -c 400 $O/bench_config4_e8.json
