O=gpurun_out/ab10; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q -k "ple or trsm or echelon or consumer or counters or newton or nj" 2>&1 | tail -2 > $O/pytest.txt; cat $O/pytest.txt
for V in default tb128; do
  L=paper_1111_6900_b200/libgf2e_b200.so; [ $V = tb128 ] && L=build/variants/lib_tb128.so
  for n in 1024 8192; do GF2E_LIB_PATH=$L timeout 300 python tools/prof_ple.py 8 $n 4 2>&1 | tail -1 | sed "s/^/$V /"; done
  GF2E_LIB_PATH=$L timeout 300 python tools/prof_trsm.py 8 8192 16384 2>&1 | tail -1 | sed "s/^/$V /"
done 2>&1 | tee $O/ab.txt
GF2E_PDL=0 timeout 300 python tools/kineto_ple.py 8 1024 > $O/kineto_ple1024_nopdl.txt 2>&1; head -8 $O/kineto_ple1024_nopdl.txt
