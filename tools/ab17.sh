O=gpurun_out/ab17; mkdir -p $O
for r in 1 2; do for V in gml8 gml24; do
 for E in 9 10; do GF2E_LIB_PATH=build/variants/lib_$V.so timeout 300 python tools/prof_trsm.py $E 8192 16384 2>&1 | tail -1 | sed "s/^/$V /"; done
 GF2E_LIB_PATH=build/variants/lib_$V.so timeout 300 python tools/prof_ple.py 10 8192 2 2>&1 | tail -1 | sed "s/^/$V /"
 GF2E_LIB_PATH=build/variants/lib_$V.so timeout 300 python tools/prof_ple.py 8 8192 2 2>&1 | tail -1 | sed "s/^/$V /"
done; done 2>&1 | tee $O/ab.txt
