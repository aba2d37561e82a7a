O=gpurun_out/k1024; mkdir -p $O
for E in 8; do
timeout 300 python tools/kineto_ple.py $E 1024 > $O/kineto_ple1024_e$E.txt 2>&1
GF2E_PDL=0 timeout 300 python tools/kineto_ple.py $E 1024 > $O/kineto_ple1024_e${E}_nopdl.txt 2>&1
done
timeout 300 python tools/prof_ple.py 8 1024 5 > $O/prof_ple1024.txt 2>&1
cat $O/*.txt
