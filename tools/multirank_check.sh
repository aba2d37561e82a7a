# functional check of the multi-rank bench flow on a one-GPU box (gloo, every rank on cuda:0;
# not a measurement): N = 2 and 4, configs 2 and 3
O=gpurun_out/multirank; mkdir -p $O
for N in 2 4; do
 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2960$N \
   bench.py --gpus $N --config 2 --dist-backend gloo-shared-gpu --steps 3 --warmup 3 > $O/gloo_n${N}_c2.json 2> $O/gloo_n${N}_c2.err
 echo "N=$N rc=$?"; tail -c 600 $O/gloo_n${N}_c2.json; echo
done
