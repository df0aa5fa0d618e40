mkdir -p gpurun_out
for N in 4 2; do
for C in c3 c4 c5; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2956$N tools/bucket_sweep.py $C stab > gpurun_out/t29_stab_${C}_n$N.json 2> gpurun_out/t29_stab_${C}_n$N.err
done
done
