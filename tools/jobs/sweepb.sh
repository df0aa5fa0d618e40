mkdir -p gpurun_out
for N in 2 4; do
for C in c2 c3 c4 c5; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N tools/bucket_sweep.py $C buckets > gpurun_out/t28_sweepb_${C}_n$N.json 2> gpurun_out/t28_sweepb_${C}_n$N.err
done
done
