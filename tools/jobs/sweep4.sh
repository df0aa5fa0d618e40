mkdir -p gpurun_out
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N tools/bucket_sweep.py c3 > gpurun_out/t25_sweep_c3_n$N.json 2> gpurun_out/t25_sweep_c3_n$N.err
tail -c 300 gpurun_out/t25_sweep_c3_n$N.err
done
