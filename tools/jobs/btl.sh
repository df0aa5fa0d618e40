mkdir -p gpurun_out
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 tools/bucket_timeline.py c3 16 0.75 nccl > gpurun_out/t27_btl_nccl16.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 tools/bucket_timeline.py c3 8 0.75 nccl > gpurun_out/t27_btl_nccl8.log 2>&1
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N tools/bucket_sweep.py c3 > gpurun_out/t27_sweep_c3_n$N.json 2> gpurun_out/t27_sweep_c3_n$N.err
done
