mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29595 tools/bucket_sweep.py c3 order > gpurun_out/t32_order.json 2> gpurun_out/t32_order.err
