mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29596 tools/bucket_sweep.py c3 tl > gpurun_out/t33_tl.log 2>&1
