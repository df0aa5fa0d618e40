mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29631 tools/bucket_sweep.py c3 tlnosync > gpurun_out/t36_tln.log 2>&1
