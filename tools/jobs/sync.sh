mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29621 tools/bucket_sweep.py c3 sync > gpurun_out/t35_sync.json 2> gpurun_out/t35_sync.err
PACT_BENCH_NO_NVML=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29622 bench.py --gpus 4 --config c3 --no-e2e > gpurun_out/t35_c3_nonvml.json 2> gpurun_out/t35_c3_nonvml.err
