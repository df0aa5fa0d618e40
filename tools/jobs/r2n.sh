# 4 GPUs: final multi-GPU parity at n=4 and the n=4 C5 line
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -k "multi_gpu" -v -rA > gpurun_out/r2n_mgpu_n4.log 2>&1
tail -3 gpurun_out/r2n_mgpu_n4.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29810 bench.py --gpus 4 > gpurun_out/r2n_bench_c5_n4.json 2> gpurun_out/r2n_bench_c5_n4.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29811 bench.py --gpus 4 --config c5 --prune per-layer --no-cpu-baseline --no-e2e > gpurun_out/r2n_bench_c5pl_n4.json 2> gpurun_out/r2n_bench_c5pl_n4.err
