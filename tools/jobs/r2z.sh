# 2 GPUs: final multi-GPU parity at n=2 and the n=2 C5 line on the final tree
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -k "multi_gpu" -v -rA > gpurun_out/r2z_mgpu_n2.log 2>&1
tail -3 gpurun_out/r2z_mgpu_n2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29820 bench.py --gpus 2 > gpurun_out/r2z_bench_c5_n2.json 2> gpurun_out/r2z_bench_c5_n2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29821 bench.py --gpus 2 --impl reference > gpurun_out/r2z_ref_c5_n2.json 2> gpurun_out/r2z_ref_c5_n2.err
