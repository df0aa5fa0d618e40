mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -v -s -k "multi_gpu" --timeout 900 > gpurun_out/t42_mgpu.log 2>&1
tail -9 gpurun_out/t42_mgpu.log
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2967$N bench.py --gpus $N > gpurun_out/t42_bench_n$N.json 2> gpurun_out/t42_bench_n$N.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2968$N bench.py --gpus $N --config c3 --no-e2e > gpurun_out/t42_bench_c3_n$N.json 2> gpurun_out/t42_bench_c3_n$N.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2969$N bench.py --gpus $N --config c3 --no-e2e --bucket-mb -1 > gpurun_out/t42_bench_c3single_n$N.json 2> gpurun_out/t42_bench_c3single_n$N.err
done
