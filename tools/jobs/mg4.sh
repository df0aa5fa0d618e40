set -x
timeout 1200 python -m pytest tests -m gpu -v -s -k "multi_gpu" --timeout 600 > gpurun_out/t24_mgpu4.log 2>&1
tail -8 gpurun_out/t24_mgpu4.log
for N in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/t24_bench_c5_n$N.json 2> gpurun_out/t24_bench_c5_n$N.err
tail -c 600 gpurun_out/t24_bench_c5_n$N.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $N --steps 20 --warmup 5 --config c3 > gpurun_out/t24_bench_c3_n$N.json 2> gpurun_out/t24_bench_c3_n$N.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus $N --steps 20 --warmup 5 --config c3 --bucket-mb 16 > gpurun_out/t24_bench_c3b16_n$N.json 2> gpurun_out/t24_bench_c3b16_n$N.err
done
