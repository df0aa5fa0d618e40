mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -v -s --timeout 900 > gpurun_out/t30_pytest_all.log 2>&1
tail -5 gpurun_out/t30_pytest_all.log
timeout 600 python bench.py > gpurun_out/t30_bench_n1.json 2> gpurun_out/t30_bench_n1.err
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2957$N bench.py --gpus $N > gpurun_out/t30_bench_n$N.json 2> gpurun_out/t30_bench_n$N.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2958$N bench.py --gpus $N --config c3 --no-e2e > gpurun_out/t30_bench_c3_n$N.json 2> gpurun_out/t30_bench_c3_n$N.err
done
