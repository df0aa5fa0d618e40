# 4 GPUs: every config on the final tree
mkdir -p gpurun_out
for C in c1 c2 c3 c4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29840 bench.py --gpus 4 --config $C > gpurun_out/r2v_bench_${C}_n4.json 2> gpurun_out/r2v_bench_${C}_n4.err
done
timeout 1500 python -m pytest tests -m gpu -k "multi_gpu" -v -rA > gpurun_out/r2v_mgpu_n4.log 2>&1
tail -3 gpurun_out/r2v_mgpu_n4.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29841 bench.py --gpus 4 > gpurun_out/r2v_bench_c5_n4.json 2> gpurun_out/r2v_bench_c5_n4.err
