# 2 GPUs: every config on the final tree
mkdir -p gpurun_out
for C in c1 c2 c3 c4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29830 bench.py --gpus 2 --config $C > gpurun_out/r2u_bench_${C}_n2.json 2> gpurun_out/r2u_bench_${C}_n2.err
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29831 bench.py --gpus 2 --config c4 --path sweep > gpurun_out/r2u_sweep_c4_n2.json 2> gpurun_out/r2u_sweep_c4_n2.err
