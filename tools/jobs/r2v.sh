# 4 GPUs: every config on the final tree
mkdir -p gpurun_out
for C in c1 c2 c3 c4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29840 bench.py --gpus 4 --config $C > gpurun_out/r2v_bench_${C}_n4.json 2> gpurun_out/r2v_bench_${C}_n4.err
done
