mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2a_bench_c5_n1.json 2> gpurun_out/r2a_bench_c5_n1.err
for C in c1 c2 c3 c4; do
timeout 600 python bench.py --config $C > gpurun_out/r2a_bench_${C}_n1.json 2> gpurun_out/r2a_bench_${C}_n1.err
done
timeout 600 python bench.py --prune per-layer --no-cpu-baseline --no-e2e > gpurun_out/r2a_bench_c5pl_n1.json 2> gpurun_out/r2a_bench_c5pl_n1.err
for N in 2 4; do
for C in c5 c1 c2 c3 c4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2970$N bench.py --gpus $N --config $C > gpurun_out/r2a_bench_${C}_n$N.json 2> gpurun_out/r2a_bench_${C}_n$N.err
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2971$N bench.py --gpus $N --config c4 --path sweep > gpurun_out/r2a_sweep_c4_n$N.json 2> gpurun_out/r2a_sweep_c4_n$N.err
done
timeout 900 python bench.py --impl reference > gpurun_out/r2a_ref_c5_n1.json 2> gpurun_out/r2a_ref_c5_n1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29721 bench.py --gpus 2 --impl reference > gpurun_out/r2a_ref_c5_n2.json 2> gpurun_out/r2a_ref_c5_n2.err
