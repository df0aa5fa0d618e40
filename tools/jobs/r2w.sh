# 1 GPU: every config on the final tree
mkdir -p gpurun_out
for C in c1 c2 c3 c4; do
timeout 600 python bench.py --config $C > gpurun_out/r2w_bench_${C}_n1.json 2> gpurun_out/r2w_bench_${C}_n1.err
done
timeout 600 python bench.py --prune per-layer --no-cpu-baseline > gpurun_out/r2w_bench_c5pl_n1.json 2> gpurun_out/r2w_bench_c5pl_n1.err
