# 1 GPU: address-chain split in pack/unpack: parity + every config
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_kernels.py tests/test_ternary.py tests/test_topk.py tests/test_fp16_wire.py -x -q -m gpu > gpurun_out/r2g_pytest.log 2>&1
tail -3 gpurun_out/r2g_pytest.log
for C in c1 c2 c3 c4; do
timeout 600 python bench.py --config $C --no-cpu-baseline > gpurun_out/r2g_bench_${C}_n1.json 2> gpurun_out/r2g_bench_${C}_n1.err
done
timeout 900 python bench.py > gpurun_out/r2g_bench_c5_n1.json 2> gpurun_out/r2g_bench_c5_n1.err
for C in c1 c2; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"unpack_kernel|pack_lm" --launch-skip 10 -c 2 -o gpurun_out/r2g_full_${C} python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2g_ncu_full_$C.log 2>&1
done
