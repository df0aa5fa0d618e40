# 1 GPU: per-layer reuse parity + the per-layer headline, the prune suite
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu -k "per_layer or reprune or prune_full_size or prune_changed" > gpurun_out/r2q_pytest.log 2>&1
tail -3 gpurun_out/r2q_pytest.log
timeout 900 python bench.py --prune per-layer --no-cpu-baseline --no-e2e > gpurun_out/r2q_bench_c5pl_n1.json 2> gpurun_out/r2q_bench_c5pl_n1.err
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2q_bench_c5_n1.json 2> gpurun_out/r2q_bench_c5_n1.err
