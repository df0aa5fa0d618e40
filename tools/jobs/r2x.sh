# 1 GPU: the seeded first-time prune: parity (the whole prune suite) + C5 bench A/B
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_kernels.py tests/test_topk.py -x -q -m gpu > gpurun_out/r2x_pytest.log 2>&1
tail -2 gpurun_out/r2x_pytest.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2x_bench_c5_n1.json 2> gpurun_out/r2x_bench_c5_n1.err
PACT_PRUNE_COUNT_PASS=1 timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2x_bench_c5_count_n1.json 2> gpurun_out/r2x_bench_c5_count_n1.err
timeout 600 python tools/prune_probe.py > gpurun_out/r2x_prune_probe.log 2>&1
