# 1 GPU: prune_bitmap two vs three stages
mkdir -p gpurun_out
PACT_BITMAP_STAGES=3 timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu -k "reprune_sequence_paths or c5_reprune or prune_full_size_bitexact" > gpurun_out/r2t_pytest_s3.log 2>&1
tail -2 gpurun_out/r2t_pytest_s3.log
for i in 1 2; do
timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2t_bench_s2_$i.json 2> gpurun_out/r2t_bench_s2_$i.err
PACT_BITMAP_STAGES=3 timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2t_bench_s3_$i.json 2> gpurun_out/r2t_bench_s3_$i.err
done
