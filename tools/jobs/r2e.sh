# 2 GPUs: NVML NVLink counter probe, n=2 bench lines after the uniform-scale unpack fast path
mkdir -p gpurun_out
timeout 300 python tools/nvml_probe.py > gpurun_out/r2e_nvml_probe.log 2>&1
for C in c5 c3 c2 c1 c4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29760 bench.py --gpus 2 --config $C --no-cpu-baseline > gpurun_out/r2e_bench_${C}_n2.json 2> gpurun_out/r2e_bench_${C}_n2.err
done
PACT_P2P_TRACE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29761 bench.py --gpus 2 --config c5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2e_trace_c5_n2.json 2> gpurun_out/r2e_trace_c5_n2.err
timeout 1200 python -m pytest tests -x -m gpu -k "multi_gpu" -v -rA > gpurun_out/r2e_mgpu_n2.log 2>&1
tail -3 gpurun_out/r2e_mgpu_n2.log
