# 2 GPUs: NVLink probe (SM stores vs copy engines), n=2 bench lines with NVML NVLink counters
mkdir -p gpurun_out
timeout 300 ./tools/nvlink_probe > gpurun_out/r2c_nvlink_probe.log 2>&1
for C in c5 c3 c2; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29730 bench.py --gpus 2 --config $C --no-cpu-baseline > gpurun_out/r2c_bench_${C}_n2.json 2> gpurun_out/r2c_bench_${C}_n2.err
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29741 bench.py --gpus 2 --config c5 --transport nccl --no-cpu-baseline --no-e2e > gpurun_out/r2c_bench_c5_nccl_n2.json 2> gpurun_out/r2c_bench_c5_nccl_n2.err
timeout 1200 python -m pytest tests -x -q -m gpu -k "multi_gpu" -v > gpurun_out/r2c_mgpu_n2.log 2>&1
tail -3 gpurun_out/r2c_mgpu_n2.log
# copy-engine push A/B (n = 2)
for B in 4 8 16; do
for C in c5 c3; do
PACT_P2P_CE=$B timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29750 bench.py --gpus 2 --config $C --no-cpu-baseline --no-e2e > gpurun_out/r2c_bench_${C}_ce${B}_n2.json 2> gpurun_out/r2c_bench_${C}_ce${B}_n2.err
done
done
PACT_P2P_CE=8 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29751 bench.py --gpus 2 --config c2 --no-cpu-baseline --no-e2e > gpurun_out/r2c_bench_c2_ce8_n2.json 2> gpurun_out/r2c_bench_c2_ce8_n2.err
PACT_P2P_CE=8 timeout 1200 python -m pytest tests/test_multi_gpu.py -x -q -m gpu -v > gpurun_out/r2c_mgpu_ce8_n2.log 2>&1
tail -3 gpurun_out/r2c_mgpu_ce8_n2.log
