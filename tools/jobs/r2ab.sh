# 2 GPUs: batched push A/B
mkdir -p gpurun_out
for C in c5 c2; do
timeout 300 python tools/nvlink_push_ncu.py $C > gpurun_out/r2ab_push_tma_$C.log 2>&1
PACT_PUSH_BATCH=1 timeout 300 python tools/nvlink_push_ncu.py $C > gpurun_out/r2ab_push_batch_$C.log 2>&1
done
grep -h "push pack" gpurun_out/r2ab_push_*.log
PACT_PUSH_BATCH=1 timeout 1200 python -m pytest tests/test_multi_gpu.py -x -m gpu -k "nccl_masked" -v -rA > gpurun_out/r2ab_mgpu_batch_n2.log 2>&1
tail -2 gpurun_out/r2ab_mgpu_batch_n2.log
for C in c5 c2 c4; do
PACT_PUSH_BATCH=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29850 bench.py --gpus 2 --config $C --no-cpu-baseline --no-e2e > gpurun_out/r2ab_bench_${C}_batch_n2.json 2> gpurun_out/r2ab_bench_${C}_batch_n2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29851 bench.py --gpus 2 --config $C --no-cpu-baseline --no-e2e > gpurun_out/r2ab_bench_${C}_tma_n2.json 2> gpurun_out/r2ab_bench_${C}_tma_n2.err
done
