# 2 GPUs: push-pack store variants (bulk copies vs SM float4 stores), one-way and in the step
mkdir -p gpurun_out
timeout 300 ./tools/nvlink_probe > gpurun_out/r2j_nvlink_probe.log 2>&1
for C in c5 c2; do
timeout 300 python tools/nvlink_push_ncu.py $C > gpurun_out/r2j_push_bulk_$C.log 2>&1
PACT_PUSH_STORES=1 timeout 300 python tools/nvlink_push_ncu.py $C > gpurun_out/r2j_push_stores_$C.log 2>&1
PACT_PUSH_STORES=1 timeout 600 ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,nvltx__bytes_data_protocol.sum --clock-control none -k regex:pack_lm -c 4 --csv --log-file gpurun_out/r2j_ncu_push_stores_$C.csv python tools/nvlink_push_ncu.py $C 1 > gpurun_out/r2j_ncu_push_stores_$C.log 2>&1
done
for C in c5 c2 c4; do
PACT_PUSH_STORES=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29800 bench.py --gpus 2 --config $C --no-cpu-baseline --no-e2e > gpurun_out/r2j_bench_${C}_stores_n2.json 2> gpurun_out/r2j_bench_${C}_stores_n2.err
done
for G in 8 16 32; do
for C in c5 c2; do
PACT_P2P_COPIER=$G timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29801 bench.py --gpus 2 --config $C --no-cpu-baseline --no-e2e > gpurun_out/r2j_bench_${C}_copier${G}_n2.json 2> gpurun_out/r2j_bench_${C}_copier${G}_n2.err
done
done
PACT_P2P_COPIER=16 timeout 1200 python -m pytest tests/test_multi_gpu.py -x -m gpu -v -rA > gpurun_out/r2j_mgpu_copier16_n2.log 2>&1
tail -2 gpurun_out/r2j_mgpu_copier16_n2.log
