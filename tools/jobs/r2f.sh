# 2 GPUs: slot-layout push parity + n=2 lines, NVLink metric names, probe under ncu
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -m gpu -k "multi_gpu" -v -rA > gpurun_out/r2f_mgpu_n2.log 2>&1
tail -3 gpurun_out/r2f_mgpu_n2.log
for C in c5 c2 c4 c1; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29770 bench.py --gpus 2 --config $C --no-cpu-baseline > gpurun_out/r2f_bench_${C}_n2.json 2> gpurun_out/r2f_bench_${C}_n2.err
done
PACT_P2P_TRACE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29771 bench.py --gpus 2 --config c5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2f_trace_c5_n2.json 2> gpurun_out/r2f_trace_c5_n2.err
ncu --query-metrics --chip gb100 2>/dev/null | grep -i -E "nvl|nvlink" > gpurun_out/r2f_ncu_nvl_metrics.txt
ncu --query-metrics 2>/dev/null | grep -i -E "nvl" >> gpurun_out/r2f_ncu_nvl_metrics.txt
M=$(grep -o -E "^nvl[a-z_]*__[a-z_]*bytes[a-z_]*" gpurun_out/r2f_ncu_nvl_metrics.txt | sort -u | head -6 | sed 's/$/.sum/' | paste -sd, -)
echo "metrics: $M" > gpurun_out/r2f_ncu_probe.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,$M --clock-control none -c 60 --csv --log-file gpurun_out/r2f_ncu_probe.csv ./tools/nvlink_probe >> gpurun_out/r2f_ncu_probe.log 2>&1
