# 2 GPUs: NVLink TX counters of the push pack; n=2 lines after the revert + address chains
mkdir -p gpurun_out
for C in c5 c2; do
timeout 300 python tools/nvlink_push_ncu.py $C > gpurun_out/r2h_push_$C.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,nvltx__bytes_data_protocol.sum,nvlrx__bytes.sum --clock-control none -k regex:pack_lm -c 6 --csv --log-file gpurun_out/r2h_ncu_push_$C.csv python tools/nvlink_push_ncu.py $C 1 > gpurun_out/r2h_ncu_push_$C.log 2>&1
done
timeout 1200 python -m pytest tests -x -m gpu -k "multi_gpu" -v -rA > gpurun_out/r2h_mgpu_n2.log 2>&1
tail -3 gpurun_out/r2h_mgpu_n2.log
for C in c5 c3 c2 c1 c4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29780 bench.py --gpus 2 --config $C --no-cpu-baseline > gpurun_out/r2h_bench_${C}_n2.json 2> gpurun_out/r2h_bench_${C}_n2.err
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29781 tools/bucket_timeline.py c3 0 1.0 auto > gpurun_out/r2h_bucket_timeline_c3_n2.txt 2>&1
