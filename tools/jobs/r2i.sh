# 4 GPUs: final multi-GPU parity + every config at n=4 + bucket timeline
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -m gpu -k "multi_gpu" -v -rA > gpurun_out/r2i_mgpu_n4.log 2>&1
tail -3 gpurun_out/r2i_mgpu_n4.log
for C in c5 c1 c2 c3 c4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29790 bench.py --gpus 4 --config $C --no-cpu-baseline > gpurun_out/r2i_bench_${C}_n4.json 2> gpurun_out/r2i_bench_${C}_n4.err
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29791 bench.py --gpus 4 --config c4 --path sweep > gpurun_out/r2i_sweep_c4_n4.json 2> gpurun_out/r2i_sweep_c4_n4.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29792 tools/bucket_timeline.py c5 0 1.0 auto > gpurun_out/r2i_bucket_timeline_c5_n4.txt 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29793 tools/bucket_timeline.py c3 0 1.0 auto > gpurun_out/r2i_bucket_timeline_c3_n4.txt 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29794 bench.py --gpus 4 --impl reference > gpurun_out/r2i_ref_c5_n4.json 2> gpurun_out/r2i_ref_c5_n4.err
