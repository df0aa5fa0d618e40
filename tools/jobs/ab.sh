mkdir -p gpurun_out
N=4
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29591 bench.py --gpus $N --config c3 --no-e2e > gpurun_out/t31_c3_auto.json 2> gpurun_out/t31_c3_auto.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29592 bench.py --gpus $N --config c3 --no-e2e --bucket-mb -1 > gpurun_out/t31_c3_single.json 2> gpurun_out/t31_c3_single.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29593 bench.py --gpus $N --config c3 --no-e2e --bucket-mb 9.6 > gpurun_out/t31_c3_b96.json 2> gpurun_out/t31_c3_b96.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29594 tools/bucket_sweep.py c3 stab > gpurun_out/t31_stab.json 2> gpurun_out/t31_stab.err
