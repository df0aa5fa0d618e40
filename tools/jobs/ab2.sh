mkdir -p gpurun_out
for N in 4 2; do
for C in c3 c5; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2960$N bench.py --gpus $N --config $C --no-e2e > gpurun_out/t34_${C}_auto_n$N.json 2> gpurun_out/t34_${C}_auto_n$N.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2961$N bench.py --gpus $N --config $C --no-e2e --bucket-mb -1 > gpurun_out/t34_${C}_single_n$N.json 2> gpurun_out/t34_${C}_single_n$N.err
done
done
