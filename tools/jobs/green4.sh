mkdir -p gpurun_out
for N in 4 2; do
for C in c3 c4 c5; do
for SMS in 8 16 32; do
PACT_NCCL_SMS=$SMS timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2966$N tools/bucket_sweep.py $C green2 > gpurun_out/t41_g_${C}_n${N}_s$SMS.json 2> gpurun_out/t41_g_${C}_n${N}_s$SMS.err
done
done
done
