mkdir -p gpurun_out
for G in "PACT_GREEN=1 PACT_NCCL_SMS=16" "PACT_GREEN=1 PACT_NCCL_SMS=32" "PACT_GREEN=1 PACT_NCCL_SMS=8" "PACT_GREEN=0"; do
tag=$(echo $G | tr ' =' '__')
env $G timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29641 tools/bucket_sweep.py c3 green > gpurun_out/t37_green_$tag.json 2> gpurun_out/t37_green_$tag.err
done
