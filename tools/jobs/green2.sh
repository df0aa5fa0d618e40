mkdir -p gpurun_out
PACT_DEBUG=1 PACT_NCCL_SMS=16 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29651 tools/bucket_sweep.py c3 green > gpurun_out/t38_green.json 2> gpurun_out/t38_green.err
grep pact gpurun_out/t38_green.err | head
