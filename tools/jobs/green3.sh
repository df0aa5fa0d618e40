mkdir -p gpurun_out
PACT_DEBUG=1 python - <<'PY' 2>&1 | grep -v Warn | tail -5
import torch, paper_2505_18563_b200 as pb
torch.cuda.set_device(0)
print(pb.Context.get().handle)
PY
PACT_DEBUG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29652 tools/bucket_sweep.py c3 green > gpurun_out/t39_green.json 2> gpurun_out/t39_green.err
grep pact gpurun_out/t39_green.err | head -3
