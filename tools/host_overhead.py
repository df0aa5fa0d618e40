"""Diagnostic: host time per bench iteration vs device time (N ranks).
torchrun --nproc-per-node 2 tools/host_overhead.py"""
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_18563_b200 as pb  # noqa: E402
from paper_2505_18563_b200 import synth  # noqa: E402

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
comm = pb.Comm.from_process_group()
shape = synth.model_shape("resnet50")
n = shape.total
w = synth.weights_device(shape, 1234, synth.W_REAL, device=dev)
mask = pb.magnitude_prune(w, 0.8)
tr = pb.MaskTracker(3)
for _ in range(4):
    tr.observe(mask)
g = torch.empty(n, device=dev)
pb.synth_fill(g, synth.grad_seed(rank, 0), synth.G_FULL)
out = torch.empty_like(g)
align = torch.zeros(1, device=dev)
flush = torch.empty(128 << 20, device=dev)
for mode in ("plain", "flush", "flush+align"):
    for i in range(10):
        pb.masked_allreduce(g, mask, tr.status(), i, comm, out=out)
    torch.cuda.synchronize()
    dist.barrier()
    K = 50
    t0 = time.perf_counter()
    host = []
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    for i in range(K):
        if "flush" in mode:
            flush.zero_()
        if "align" in mode:
            dist.all_reduce(align)
        h0 = time.perf_counter()
        pb.masked_allreduce(g, mask, tr.status(), i, comm, out=out)
        host.append(time.perf_counter() - h0)
    t_host = time.perf_counter() - t0
    ev1.record()
    torch.cuda.synchronize()
    t_dev = ev0.elapsed_time(ev1) * 1e-3
    if rank == 0:
        print(f"{mode}: host loop {t_host / K * 1e6:.1f} us/iter (masked_allreduce call {sorted(host)[K // 2] * 1e6:.1f} us), "
              f"device {t_dev / K * 1e6:.1f} us/iter", flush=True)
comm.close()
dist.destroy_process_group()
