"""Device timeline (torch.profiler / CUPTI) of one bucketed masked_allreduce
step on rank 0: kernel, stream, start, duration -- shows whether pack(b+1),
the exchange of b and unpack(b-1) actually overlap. torchrun, N ranks.

    python -m torch.distributed.run --nproc-per-node 2 tools/bucket_timeline.py c3 16 0.75 [nccl|p2p|auto]

bucket MB 0 = the library's AUTO plan (equal-chunk buckets on the green-
context SM partition when the packed vector is >= 24 MB).
"""
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2505_18563_b200 as pb  # noqa: E402
from paper_2505_18563_b200 import synth  # noqa: E402

CFG = {"c2": ("resnet50", 0.8), "c3": ("vgg19", 0.95), "c4": ("bert-base", 0.5), "c5": ("gpt2-medium", 0.9)}


def main():
    cfg = sys.argv[1]
    mb = float(sys.argv[2])
    os.environ["PACT_BUCKET_GRID_FRAC"] = sys.argv[3]
    tr = {"auto": 0, "nccl": 1, "p2p": 2}[sys.argv[4] if len(sys.argv) > 4 else "nccl"]
    model, ratio = CFG[cfg]
    rank = int(os.environ["RANK"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    comm = pb.Comm.from_process_group()
    shape = synth.model_shape(model)
    n = shape.total
    w = synth.weights_device(shape, 1234, synth.W_REAL)
    mask = pb.magnitude_prune(w, ratio)
    del w
    g = torch.empty(n, device="cuda")
    pb.synth_fill(g, synth.grad_seed(rank, 0), synth.G_FULL)
    out = torch.empty_like(g)
    pol = pb.SyncPolicy(transport=tr, bucket_bytes=int(mb * (1 << 20)))
    for i in range(4):
        pb.masked_allreduce(g, mask, pb.TrackerStatus.Stable, i, comm, policy=pol, out=out)
    torch.cuda.synchronize()
    dist.barrier()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        torch.cuda._sleep(2_000_000)
        pb.masked_allreduce(g, mask, pb.TrackerStatus.Stable, 9, comm, policy=pol, out=out)
        torch.cuda.synchronize()
    if rank == 0:
        evs = [e for e in prof.events() if e.device_type.name == "CUDA" and "sleep" not in e.name]
        evs.sort(key=lambda e: e.time_range.start)
        t0 = evs[0].time_range.start
        for e in evs:
            name = e.name.replace("(anonymous namespace)::", "").replace("void ", "").replace("pactk::", "").split("(")[0]
            print(f"{e.time_range.start - t0:8.1f} {e.time_range.elapsed_us():7.1f} s{getattr(e, 'device_resource_id', '?')}  {name[:60]}",
                  flush=True)
    dist.barrier()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
