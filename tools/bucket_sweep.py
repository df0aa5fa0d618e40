"""Bucketed pipeline sweep (torchrun, N ranks): masked_allreduce step time
for bucket sizes x codec grid fractions x transports on one workload,
device-timed (CUDA events, L2 flushed, max over ranks). One JSON line.

    python -m torch.distributed.run --nproc-per-node N tools/bucket_sweep.py c3
"""
import json
import os
import statistics
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2505_18563_b200 as pb  # noqa: E402
from paper_2505_18563_b200 import synth  # noqa: E402

CFG = {"c2": ("resnet50", 0.8), "c3": ("vgg19", 0.95), "c4": ("bert-base", 0.5), "c5": ("gpt2-medium", 0.9)}


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
    model, ratio = CFG[cfg]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
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
    pb.enforce_gradient_sparsity(g, mask, out=g)
    out = torch.empty_like(g)
    flush = torch.empty(128 << 20, device="cuda")
    flush_r = torch.zeros(128 << 20, device="cuda")
    sink = torch.empty((), device="cuda")
    align = torch.zeros(1, device="cuda")

    def t_of(pol, k=10):
        for i in range(3):
            pb.masked_allreduce(g, mask, pb.TrackerStatus.Stable, i, comm, policy=pol, out=out)
        ts = []
        for i in range(k):
            flush.zero_()
            torch.sum(flush_r, dim=0, out=sink)
            dist.all_reduce(align)
            torch.cuda._sleep(2_000_000)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            r = pb.masked_allreduce(g, mask, pb.TrackerStatus.Stable, i, comm, policy=pol, out=out)
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        t = torch.tensor([statistics.median(ts)], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()), r.stats.buckets, r.stats.transport

    rows = []
    mode = sys.argv[2] if len(sys.argv) > 2 else "full"
    if mode == "buckets":  # B equal-chunk NCCL buckets at two grid fractions vs each single-bucket transport
        pbytes = mask.nnz() * 4
        singles = {}
        for transport, tn in ((pb.SyncPolicy.NCCL, "nccl"), (pb.SyncPolicy.P2P, "p2p"), (pb.SyncPolicy.AUTO, "auto")):
            t, nb, tr = t_of(pb.SyncPolicy(transport=transport))
            singles[tn] = t
            rows.append({"transport": tn, "buckets": nb, "us": round(t, 1), "used": tr})
        best1 = min(singles.values())
        for B in (2, 3, 4, 6, 8):
            for frac in (0.75, 1.0):
                os.environ["PACT_BUCKET_GRID_FRAC"] = str(frac)
                t, nb, tr = t_of(pb.SyncPolicy(transport=pb.SyncPolicy.NCCL, bucket_bytes=(pbytes + B - 1) // B))
                rows.append({"transport": "nccl", "buckets": nb, "frac": frac, "us": round(t, 1),
                             "vs_best_single": round(t / best1, 3)})
    if mode == "stab":  # repeated: single (each transport) vs 2 / 3 NCCL buckets at 0.75
        pbytes = mask.nnz() * 4
        os.environ["PACT_BUCKET_GRID_FRAC"] = "0.75"
        for rep in range(3):
            for label, pol in (("nccl1", pb.SyncPolicy(transport=pb.SyncPolicy.NCCL)),
                               ("p2p1", pb.SyncPolicy(transport=pb.SyncPolicy.P2P)),
                               ("nccl2", pb.SyncPolicy(transport=pb.SyncPolicy.NCCL, bucket_bytes=(pbytes + 1) // 2)),
                               ("nccl3", pb.SyncPolicy(transport=pb.SyncPolicy.NCCL, bucket_bytes=(pbytes + 2) // 3))):
                t, nb, tr = t_of(pol)
                rows.append({"rep": rep, "policy": label, "buckets": nb, "us": round(t, 1)})
    for transport, tn in (((pb.SyncPolicy.NCCL, "nccl"), (pb.SyncPolicy.P2P, "p2p")) if mode == "full" else ()):
        base, _, _ = t_of(pb.SyncPolicy(transport=transport))
        rows.append({"transport": tn, "bucket_mb": 0, "frac": None, "us": round(base, 1)})
        for mb in (2, 4, 8, 16):
            for frac in (0.25, 0.5, 0.75, 1.0):
                os.environ["PACT_BUCKET_GRID_FRAC"] = str(frac)
                t, nb, tr = t_of(pb.SyncPolicy(transport=transport, bucket_bytes=mb << 20))
                rows.append({"transport": tn, "bucket_mb": mb, "frac": frac, "buckets": nb, "us": round(t, 1),
                             "vs_single": round(t / base, 3)})
    if rank == 0:
        print(json.dumps({"config": cfg, "n": world, "nnz": mask.nnz(), "rows": rows}), flush=True)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
