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

    def t_of_nosync(pol, k=10):
        """bench.py's loop: no per-step synchronisation, host runs ahead"""
        for i in range(3):
            pb.masked_allreduce(g, mask, pb.TrackerStatus.Stable, i, comm, policy=pol, out=out)
        evs = []
        for i in range(k):
            flush.zero_()
            torch.sum(flush_r, dim=0, out=sink)
            dist.all_reduce(align)
            torch.cuda._sleep(2_000_000)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            r = pb.masked_allreduce(g, mask, pb.TrackerStatus.Stable, i, comm, policy=pol, out=out)
            b.record()
            evs.append((a, b))
        torch.cuda.synchronize()
        ts = [a.elapsed_time(b) * 1e3 for a, b in evs]
        t = torch.tensor([statistics.median(ts)], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()), r.stats.buckets, r.stats.transport

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
    if mode == "tl":  # timelines of a 3-bucket step before and after 2-bucket steps
        from torch.profiler import ProfilerActivity, profile
        pbytes = mask.nnz() * 4
        os.environ["PACT_BUCKET_GRID_FRAC"] = "0.75"
        n3 = pb.SyncPolicy(transport=pb.SyncPolicy.NCCL, bucket_bytes=(pbytes + 2) // 3)
        n2 = pb.SyncPolicy(transport=pb.SyncPolicy.NCCL, bucket_bytes=(pbytes + 1) // 2)
        for tag, warm in (("before", n3), ("after2", n2)):
            t_of(warm, 3)
            t_of(n3, 3)
            dist.barrier()
            with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
                torch.cuda._sleep(2_000_000)
                pb.masked_allreduce(g, mask, pb.TrackerStatus.Stable, 77, comm, policy=n3, out=out)
                torch.cuda.synchronize()
            if rank == 0:
                evs = [e for e in prof.events() if e.device_type.name == "CUDA" and "sleep" not in e.name]
                evs.sort(key=lambda e: e.time_range.start)
                t0 = evs[0].time_range.start
                print("----", tag, flush=True)
                for e in evs:
                    nm = e.name.replace("(anonymous namespace)::", "").replace("void ", "").replace("pactk::", "")
                    print(f"{e.time_range.start - t0:8.1f} {e.time_range.elapsed_us():7.1f} "
                          f"s{getattr(e, 'device_resource_id', '?')}  {nm.split('(')[0][:60]}", flush=True)
            dist.barrier()
    if mode == "sync":  # per-step sync (this tool) vs host running ahead (bench.py)
        pbytes = mask.nnz() * 4
        os.environ["PACT_BUCKET_GRID_FRAC"] = "0.75"
        n3 = pb.SyncPolicy(transport=pb.SyncPolicy.NCCL, bucket_bytes=(pbytes + 2) // 3)
        n1 = pb.SyncPolicy(transport=pb.SyncPolicy.NCCL)
        for label, fn, pol in (("n1_sync", t_of, n1), ("n1_nosync", t_of_nosync, n1), ("n3_sync", t_of, n3),
                               ("n3_nosync", t_of_nosync, n3), ("n3_sync_again", t_of, n3)):
            t, nb, tr = fn(pol)
            rows.append({"policy": label, "buckets": nb, "us": round(t, 1)})
    if mode == "tlnosync":  # device timeline of back-to-back bucketed steps (host ahead)
        from torch.profiler import ProfilerActivity, profile
        pbytes = mask.nnz() * 4
        os.environ["PACT_BUCKET_GRID_FRAC"] = "0.75"
        n3 = pb.SyncPolicy(transport=pb.SyncPolicy.NCCL, bucket_bytes=(pbytes + 2) // 3)
        t_of(n3, 3)
        dist.barrier()
        with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
            for i in range(3):
                flush.zero_()
                torch.sum(flush_r, dim=0, out=sink)
                dist.all_reduce(align)
                torch.cuda._sleep(2_000_000)
                pb.masked_allreduce(g, mask, pb.TrackerStatus.Stable, 50 + i, comm, policy=n3, out=out)
            torch.cuda.synchronize()
        if rank == 0:
            evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
            evs.sort(key=lambda e: e.time_range.start)
            t0 = evs[0].time_range.start
            for e in evs:
                nm = e.name.replace("(anonymous namespace)::", "").replace("void ", "").replace("pactk::", "")
                print(f"{e.time_range.start - t0:8.1f} {e.time_range.elapsed_us():7.1f} "
                      f"s{getattr(e, 'device_resource_id', '?')}  {nm.split('(')[0][:60]}", flush=True)
    if mode == "green2":  # host ahead (bench loop): single per transport vs B buckets on the SM partition
        pbytes = mask.nnz() * 4
        for label, pol in (("nccl1", pb.SyncPolicy(transport=pb.SyncPolicy.NCCL)),
                           ("p2p1", pb.SyncPolicy(transport=pb.SyncPolicy.P2P))):
            t, _, _ = t_of_nosync(pol)
            rows.append({"policy": label, "us": round(t, 1)})
        for B in (2, 3, 4, 6):
            pol = pb.SyncPolicy(transport=pb.SyncPolicy.NCCL, bucket_bytes=(pbytes + B - 1) // B)
            for frac in (0.75, 1.0):
                os.environ["PACT_BUCKET_GRID_FRAC"] = str(frac)
                t, nb, _ = t_of_nosync(pol)
                rows.append({"B": nb, "frac": frac, "us": round(t, 1), "nccl_sms": os.environ.get("PACT_NCCL_SMS", "16")})
    if mode == "green":  # SM partition sizes for the exchange, host ahead (bench loop) and synced
        pbytes = mask.nnz() * 4
        n1 = pb.SyncPolicy(transport=pb.SyncPolicy.NCCL)
        t, _, _ = t_of_nosync(n1)
        rows.append({"policy": "single_nosync", "us": round(t, 1)})
        for B in (2, 3):
            pol = pb.SyncPolicy(transport=pb.SyncPolicy.NCCL, bucket_bytes=(pbytes + B - 1) // B)
            for frac in (0.5, 0.75, 1.0):
                os.environ["PACT_BUCKET_GRID_FRAC"] = str(frac)
                t1, nb, _ = t_of_nosync(pol)
                t2, _, _ = t_of(pol)
                rows.append({"B": nb, "frac": frac, "nosync_us": round(t1, 1), "sync_us": round(t2, 1),
                             "nccl_sms": os.environ.get("PACT_NCCL_SMS", "16"),
                             "green": os.environ.get("PACT_GREEN", "1")})
    if mode == "order":  # is the bucketed pipeline sensitive to what ran before (P2P setup)?
        pbytes = mask.nnz() * 4
        os.environ["PACT_BUCKET_GRID_FRAC"] = "0.75"
        n3 = pb.SyncPolicy(transport=pb.SyncPolicy.NCCL, bucket_bytes=(pbytes + 2) // 3)
        for label, pol in (("nccl3_first", n3), ("nccl1", pb.SyncPolicy(transport=pb.SyncPolicy.NCCL)),
                           ("nccl3_after_nccl1", n3), ("p2p1", pb.SyncPolicy(transport=pb.SyncPolicy.P2P)),
                           ("nccl3_after_p2p", n3)):
            t, nb, tr = t_of(pol)
            rows.append({"policy": label, "buckets": nb, "us": round(t, 1)})
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
