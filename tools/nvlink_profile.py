"""NVLink counters of the n = 2 P2P exchange kernels (one rank profiled).

Rank 0 runs under ncu, rank 1 plainly (two processes sharing a file-based
NCCL id, not torchrun): the profiled consumer kernels only wait on flags the
peer has already raised, so kernel replay is safe; NCCL kernels are excluded
(their replay would wait on the peer forever).

    ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,... \
        -k regex:"pack_lm|unpack" --csv --log-file nvl.csv \
        python tools/nvlink_profile.py 0 2 /tmp/id c2 &
    python tools/nvlink_profile.py 1 2 /tmp/id c2
"""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2505_18563_b200 as pb  # noqa: E402
from paper_2505_18563_b200 import synth  # noqa: E402

CFG = {"c2": ("resnet50", 0.8), "c3": ("vgg19", 0.95), "c5": ("gpt2-medium", 0.9)}


def main():
    rank, world, idf, cfg = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4]
    steps = int(sys.argv[5]) if len(sys.argv) > 5 else 4
    torch.cuda.set_device(rank)
    if rank == 0:
        with open(idf + ".tmp", "wb") as f:
            f.write(pb.Comm.unique_id())
        os.replace(idf + ".tmp", idf)
    while not os.path.exists(idf):
        time.sleep(0.01)
    comm = pb.Comm(rank, world, open(idf, "rb").read())
    model, ratio = CFG[cfg]
    shape = synth.model_shape(model)
    w = synth.weights_device(shape, 1234, synth.W_REAL)
    mask = pb.magnitude_prune(w, ratio)
    del w
    g = torch.empty(shape.total, device="cuda")
    pb.synth_fill(g, synth.grad_seed(rank, 0), synth.G_FULL)
    pol = pb.SyncPolicy(transport=pb.SyncPolicy.P2P)
    for e in range(steps):
        r = pb.masked_allreduce(g, mask, pb.TrackerStatus.Stable, e, comm, policy=pol)
        comm.check(120_000)
    print(f"[rank {rank}] {cfg} nnz={mask.nnz()} packed bytes per direction={4 * mask.nnz()} "
          f"transport={r.stats.transport}", flush=True)
    os._exit(0)


if __name__ == "__main__":
    main()
