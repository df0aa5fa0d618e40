"""Fail-fast worker for tests/test_multi_gpu.py: two processes, one per GPU
(plain processes, not torchrun, which would tear the survivor down too).
Both run healthy masked_allreduce steps; then rank 1 is SIGKILLed in the
middle of a step (its kernels enqueued, the process gone) and rank 0 must
see LinkError within the link timeout -- the reference's
SimCluster::poison / LinkError contract (collective.cpp:430-458,
trainer.cpp:416-437) -- and every later call must fail at once.

    python tests/mp_failfast_worker.py <rank> <world> <id-file> <transport>
"""
import os
import signal
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2505_18563_b200 as pb  # noqa: E402


def main():
    rank, world, idf, transport = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4]
    torch.cuda.set_device(rank)
    if rank == 0:
        uid = pb.Comm.unique_id()
        with open(idf + ".tmp", "wb") as f:
            f.write(uid)
        os.replace(idf + ".tmp", idf)
    else:
        while not os.path.exists(idf):
            time.sleep(0.01)
        uid = open(idf, "rb").read()
    comm = pb.Comm(rank, world, uid)
    n = 1 << 22
    g = torch.randn(n, device="cuda")
    bits = torch.arange(n, device="cuda") % 3 == 0
    mask = pb.SparsityMask.from_bits(bits.cpu())
    g = pb.enforce_gradient_sparsity(g, mask)
    pol = pb.SyncPolicy(transport={"nccl": 1, "p2p": 2}[transport])
    for e in range(3):
        r = pb.masked_allreduce(g, mask, pb.TrackerStatus.Stable, e, comm, policy=pol)
        comm.check(60_000)
        assert r.stats.mode_used == pb.SyncMode.PackedAllReduce
    print(f"[rank {rank}] healthy steps done", flush=True)
    if rank == 1:
        time.sleep(0.5)
        pb.masked_allreduce(g, mask, pb.TrackerStatus.Stable, 3, comm, policy=pol)  # enqueued...
        os.kill(os.getpid(), signal.SIGKILL)  # ...and gone mid-step
    time.sleep(0.5)
    t0 = time.time()
    code = None
    try:
        for e in range(3, 8):
            pb.masked_allreduce(g, mask, pb.TrackerStatus.Stable, e, comm, policy=pol)
            comm.check()
    except pb.Error as ex:
        code = ex.code
        print(f"[rank 0] {ex.code.name} after {time.time() - t0:.2f} s: {ex}", flush=True)
    if code != pb.Errc.LinkError:
        print("[rank 0] FAIL: no LinkError", flush=True)
        sys.exit(1)
    dt = time.time() - t0
    limit = float(os.environ.get("PACT_LINK_TIMEOUT_MS", "30000")) / 1000.0
    if dt > 2.5 * limit + 5.0:
        print(f"[rank 0] FAIL: LinkError took {dt:.1f} s (timeout {limit} s)", flush=True)
        sys.exit(1)
    t1 = time.time()
    try:
        pb.masked_allreduce(g, mask, pb.TrackerStatus.Stable, 9, comm, policy=pol)
        print("[rank 0] FAIL: a call on the poisoned comm succeeded", flush=True)
        sys.exit(1)
    except pb.Error as ex:
        if ex.code != pb.Errc.LinkError or time.time() - t1 > 0.5:
            print(f"[rank 0] FAIL: poisoned comm answered {ex.code.name} after {time.time() - t1:.2f} s", flush=True)
            sys.exit(1)
    assert comm.failed
    print(f"[rank 0] fail-fast ok ({transport}): LinkError {dt:.2f} s after the peer died, "
          f"then immediately", flush=True)
    os._exit(0)  # skip teardown of a comm whose peer is gone


if __name__ == "__main__":
    main()
