"""N > 1 paths.

* CPU (gloo, world_size 2): the host-side control logic of masked_allreduce
  -- header frames, the unanimous vote (collective.cpp:280-293), the density
  rule and the byte accounting -- exercised across two real processes, with
  the frames exchanged by torch.distributed (gloo) instead of NCCL.
* GPU (>= 2 devices): the full NCCL path, one process per GPU under torchrun
  (tests/mp_masked_worker.py), checked against the CPU oracle.
"""
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _torchrun(nproc, script, env=None, timeout=600):
    """torchrun on 127.0.0.1 with a fresh port; retried (new port) when the
    rendezvous store cannot bind it (EADDRINUSE: a port probed free can be
    taken, or in TIME_WAIT, by the time torchrun listens)."""
    for _ in range(4):
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", script]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT, env=env)
        if r.returncode == 0 or "EADDRINUSE" not in r.stderr:
            return r
    return r


def _gloo_vote_worker(rank, world, port, q):
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    import oracle
    import paper_2505_18563_b200 as pb

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    P = oracle.port()
    results = []
    # scenarios: (stable per rank, digest per rank, nnz per rank, density threshold)
    scen = [
        ([1, 1], [7, 7], [100, 100], 0.0),
        ([1, 0], [7, 7], [100, 100], 0.0),
        ([1, 1], [7, 8], [100, 100], 0.0),
        ([1, 1], [7, 7], [100, 99], 0.0),
        ([1, 1], [7, 7], [600, 600], 0.5),
    ]
    n_len = 1000
    for stable, dig, nnz, dens in scen:
        mine = pb.FrameHeader(pb.PayloadKind.Packed if stable[rank] else pb.PayloadKind.Full, 3, dig[rank], nnz[rank])
        frame = pb.encode_header(mine)
        frames = [None] * world
        dist.all_gather_object(frames, frame)
        agree = pb.vote_decide(frames, mine, bool(stable[rank]))
        if agree and 0 < dens < 1 and nnz[rank] / n_len > dens:
            agree = False
        # oracle decision on the same frames, rank-local
        oagree = bool(stable[rank]) and all(
            f[5] == 1 and int.from_bytes(f[10:18], "little") == dig[rank]
            and int.from_bytes(f[18:26], "little") == nnz[rank] for f in frames)
        if oagree and 0 < dens < 1 and nnz[rank] / n_len > dens:
            oagree = False
        count = nnz[rank] if agree else n_len
        results.append((agree, oagree, pb.masked_bytes(world, rank, count), P.ring_bytes(world, rank, count) + 26 * (world - 1)))
    dec = [None] * world
    dist.all_gather_object(dec, [r[0] for r in results])
    q.put((rank, results, dec))
    dist.destroy_process_group()


def test_gloo_two_process_vote(pb):
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_vote_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    expect = [True, False, False, False, False]
    for rank, results, dec in got:
        assert [r[0] for r in results] == expect
        assert all(r[0] == r[1] for r in results)      # same rule as the oracle
        assert all(r[2] == r[3] for r in results)      # same bytes_on_wire
        assert dec[0] == dec[1]                         # unanimous on every rank


@pytest.mark.gpu
def test_nccl_masked_allreduce_multi_gpu(pb):
    import torch

    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs (run with gpurun --gpus 2)")
    world = min(n, 4)
    # default exchange, then the opt-in unpack-fused P2P consumer (PACT_P2P_FUSED)
    for extra in ({}, {"PACT_P2P_FUSED": "1"}):
        env = dict(os.environ, **extra)
        r = _torchrun(world, os.path.join(ROOT, "tests", "mp_masked_worker.py"), env=env)
        print(r.stdout[-4000:], r.stderr[-4000:])
        assert r.returncode == 0, str(extra) + r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.gpu
@pytest.mark.parametrize("transport", ["nccl", "p2p"])
def test_fail_fast_link_error_multi_gpu(pb, transport):
    """A rank killed mid-step: the survivor gets LinkError within the link
    timeout and the comm stays poisoned (reference SimCluster::poison,
    collective.cpp:430-458; trainer.cpp:416-437)."""
    import tempfile

    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs (run with gpurun --gpus 2)")
    env = dict(os.environ, PACT_LINK_TIMEOUT_MS="4000")
    with tempfile.TemporaryDirectory() as d:
        idf = os.path.join(d, "id")
        procs = [subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "mp_failfast_worker.py"), str(r), "2",
                                   idf, transport], stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True,
                                  env=env, cwd=ROOT) for r in range(2)]
        try:
            out0, _ = procs[0].communicate(timeout=240)
            procs[1].wait(timeout=60)
        finally:
            for p in procs:
                if p.poll() is None:
                    p.kill()
        print(out0)
        assert procs[0].returncode == 0, out0
        assert "fail-fast ok" in out0
        assert procs[1].returncode == -9  # the killed rank
