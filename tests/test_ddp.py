"""DDP comm-hook adapter (paper_2505_18563_b200/ddp.py).

* CPU (gloo, world_size 2): the host-side bucket planning -- every DDP
  GradBucket's gradient views tile its buffer, and the (flat offset, length)
  segments the hook gathers the bucket mask from address exactly the bucket's
  parameters in the flattened model (tensor.cpp:49-79 flatten order). The
  planning hook finishes the bucket with a plain gloo all-reduce.
* GPU (>= 2 devices): tests/ddp_worker.py under torchrun -- real DDP
  training steps through pact_hook over NCCL / NVLink, checked bit-exactly
  against GSE(local grads) summed and scaled by 1/n, with the tracker's
  Unstable -> Stable switch from the dense to the packed path.
"""
import os
import subprocess
import sys

import pytest

from conftest import ROOT
from test_multi_gpu import _free_port, _torchrun


def _planning_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    from paper_2505_18563_b200 import ddp

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.manual_seed(0)
    model = torch.nn.Sequential(torch.nn.Linear(37, 300), torch.nn.ReLU(), torch.nn.Linear(300, 129),
                                torch.nn.ReLU(), torch.nn.Linear(129, 11))
    model.get_parameter("2.bias").requires_grad_(False)  # excluded from the flattened model
    m = torch.nn.parallel.DistributedDataParallel(model, bucket_cap_mb=0.05)
    params = [p for p in model.parameters() if p.requires_grad]
    layout, total = ddp.flat_layout(params)
    flat = torch.cat([p.detach().reshape(-1) for p in params])
    seen = []
    errors = []
    cur = [0]

    def hook(state, bucket):
        try:
            segs = ddp.bucket_segments(layout, bucket)
            got = torch.cat([flat[b:b + n] for b, n in segs])
            want = torch.cat([p.detach().reshape(-1) for p in bucket.parameters()])
            if not torch.equal(got, want):
                errors.append(f"bucket {bucket.index()}: segments address other parameters")
            if sum(n for _, n in segs) != bucket.buffer().numel():
                errors.append(f"bucket {bucket.index()}: segments do not cover the buffer")
            seen.append((cur[0], bucket.index(), segs))
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))
        buf = bucket.buffer()
        return dist.all_reduce(buf.div_(world), async_op=True).get_future().then(lambda f: f.value()[0])

    m.register_comm_hook(None, hook)
    for step in range(3):
        cur[0] = step
        torch.manual_seed(100 + rank + 10 * step)
        x = torch.randn(8, 37)
        m(x).square().sum().backward()
    last = [x for x in seen if x[0] == 2]
    covered = sorted((b, n) for _, _, segs in last for b, n in segs)
    q.put((rank, errors, len(last), covered, total))
    dist.destroy_process_group()


def test_ddp_bucket_planning_gloo():
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_planning_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, errors, nb, covered, total in got:
        assert not errors, errors
        assert nb >= 2  # DDP rebuilds buckets after step 0: several per step
        # the buckets' segments tile the flattened model exactly
        pos = 0
        for b, n in covered:
            assert b == pos
            pos += n
        assert pos == total


def test_flat_layout_and_segment_errors():
    import torch

    from paper_2505_18563_b200 import ddp

    ps = [torch.zeros(3, 4), torch.zeros(5), torch.zeros(2, 2)]
    layout, total = ddp.flat_layout(ps)
    assert total == 21
    assert [layout[id(p)] for p in ps] == [(0, 12), (12, 5), (17, 4)]

    class FakeBucket:
        def __init__(self, params, gap=0):
            n = sum(p.numel() for p in params) + gap
            self._buf = torch.zeros(n)
            self._params = params
            self._gap = gap

        def buffer(self):
            return self._buf

        def parameters(self):
            return self._params

        def gradients(self):
            out, at = [], 0
            for i, p in enumerate(self._params):
                if i == 1:
                    at += self._gap
                out.append(self._buf[at:at + p.numel()].view_as(p))
                at += p.numel()
            return out

    # reversed parameter order (DDP buckets run last layer first)
    assert ddp.bucket_segments(layout, FakeBucket([ps[2], ps[1]])) == [(17, 4), (12, 5)]
    assert ddp.bucket_segments(layout, FakeBucket([ps[0], ps[1]])) == [(0, 17)]  # merged run
    from paper_2505_18563_b200 import Error

    with pytest.raises(Error):
        ddp.bucket_segments(layout, FakeBucket([ps[0], ps[1]], gap=3))
    with pytest.raises(Error):
        ddp.bucket_segments(layout, FakeBucket([torch.zeros(3)]))


@pytest.mark.gpu
def test_ddp_hook_multi_gpu(pb):
    import torch

    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs (run with gpurun --gpus 2)")
    r = _torchrun(2, os.path.join(ROOT, "tests", "ddp_worker.py"))
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
