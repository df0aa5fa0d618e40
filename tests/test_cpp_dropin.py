"""The C++ drop-in header (include/pact_b200.hpp) compiles against the C-ABI
(CPU) and passes the reference's own unit assertions on the GPU."""
import os
import subprocess

import pytest

from conftest import ROOT

SRC = os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp")
OUT = os.path.join(ROOT, "tests", "cpp", "_build", "dropin_test")
CLUSTER_SRC = os.path.join(ROOT, "tests", "cpp", "cluster_test.cpp")
CLUSTER_OUT = os.path.join(ROOT, "tests", "cpp", "_build", "cluster_test")


def _build(pb, src=SRC, out=OUT):
    from paper_2505_18563_b200 import _lib

    os.makedirs(os.path.dirname(out), exist_ok=True)
    libdir = os.path.dirname(_lib.PATH)
    if os.path.exists(out) and os.path.getmtime(out) > max(
            os.path.getmtime(src), os.path.getmtime(_lib.PATH),
            os.path.getmtime(os.path.join(ROOT, "include", "pact_b200.hpp"))):
        return out
    cmd = ["nvcc", "-std=c++17", "-O2", "-x", "cu", "-gencode", "arch=compute_100a,code=sm_100a",
           "-Xcompiler", "-pthread", "-I" + os.path.join(ROOT, "include"), src, "-L" + libdir, "-lpact_b200",
           "-Xlinker", "-rpath," + libdir, "-o", out]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return out


def test_header_compiles(pb):
    assert os.path.exists(_build(pb))
    assert os.path.exists(_build(pb, CLUSTER_SRC, CLUSTER_OUT))


@pytest.mark.gpu
def test_reference_collective_assertions_multi_gpu(pb, cuda):
    """The reference's collective unit tests (test_collective.cpp:46-285) over
    the C++ drop-in header on real GPUs, one worker PROCESS per GPU (the
    reference's workers are threads of one SimCluster process)."""
    import tempfile

    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs (run with gpurun --gpus 2)")
    exe = _build(pb, CLUSTER_SRC, CLUSTER_OUT)
    world = min(torch.cuda.device_count(), 4)
    with tempfile.TemporaryDirectory() as d:
        idf = os.path.join(d, "ncclid")
        procs = [subprocess.Popen([exe, str(r), str(world), idf], stdout=subprocess.PIPE,
                                  stderr=subprocess.STDOUT, text=True) for r in range(world)]
        outs = []
        try:
            for p in procs:
                outs.append((p.wait(timeout=300), p.stdout.read()))
        finally:
            for p in procs:
                if p.poll() is None:
                    p.kill()
    for rc, out in outs:
        print(out[-2000:])
    assert all(rc == 0 for rc, _ in outs), [o[-1500:] for _, o in outs]


@pytest.mark.gpu
def test_reference_collective_assertions_threaded_multi_gpu(pb, cuda):
    """The same assertions with every worker a THREAD of one process driving
    its own GPU -- the reference's own SimCluster topology (SURVEY 8(b)
    "Threading"): NCCL communicators per thread, NVLink peer access instead
    of CUDA IPC between the threads."""
    import tempfile

    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs (run with gpurun --gpus 2)")
    exe = _build(pb, CLUSTER_SRC, CLUSTER_OUT)
    world = min(torch.cuda.device_count(), 4)
    with tempfile.TemporaryDirectory() as d:
        r = subprocess.run([exe, "threads", str(world), os.path.join(d, "ncclid")], capture_output=True,
                           text=True, timeout=600)
    print(r.stdout[-3000:], r.stderr[-2000:])
    assert r.returncode == 0, r.stdout[-3000:]


@pytest.mark.gpu
def test_reference_unit_assertions_on_gpu(pb, cuda):
    exe = _build(pb)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout[-3000:], r.stderr[-2000:])
    assert r.returncode == 0, r.stdout[-3000:]
