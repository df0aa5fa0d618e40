"""The C++ drop-in header (include/pact_b200.hpp) compiles against the C-ABI
(CPU) and passes the reference's own unit assertions on the GPU."""
import os
import subprocess

import pytest

from conftest import ROOT

SRC = os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp")
OUT = os.path.join(ROOT, "tests", "cpp", "_build", "dropin_test")


def _build(pb):
    from paper_2505_18563_b200 import _lib

    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    libdir = os.path.dirname(_lib.PATH)
    if os.path.exists(OUT) and os.path.getmtime(OUT) > max(
            os.path.getmtime(SRC), os.path.getmtime(_lib.PATH),
            os.path.getmtime(os.path.join(ROOT, "include", "pact_b200.hpp"))):
        return OUT
    cmd = ["nvcc", "-std=c++17", "-O2", "-x", "cu", "-gencode", "arch=compute_100a,code=sm_100a",
           "-I" + os.path.join(ROOT, "include"), SRC, "-L" + libdir, "-lpact_b200",
           "-Xlinker", "-rpath," + libdir, "-o", OUT]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return OUT


def test_header_compiles(pb):
    assert os.path.exists(_build(pb))


@pytest.mark.gpu
def test_reference_unit_assertions_on_gpu(pb, cuda):
    exe = _build(pb)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout[-3000:], r.stderr[-2000:])
    assert r.returncode == 0, r.stdout[-3000:]
