"""In-tree build of the native library (libpact_b200.so) for sm_100a.

Run by ``__graft_entry__.build()`` (CPU container: nvcc cross-compiles) and
usable directly: ``python -m paper_2505_18563_b200._build``. The .so lands in
``paper_2505_18563_b200/_native/`` so it travels to the GPU box with the repo.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT_DIR = os.path.join(PKG, "_native")
LIB = os.path.join(OUT_DIR, "libpact_b200.so")
# A/B experiments: PACT_LIB points the loader at an alternative build
LIB = os.environ.get("PACT_LIB", LIB)
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_paths():
    """NCCL headers/lib: the torch-bundled NCCL (the one a torch process has
    already loaded), else the system one."""
    cands = []
    try:
        import nvidia.nccl  # type: ignore

        base = list(nvidia.nccl.__path__)[0]
        cands.append((os.path.join(base, "include"), os.path.join(base, "lib")))
    except Exception:
        pass
    cands.append(("/usr/include", "/usr/lib/x86_64-linux-gnu"))
    for inc, lib in cands:
        if os.path.exists(os.path.join(inc, "nccl.h")) and glob.glob(os.path.join(lib, "libnccl.so*")):
            return inc, lib
    raise RuntimeError("NCCL headers/library not found")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu"))) + sorted(glob.glob(os.path.join(CSRC, "*.cpp")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))
    deps += glob.glob(os.path.join(ROOT, "include", "*.h")) + [os.path.abspath(__file__)]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(OUT_DIR, exist_ok=True)
    inc, lib = nccl_paths()
    nccl_so = "libnccl.so.2" if os.path.exists(os.path.join(lib, "libnccl.so.2")) else "libnccl.so"
    tmp = LIB + ".tmp"
    cmd = [
        "nvcc", "-shared", "-Xcompiler", "-fPIC", *ARCH, "-lineinfo", "-O3", "-std=c++17",
        "-I" + os.path.join(ROOT, "include"), "-I" + inc,
        *sources(),
        "-L" + lib, "-l:" + nccl_so, "-Xlinker", "-rpath," + lib,
        "-o", tmp,
    ]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
