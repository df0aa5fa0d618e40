"""Times the exact FNV-1a mask digest (csrc/digest.cu) at the BASELINE mask
sizes and checks it against the oracle port on the same words.

    python tools/digest_probe.py        (GPU box)
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (checker only)
import paper_2505_18563_b200 as pb  # noqa: E402

SIZES = {"c1": 11_689_512, "c2": 25_557_032, "c3": 143_667_240, "c4": 109_482_240, "c5": 354_823_168}


def main():
    port = oracle.port()
    torch.cuda.set_device(0)
    for name, n in SIZES.items():
        nw = (n + 63) // 64
        rng = np.random.default_rng(nw)
        w = rng.integers(0, 2**63, nw, dtype=np.uint64)
        if n % 64:
            w[-1] &= np.uint64((1 << (n % 64)) - 1)
        wd = torch.from_numpy(w.view(np.int64)).cuda()
        m = pb.SparsityMask.from_words(wd, n)
        want = port.mask_digest(w, n)
        ts = []
        for _ in range(6):
            m2 = pb.SparsityMask.from_words(wd, n)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            d = m2.digest()
            ts.append(time.perf_counter() - t0)
            assert d == want, (name, hex(d), hex(want))
        print(f"{name}: n={n} digest ok, host-timed {min(ts[1:]) * 1e6:.1f} us (incl. launch + readback)")


if __name__ == "__main__":
    main()
