"""Times the prune paths at a BASELINE size (default C5): first-time
(sampled), temporal-reuse hit, a moved threshold resolved from the window
candidates with the mask unchanged (A.9: w <- GSE(w) + fresh dense noise),
and a real mask change (+digest). CUDA events, L2 flushed before each call.

    python tools/prune_probe.py [model] [ratio]
"""
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2505_18563_b200 as pb  # noqa: E402
from paper_2505_18563_b200 import synth  # noqa: E402


def main():
    model = sys.argv[1] if len(sys.argv) > 1 else "gpt2-medium"
    ratio = float(sys.argv[2]) if len(sys.argv) > 2 else 0.9
    torch.cuda.set_device(0)
    shape = synth.model_shape(model)
    n = shape.total
    w = synth.weights_device(shape, 1234, synth.W_REAL)
    flush = torch.empty(128 << 20, dtype=torch.float32, device="cuda")
    flush_r = torch.zeros(128 << 20, dtype=torch.float32, device="cuda")
    sink = torch.empty((), dtype=torch.float32, device="cuda")
    noise = torch.empty(n, dtype=torch.float32, device="cuda")

    def timed(fn):
        # bench.py's L2 flush: write 512 MiB, then read another 512 MiB so the
        # dirty lines are written back before the timed call
        flush.zero_()
        torch.sum(flush_r, dim=0, out=sink)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        return a.elapsed_time(b) * 1e3

    res = {}
    m = pb.SparsityMask(n)
    st = {}
    res["first_us"] = timed(lambda: pb.magnitude_prune(w, ratio, out=m, stats=st))
    res["first_path"] = st["path"]
    w2 = synth.weights_device(shape, 4321, synth.W_REAL)
    res["full_us"] = timed(lambda: pb.magnitude_prune(w2, ratio, out=m, stats=st))
    res["full_path"] = st["path"]
    del w2
    pb.magnitude_prune(w, ratio, out=m)
    hit = []
    for _ in range(5):
        hit.append(timed(lambda: pb.magnitude_prune(w, ratio, out=m, stats=st)))
    res["hit_us"] = statistics.median(hit)
    res["hit_path"] = st["path"]
    # A.9: kept entries keep their values, pruned ones get fresh tiny noise
    move, paths, changed = [], [], []
    for t in range(8):
        words = m.words()
        sh = torch.arange(64, device="cuda", dtype=torch.int64)
        keep = ((words.view(-1, 1) >> sh) & 1).view(-1)[:n].bool()
        # dense drift (no GSE): the threshold sits inside the distribution and
        # moves every step; a few hundred elements cross it
        pb.synth_fill(noise, 900 + t, synth.W_REAL, 2.0 ** -17)
        w = w + noise
        del keep
        d0 = m.digest()
        move.append(timed(lambda: pb.magnitude_prune(w, ratio, out=m, stats=st)))
        paths.append(st["path"])
        changed.append((m.changed, m.digest() != d0))
    res["move_us"] = statistics.median(move[2:])
    res["move_paths"] = paths
    res["move_changed"] = changed
    # a real mask change: 4000 dropped elements become large
    chg, paths = [], []
    for t in range(5):
        words = m.words()
        sh = torch.arange(64, device="cuda", dtype=torch.int64)
        keep = ((words.view(-1, 1) >> sh) & 1).view(-1)[:n].bool()
        idx = torch.nonzero(~keep)[t * 4000:(t + 1) * 4000, 0]
        w[idx] = 1.0
        del keep

        def f():
            pb.magnitude_prune(w, ratio, out=m, stats=st)
            m.digest()
        chg.append(timed(f))
        paths.append(st["path"])
    res["change_plus_digest_us"] = statistics.median(chg)
    res["change_paths"] = paths
    print(model, n, {k: (round(v, 1) if isinstance(v, float) else v) for k, v in res.items()})


if __name__ == "__main__":
    main()
