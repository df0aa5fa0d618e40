"""Exercise every single-GPU kernel once at small, ragged sizes, for
compute-sanitizer (memcheck / racecheck / synccheck):

    compute-sanitizer --tool memcheck python tools/sanitize_probe.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_18563_b200 as pb  # noqa: E402
from paper_2505_18563_b200 import synth  # noqa: E402

dev = torch.device("cuda", 0)
for n in (1, 63, 1000, 4097, 131_073, 1_000_003):
    for ratio in (0.0, 0.5, 0.9, 0.99):
        w = torch.empty(n, device=dev)
        pb.synth_fill(w, 7 + n, synth.W_TIES, 0.125)
        g = torch.empty(n, device=dev)
        pb.synth_fill(g, 9 + n, synth.G_FULL)
        m = pb.magnitude_prune(w, ratio)
        pb.magnitude_prune(w, ratio, out=m)  # the temporal-reuse path
        p = pb.pack(g, m, 1)
        u = pb.unpack(p, m)
        pb.unpack(p, m, scale=0.5)
        pb.enforce_gradient_sparsity(g, m)
        wt = w.clone()
        pb.unpack_sgd(p.values, m, 0.5, 0.1, wt)
        pb.masked_allreduce(g, m, pb.TrackerStatus.Stable, 0, None)
        pb.masked_allreduce(g, m, pb.TrackerStatus.Unstable, 0, None)
        m.digest()
        if n >= 64:
            gh = g.cpu().pin_memory()
            oh = torch.empty(n).pin_memory()
            pb.masked_allreduce_host(gh, m, pb.TrackerStatus.Stable, 0, None, oh)
            pb.topk_select(g, 0.05)
            t = pb.ternarize(p.values, 3) if p.values.numel() else None
            if t is not None:
                pb.deternarize(t)
            pb.fp16_roundtrip(g)
        if n >= 4097:
            segs = [0, n // 3, n // 2, n]
            pb.magnitude_prune_per_layer(w, segs, ratio)
        # unaligned base pointers
        if n > 8:
            g1 = g[1:]
            m1 = pb.magnitude_prune(w[1:], ratio)
            pb.unpack(pb.pack(g1, m1, 0), m1)
torch.cuda.synchronize()
print("sanitize probe ok")
