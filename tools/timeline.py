"""Device timeline of the prune paths (torch.profiler / CUPTI kernel records):
kernel name, start offset, duration and the idle gap before it, so host
round trips show up as gaps. nsys is not in this image.

    python tools/timeline.py [model] [ratio] [scenario: hit|drift|regrow|step|a9|a9step]
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2505_18563_b200 as pb  # noqa: E402
from paper_2505_18563_b200 import synth  # noqa: E402


def main():
    model = sys.argv[1] if len(sys.argv) > 1 else "gpt2-medium"
    ratio = float(sys.argv[2]) if len(sys.argv) > 2 else 0.9
    scen = sys.argv[3] if len(sys.argv) > 3 else "drift"
    torch.cuda.set_device(0)
    shape = synth.model_shape(model)
    n = shape.total
    w = synth.weights_device(shape, 1234, synth.W_REAL)
    noise = torch.empty(n, dtype=torch.float32, device="cuda")
    g = torch.empty(n, dtype=torch.float32, device="cuda")
    pb.synth_fill(g, 5, synth.G_FULL)
    out = torch.empty_like(g)
    m = pb.magnitude_prune(w, ratio)
    pb.magnitude_prune(w, ratio, out=m)

    def keep_of(mask):
        b = mask.words().view(torch.uint8)
        sh = torch.arange(8, device="cuda", dtype=torch.uint8)
        return ((b.view(-1, 1) >> sh) & 1).view(-1)[:n].bool()

    def prep(t):
        if scen == "drift" or scen == "step":
            pb.synth_fill(noise, 900 + t, synth.W_REAL, 2.0 ** -17)
            w.add_(noise)
        elif scen in ("a9", "a9step"):  # bench.py's A.9 perturbation
            kb = keep_of(m)
            pb.synth_fill(noise, 700 + t, synth.W_REAL, 2.0 ** -14)
            wd = w + noise
            pb.synth_fill(noise, 800 + t, synth.W_REAL, 2.0 ** -20)
            torch.where(kb, wd, noise, out=w)

    def run(t):
        pb.magnitude_prune(w, ratio, out=m)
        m.digest()
        if scen in ("step", "a9step"):
            pb.masked_allreduce(g, m, pb.TrackerStatus.Stable, t, None, out=out)

    for t in range(3):
        prep(t)
        run(t)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for t in range(3, 5):
            prep(t)
            torch.cuda.synchronize()
            run(t)
            torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    evs.sort(key=lambda e: e.time_range.start)
    t0 = None
    prev_end = None
    for e in evs:
        s, d = e.time_range.start, e.time_range.elapsed_us()
        if t0 is None:
            t0 = s
        gap = 0 if prev_end is None else s - prev_end
        name = e.name.replace("(anonymous namespace)::", "").replace("void ", "").replace("pactk::", "").split("(")[0]
        print(f"{(s - t0):9.1f} {d:8.1f} gap {gap:7.1f}  {name[:70]}")
        prev_end = s + d


if __name__ == "__main__":
    main()
