"""PCIe roofline for the host-buffer (e2e) entry point: pinned H2D alone,
D2H alone, and both directions at once (separate streams), 102 MB each
(the c2 gradient). Prints one JSON line."""
import json
import sys

import torch


def main(nbytes=102_228_128, reps=20):
    n = nbytes // 4
    h_in = torch.empty(n, dtype=torch.float32).pin_memory()
    h_out = torch.empty(n, dtype=torch.float32).pin_memory()
    d_in = torch.empty(n, dtype=torch.float32, device="cuda")
    d_out = torch.empty(n, dtype=torch.float32, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps * 1e-3

    def h2d():
        d_in.copy_(h_in, non_blocking=True)

    def d2h():
        h_out.copy_(d_out, non_blocking=True)

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    t_h2d, t_d2h, t_both = timed(h2d), timed(d2h), timed(both)
    print(json.dumps({"bytes": nbytes, "h2d_gbs": round(nbytes / t_h2d / 1e9, 2),
                      "d2h_gbs": round(nbytes / t_d2h / 1e9, 2),
                      "bidir_gbs_per_direction": round(nbytes / t_both / 1e9, 2),
                      "bidir_ms": round(t_both * 1e3, 3)}))


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:]))
