"""NVLink bytes of the n = 2 push pack kernel (pack_lm_kernel<kPushTma>),
one process, GPU 0 packing into its own buffer and pushing every run into a
buffer on GPU 1 (pact_debug_pack_push: the exchange's kernel without its
peer flags, so ncu can replay it). Prints event timings of the plain pack and
the push pack and checks the remote copy.

    python tools/nvlink_push_ncu.py c5
    ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,... \
        -k regex:pack_lm python tools/nvlink_push_ncu.py c5 1
"""
import ctypes as C
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2505_18563_b200 as pb  # noqa: E402
from paper_2505_18563_b200 import api, synth  # noqa: E402

CFG = {"c2": ("resnet50", 0.8), "c3": ("vgg19", 0.95), "c5": ("gpt2-medium", 0.9)}


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    model, ratio = CFG[cfg]
    torch.cuda.set_device(0)
    shape = synth.model_shape(model)
    n = shape.total
    w = synth.weights_device(shape, 1234, synth.W_REAL)
    m = pb.magnitude_prune(w, ratio)
    del w
    g = torch.empty(n, device="cuda:0")
    pb.synth_fill(g, 5, synth.G_FULL)
    nnz = m.nnz()
    packed = torch.empty(nnz, device="cuda:0")
    remote = torch.zeros(nnz, device="cuda:1")
    ctx = api.Context.get(0)
    st = api._stream()

    def push():
        api._call(api.lib.pact_debug_pack_push, ctx.handle, api._ptr(g), n, m.handle, api._ptr(packed),
                  api._ptr(remote), st)

    def plain():
        api._call(api.lib.pact_pack, ctx.handle, api._ptr(g), n, m.handle, api._ptr(packed), 0,
                  C.c_uint64(2 ** 64 - 1), st)

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            best = min(best, a.elapsed_time(b) * 1e3)
        return best

    t_plain = timed(plain)
    t_push = timed(push)
    ok = torch.equal(remote.to("cuda:0"), packed)
    print(f"{cfg}: nnz={nnz} pushed bytes={4 * nnz} | pack {t_plain:.1f} us | push pack {t_push:.1f} us "
          f"({4 * nnz / t_push / 1e3:.1f} GB/s one-way NVLink payload, no reverse traffic) | remote == packed: {ok}",
          flush=True)


if __name__ == "__main__":
    main()
