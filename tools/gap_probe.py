import sys, statistics, torch
sys.path.insert(0, '/root/repo')
import paper_2505_18563_b200 as pb
from paper_2505_18563_b200 import synth
dev = torch.device('cuda', 0)
shape = synth.model_shape('resnet50'); n = shape.total
w = synth.weights_device(shape, 1234, synth.W_REAL, device=dev)
mask = pb.magnitude_prune(w, 0.8); nnz = mask.nnz()
g = torch.empty(n, device=dev); pb.synth_fill(g, synth.grad_seed(0, 0), synth.G_FULL)
out = torch.empty_like(g); packed = torch.empty(nnz, device=dev)
pk = pb.PackedGradient(mask.digest(), 0, packed)
flush = torch.empty(128 << 20, device=dev); fr = torch.zeros(128 << 20, device=dev); sink = torch.empty((), device=dev)
ctx = pb.Context.get(0); s = torch.cuda.current_stream()
def do_pack(): pb.api._call(pb.api.lib.pact_pack, ctx.handle, pb.api._ptr(g), n, mask.handle, pb.api._ptr(packed), 0, pb.api.C.c_uint64(2**64-1), pb.api._stream())
def do_unpack(): pb.unpack(pk, mask, out=out)
pol = pb.SyncPolicy()
def do_step(): pb.masked_allreduce(g, mask, pb.TrackerStatus.Stable, 0, None, policy=pol, out=out)
def both(): do_pack(); do_unpack()
def t(fn, k=30, flush_it=True, sleep=False):
    r = []
    for i in range(k + 3):
        if flush_it:
            flush.zero_(); torch.sum(fr, dim=0, out=sink)
        if sleep: torch.cuda._sleep(200000)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(s); fn(); b.record(s); r.append((a, b))
    torch.cuda.synchronize()
    return statistics.median([a.elapsed_time(b) * 1000 for a, b in r[3:]])
for name, fn in (('pack', do_pack), ('unpack', do_unpack), ('pack+unpack', both), ('step', do_step)):
    print(name, 'flushed', round(t(fn), 2), 'flushed+sleep', round(t(fn, sleep=True), 2), 'noflush', round(t(fn, flush_it=False), 2))
