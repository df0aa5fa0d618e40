"""Multi-rank worker for tests/test_multi_gpu.py (launched by torchrun, one
process per GPU). Every rank generates all ranks' inputs from the shared
seeds, runs the library's masked_allreduce over NCCL, and checks its own
result against the CPU oracle (oracle/pact_oracle.c restatement of
collective.cpp:269-309). Exit code != 0 on any mismatch."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2505_18563_b200 as pb  # noqa: E402
from oracle import words_from_bits  # noqa: E402
from paper_2505_18563_b200 import synth  # noqa: E402


def u32(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    comm = pb.Comm.from_process_group()
    port = oracle.port()
    failures = []
    passed = []

    def check(name, ok):
        if not ok:
            failures.append(name)
            print(f"[rank {rank}] FAIL {name}", flush=True)
        else:
            passed.append(name)

    rng = np.random.default_rng(1234)
    n = 300_007
    bits = rng.random(n) < 0.2
    words = words_from_bits(bits)
    mask = pb.SparsityMask.from_words(torch.from_numpy(words.view(np.int64)).to(dev), n)
    check("nnz", mask.nnz() == int(bits.sum()))

    for (recipe, tag), transport in [(r_, t_) for r_ in ((synth.G_DYADIC, "dyadic"), (synth.G_FULL, "full"))
                                     for t_ in (pb.SyncPolicy.NCCL, pb.SyncPolicy.P2P)]:
        tag = f"{tag}/{'p2p' if transport == pb.SyncPolicy.P2P else 'nccl'}"
        grads = [port.gse(synth.synth_host(n, synth.grad_seed(r, 1), recipe), words) for r in range(world)]
        outs, modes, byts = port.masked_allreduce(grads, [words] * world, [1] * world, 3)
        g = torch.from_numpy(grads[rank]).to(dev)
        res = pb.masked_allreduce(g, mask, pb.TrackerStatus.Stable, 3, comm,
                                  policy=pb.SyncPolicy(transport=transport))
        got = res.tensor.cpu().numpy()
        check(f"{tag}: packed mode", res.stats.mode_used == pb.SyncMode.PackedAllReduce and modes[rank] == 1)
        check(f"{tag}: transport", res.stats.transport == transport)
        check(f"{tag}: bytes_on_wire", res.stats.bytes_on_wire == byts[rank])
        if recipe == synth.G_DYADIC or world == 2 or transport == pb.SyncPolicy.P2P:
            # exact partial sums (dyadic), order-free n=2, or the P2P path that
            # folds in the reference ring order: bit-exact
            check(f"{tag}: bit-exact", np.array_equal(u32(got), u32(outs[rank])))
        else:
            tol = 1e-6 * np.maximum(sum(np.abs(x) for x in grads), 2.0 ** -126)
            check(f"{tag}: within 1e-6*sum|x|", bool(np.all(np.abs(got - outs[rank]) <= tol)))
        # repeated P2P steps exercise the double-buffered regions and flags
        for step in range(3):
            r2 = pb.masked_allreduce(g, mask, pb.TrackerStatus.Stable, 3 + step, comm,
                                     policy=pb.SyncPolicy(transport=transport))
            check(f"{tag}: repeat {step}", torch.equal(r2.tensor, res.tensor))
        # every rank holds identical bits (collective.hpp:121-122)
        t = torch.from_numpy(got.view(np.int32).copy()).to(dev)
        lst = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(lst, t)
        check(f"{tag}: replicas identical", all(torch.equal(lst[0], x) for x in lst))

        # bucketed pipeline (pack / exchange / unpack on three streams)
        pol = pb.SyncPolicy(bucket_bytes=64 << 10, transport=transport)
        if transport == pb.SyncPolicy.P2P:
            for step in range(3):  # the P2P fold order is global: buckets stay bit-exact
                rp = pb.masked_allreduce(g, mask, pb.TrackerStatus.Stable, 9 + step, comm, policy=pol)
                check(f"{tag}: p2p buckets>1", rp.stats.buckets > 1 and rp.stats.transport == transport)
                check(f"{tag}: p2p bucketed bit-exact", np.array_equal(u32(rp.tensor.cpu().numpy()), u32(outs[rank])))
            pol = pb.SyncPolicy(bucket_bytes=64 << 10, transport=pb.SyncPolicy.NCCL)
        res_b = pb.masked_allreduce(g, mask, pb.TrackerStatus.Stable, 3, comm, policy=pol)
        check(f"{tag}: buckets>1", res_b.stats.buckets > 1)
        if recipe == synth.G_DYADIC or world == 2:  # NCCL's order depends on the message size
            check(f"{tag}: bucketed == single", torch.equal(res_b.tensor, res.tensor))
        else:
            tol = 1e-6 * np.maximum(sum(np.abs(x) for x in grads), 2.0 ** -126)
            check(f"{tag}: bucketed within 1e-6*sum|x|",
                  bool(np.all(np.abs(res_b.tensor.cpu().numpy() - outs[rank]) <= tol)))
        # fused mean (to_mean, trainer.cpp:268-273)
        res_m = pb.masked_allreduce(g, mask, pb.TrackerStatus.Stable, 3, comm,
                                    policy=pb.SyncPolicy(scale=1.0 / world, transport=transport))
        check(f"{tag}: fused mean", np.array_equal(u32(res_m.tensor.cpu().numpy()),
                                                  u32(port.to_mean(got, world))))

    grads = [synth.synth_host(n, synth.grad_seed(r, 2), synth.G_DYADIC) for r in range(world)]
    g = torch.from_numpy(grads[rank]).to(dev)
    # one unstable tracker -> every rank falls back to the dense sum
    stable = [1] * world
    stable[world - 1] = 0
    outs, modes, byts = port.masked_allreduce(grads, [words] * world, stable, 4)
    res = pb.masked_allreduce(g, mask, pb.TrackerStatus.Stable if stable[rank] else pb.TrackerStatus.Unstable, 4, comm)
    check("unstable: full mode", res.stats.mode_used == pb.SyncMode.FullAllReduce and modes[rank] == 0)
    check("unstable: bytes", res.stats.bytes_on_wire == byts[rank])
    check("unstable: exact", np.array_equal(u32(res.tensor.cpu().numpy()), u32(outs[rank])))

    # advertised-digest fault on rank 0 (trainer.cpp:286-290) -> fallback
    d0 = mask.digest()
    adv = [d0] * world
    adv[0] = d0 ^ 0x5A5A5A5A5A5A5A5A
    outs, modes, byts = port.masked_allreduce(grads, [words] * world, [1] * world, 5, adv)
    res = pb.masked_allreduce(g, mask, pb.TrackerStatus.Stable, 5, comm, advertised_digest=adv[rank])
    check("fault: full mode", res.stats.mode_used == pb.SyncMode.FullAllReduce and modes[rank] == 0)
    check("fault: exact", np.array_equal(u32(res.tensor.cpu().numpy()), u32(outs[rank])))

    # divergent masks on the last rank -> fallback (test_collective.cpp:263-285)
    bad = bits.copy()
    bad[6] = not bad[6]
    wbad = words_from_bits(bad)
    mine = wbad if rank == world - 1 else words
    m2 = pb.SparsityMask.from_words(torch.from_numpy(mine.view(np.int64)).to(dev), n)
    outs, modes, byts = port.masked_allreduce(grads, [words] * (world - 1) + [wbad], [1] * world, 7)
    res = pb.masked_allreduce(g, m2, pb.TrackerStatus.Stable, 7, comm)
    check("divergent: full mode", res.stats.mode_used == pb.SyncMode.FullAllReduce)
    check("divergent: exact", np.array_equal(u32(res.tensor.cpu().numpy()), u32(outs[rank])))

    # density rule: unanimous dense fallback above the threshold
    res = pb.masked_allreduce(g, mask, pb.TrackerStatus.Stable, 8, comm,
                              policy=pb.SyncPolicy(density_threshold=0.1))
    check("density: full mode", res.stats.mode_used == pb.SyncMode.FullAllReduce and res.stats.fallback_reason == 3)

    # full_allreduce == ring semantics; allgather of frames
    res = pb.full_allreduce(g, comm)  # dyadic inputs: exact in any reduction order
    check("full_allreduce exact",
          np.array_equal(u32(res.tensor.cpu().numpy()), u32(port.ring_allreduce(grads)[rank])))
    check("full bytes", res.stats.bytes_on_wire == port.ring_bytes(world, rank, n))
    frames = pb.allgather(bytes([rank]) * 26, comm)
    check("allgather", frames == [bytes([r]) * 26 for r in range(world)])

    # host-buffer entry point
    gh = torch.from_numpy(grads[rank]).pin_memory()
    oh = torch.empty(n, dtype=torch.float32).pin_memory()
    st = pb.masked_allreduce_host(gh, mask, pb.TrackerStatus.Stable, 9, comm, oh)
    outs, modes, byts = port.masked_allreduce([port.gse(x, words) for x in grads], [words] * world, [1] * world, 9)
    gse_outs = outs
    check("host: packed", st.mode_used == pb.SyncMode.PackedAllReduce)
    check("host: exact", np.array_equal(u32(oh.numpy()), u32(gse_outs[rank])))

    # ---- ternary-on-packed (collective.cpp:311-368), SURVEY 8f-2
    nnz = int(bits.sum())
    seeds = [port.derive_seed(0x7E, r, 11) for r in range(world)]
    grads = [synth.synth_host(n, synth.grad_seed(r, 12), synth.G_FULL) for r in range(world)]
    g = torch.from_numpy(grads[rank]).to(dev)
    rt = pb.ternary_allgather_aggregate(g, mask, pb.TrackerStatus.Stable, seeds[rank], 11, comm)
    tern = [port.ternarize(port.pack(x, words), sd) for x, sd in zip(grads, seeds)]
    want = port.unpack(port.ternary_mean([t[0] for t in tern], [t[1] for t in tern], nnz),
                       port.mask_digest(words, n), words, n)
    check("ternary: mode", rt.stats.mode_used == pb.SyncMode.TernaryAllGather)
    check("ternary: bit-exact vs oracle", np.array_equal(u32(rt.tensor.cpu().numpy()), u32(want)))
    check("ternary: bytes", rt.stats.bytes_on_wire == (world - 1) * (30 + (nnz + 3) // 4))
    if oracle.ref_available():  # draw-independent inputs: the reference itself
        R = oracle.ref()
        sat = [port.gse(np.where(np.arange(n) % 3 == r % 3, 0.0, (r + 1.0) * np.sign(x)).astype(np.float32),
                        words) for r, x in enumerate(grads)]
        outs, modes, byts = R.ternary_aggregate(sat, [words] * world, [1] * world, seeds, 11)
        rs = pb.ternary_allgather_aggregate(torch.from_numpy(sat[rank]).to(dev), mask, pb.TrackerStatus.Stable,
                                            seeds[rank], 11, comm)
        check("ternary: saturated == reference",
              np.array_equal(u32(rs.tensor.cpu().numpy()), u32(outs[rank])) and modes[rank] == 2)
        check("ternary: bytes == reference", rs.stats.bytes_on_wire == byts[rank])
        stable = [1] * world
        stable[0] = 0
        outs, modes, byts = R.ternary_aggregate(grads, [words] * world, stable, seeds, 12)
        rf = pb.ternary_allgather_aggregate(g, mask, pb.TrackerStatus.Stable if stable[rank] else
                                            pb.TrackerStatus.Unstable, seeds[rank], 12, comm)
        check("ternary fallback: mode", rf.stats.mode_used == pb.SyncMode.FullAllReduce and modes[rank] == 0)
        check("ternary fallback: bytes == reference", rf.stats.bytes_on_wire == byts[rank])
        if world == 2:  # NCCL's sum is order-free only for two ranks
            check("ternary fallback: == reference", np.array_equal(u32(rf.tensor.cpu().numpy()), u32(outs[rank])))

    # ---- binary16 wire (collective.cpp:133-216, 261-267), SURVEY 8f-3
    grads = [(synth.synth_host(n, synth.grad_seed(r, 13), synth.G_FULL) * (1000.0 if r % 2 else 0.001)
              ).astype(np.float32) for r in range(world)]
    g = torch.from_numpy(grads[rank]).to(dev)
    rh = pb.fp16_allreduce(g, comm)
    want = port.ring_allreduce_fp16(grads)[rank]
    check("fp16: bit-exact vs ring", np.array_equal(u32(rh.tensor.cpu().numpy()), u32(want)))
    check("fp16: bytes", rh.stats.bytes_on_wire == port.ring_bytes(world, rank, n) // 2)
    check("fp16: mode", rh.stats.mode_used == pb.SyncMode.Fp16AllReduce)
    rp = pb.masked_allreduce(g, mask, pb.TrackerStatus.Stable, 14, comm, policy=pb.SyncPolicy(wire=pb.SyncPolicy.F16))
    pk = port.ring_allreduce_fp16([port.pack(x, words) for x in grads])[rank]
    want = port.unpack(pk, port.mask_digest(words, n), words, n)
    check("fp16 packed: bit-exact", np.array_equal(u32(rp.tensor.cpu().numpy()), u32(want)))
    check("fp16 packed: bytes",
          rp.stats.bytes_on_wire == 26 * (world - 1) + port.ring_bytes(world, rank, int(bits.sum())) // 2)

    # ---- TopK all-gather baseline (collective.cpp:370-390), SURVEY 8f-4
    grads = [(np.round(synth.synth_host(n, synth.grad_seed(r, 15), synth.G_FULL) * 8) / 8).astype(np.float32)
             for r in range(world)]  # coarse grid: heavy ties across ranks
    g = torch.from_numpy(grads[rank]).to(dev)
    rk = pb.topk_allgather_aggregate(g, 0.02, 0, comm)
    sel = [port.topk_select(x, 0.02) for x in grads]
    want = port.topk_mean([q[0] for q in sel], [q[1] for q in sel], n)
    check("topk: bit-exact vs oracle", np.array_equal(u32(rk.tensor.cpu().numpy()), u32(want)))
    check("topk: bytes", rk.stats.bytes_on_wire == (world - 1) * (26 + 8 * sel[0][0].size))
    check("topk: mode", rk.stats.mode_used == pb.SyncMode.TopKAllGather)

    # ---- n = 2 push exchange, compact pair unpack with a few dense chunks
    # (runs > 512 values read the peer's run from global memory)
    if world == 2:
        nb = 200_003
        bits2 = rng.random(nb) < 0.1
        bits2[:10 * 1024 + 77] = True
        words2 = words_from_bits(bits2)
        mask2 = pb.SparsityMask.from_words(torch.from_numpy(words2.view(np.int64)).to(dev), nb)
        grads2 = [port.gse(synth.synth_host(nb, synth.grad_seed(r, 21), synth.G_FULL), words2) for r in range(world)]
        outs2, _, _ = port.masked_allreduce(grads2, [words2] * world, [1] * world, 5)
        g2 = torch.from_numpy(grads2[rank]).to(dev)
        for step in range(3):
            r2 = pb.masked_allreduce(g2, mask2, pb.TrackerStatus.Stable, 5 + step, comm,
                                     policy=pb.SyncPolicy(transport=pb.SyncPolicy.P2P))
            check(f"compact pair with dense chunks: bit-exact (step {step})",
                  np.array_equal(u32(r2.tensor.cpu().numpy()), u32(outs2[rank])))

    # ---- measured dense/sparse crossover: unanimous threshold,
    # and the policy it feeds picks packed below / dense above it
    cal = pb.calibrate_density(1 << 22, comm, densities=[0.05, 0.3, 0.6, 0.9])
    th = torch.tensor([cal.threshold], dtype=torch.float64, device=dev)
    ths = [torch.empty_like(th) for _ in range(world)]
    dist.all_gather(ths, th)
    check("calibrate: same threshold on every rank", all(float(x) == cal.threshold for x in ths))
    check("calibrate: timings", len(cal.t_packed) == 4 and all(t > 0 for t in cal.t_packed) and cal.t_dense > 0)
    check("calibrate: threshold in (0, 1]", 0.0 < cal.threshold <= 1.0)
    pol = pb.SyncPolicy(density_threshold=min(cal.threshold, 0.999))
    g = torch.from_numpy(grads[rank][:n].copy()).to(dev)
    r = pb.masked_allreduce(g, mask, pb.TrackerStatus.Stable, 1, comm, policy=pol)
    dens = mask.nnz() / n
    want_mode = pb.SyncMode.PackedAllReduce if dens <= pol.density_threshold else pb.SyncMode.FullAllReduce
    check("calibrate: policy decision follows the threshold", r.stats.mode_used == want_mode)

    # ---- ring_allreduce in the reference's fold order (collective.cpp:165-216)
    grads = [synth.synth_host(n, synth.grad_seed(r, 31), synth.G_FULL) for r in range(world)]
    g = torch.from_numpy(grads[rank]).to(dev)
    ro = pb.ring_allreduce(g, comm, exact=True)
    check("ring_allreduce exact: == reference ring order",
          np.array_equal(u32(ro.cpu().numpy()), u32(port.ring_allreduce(grads)[rank])))
    try:
        pb.ring_allreduce(g[: n - (rank == 0)], comm, exact=True)
        check("ring_allreduce: length mismatch raises", False)
    except pb.Error as e:
        check("ring_allreduce: length mismatch raises", e.code == pb.Errc.ShapeMismatch)

    # ---- BASELINE size: C2 (ResNet-50 shape, 25,557,032, 80%) on the
    # device-pruned global mask, full-mantissa gradients, both transports
    shape = synth.model_shape("resnet50")
    nb = shape.total
    wd = synth.weights_device(shape, 1234, synth.W_REAL, device=dev)
    mb = pb.magnitude_prune(wd, 0.8)
    wb = mb.words_host()
    check("C2: nnz", mb.nnz() == 5_111_404)
    check("C2: mask == oracle prune", np.array_equal(wb, port.magnitude_prune(wd.cpu().numpy(), 0.8)))
    gradsb = [port.gse(synth.synth_host(nb, synth.grad_seed(r, 41), synth.G_FULL), wb) for r in range(world)]
    outsb, modesb, bytsb = port.masked_allreduce(gradsb, [wb] * world, [1] * world, 2)
    gb = torch.from_numpy(gradsb[rank]).to(dev)
    sumabs = sum(np.abs(x) for x in gradsb)
    for transport, tname in ((pb.SyncPolicy.NCCL, "nccl"), (pb.SyncPolicy.P2P, "p2p"), (pb.SyncPolicy.AUTO, "auto")):
        rb = pb.masked_allreduce(gb, mb, pb.TrackerStatus.Stable, 2, comm, policy=pb.SyncPolicy(transport=transport))
        got = rb.tensor.cpu().numpy()
        check(f"C2/{tname}: packed", rb.stats.mode_used == pb.SyncMode.PackedAllReduce and modesb[rank] == 1)
        check(f"C2/{tname}: bytes_on_wire", rb.stats.bytes_on_wire == bytsb[rank])
        if world == 2 or rb.stats.transport == pb.SyncPolicy.P2P:
            check(f"C2/{tname}: bit-exact", np.array_equal(u32(got), u32(outsb[rank])))
        else:
            tol = 1e-6 * np.maximum(sumabs, 2.0 ** -126)
            check(f"C2/{tname}: within 1e-6*sum|x|", bool(np.all(np.abs(got - outsb[rank]) <= tol)))
    del wd, gb

    flag = torch.tensor([len(failures)], device=dev)
    dist.all_reduce(flag)
    if rank == 0:
        print(f"mp_masked_worker world={world} checks passed on rank 0: {len(passed)}", flush=True)
        for nm in passed:
            print(f"  ok {nm}", flush=True)
    comm.close()
    dist.destroy_process_group()
    if rank == 0:
        print(f"mp_masked_worker world={world} failures={int(flag.item())}", flush=True)
    sys.exit(1 if int(flag.item()) else 0)


if __name__ == "__main__":
    main()
