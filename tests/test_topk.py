"""TopK select + all-gather baseline (codec.cpp:147-182,
345-369; collective.cpp:370-390).

CPU: the oracle restatement against the reference (oracle/_ref): selection
with heavy ties (lower index wins), k rounding incl. the 1e-7 epsilon, rate
errors, densify, frame checks, and the SimCluster aggregate. GPU: the
product (prune kernels with the keep-low tie rule + index/value packing)
bit-exact against the oracle, and the all-gather aggregate."""
import struct

import numpy as np
import pytest

from conftest import u32


def tie_heavy(rng, n):
    g = (rng.integers(-20, 21, n) * 0.25).astype(np.float32)  # ~41 distinct values, massive ties
    g[rng.random(n) < 0.05] = -0.0
    return g


@pytest.mark.parametrize("n,rate", [(1, 0.5), (7, 1.0), (10, 0.01), (100, 0.2), (1000, 0.01),
                                    (12_345, 0.1), (4096, 0.999)])
def test_oracle_topk_matches_reference(port, ref, n, rate):
    rng = np.random.default_rng(n)
    for g in (rng.standard_normal(n).astype(np.float32), tie_heavy(rng, n)):
        a, b = port.topk_select(g, rate), ref.topk_select(g, rate)
        assert np.array_equal(a[0], b[0]) and np.array_equal(u32(a[1]), u32(b[1]))


def test_topk_count_and_rate_errors(pb, port, ref):
    for n, rate in ((100, 0.01), (1000, 0.001), (100_000, 0.07), (10, 1.0), (3, 1e-9), (1, 0.3)):
        assert pb.topk_count(n, rate) == ref.topk_select(np.ones(n, np.float32), rate)[0].size  # k incl. epsilon
    assert pb.topk_count(25_557_032, 0.01) == 255_572  # floor(0.01f * len + len * 1e-7)
    for bad in (0.0, -0.1, 1.5, float("nan")):
        with pytest.raises(pb.Error) as e:
            pb.topk_count(10, bad)
        assert e.value.code == pb.Errc.InvalidRate


def test_topk_frame_checks_match_reference(pb, ref):
    import torch

    rng = np.random.default_rng(4)
    g = rng.standard_normal(55).astype(np.float32)
    idx, val = ref.topk_select(g, 0.2)
    p = pb.TopKPayload(torch.from_numpy(idx.view(np.int32)), torch.from_numpy(val), 55)
    frame = pb.encode_topk(p, 7)
    assert len(frame) == 26 + 8 * idx.size
    q = pb.decode_topk(frame, 55)
    assert np.array_equal(q.indices.numpy().view(np.uint32), idx) and np.array_equal(q.values.numpy(), val)
    bads = []
    f = bytearray(frame)
    f[26:30] = struct.pack("<I", 55)  # out of range
    bads.append(bytes(f))
    f = bytearray(frame)
    f[30:34] = f[26:30]  # not strictly increasing
    bads.append(bytes(f))
    bads.append(frame[:-1])
    for fb in bads:
        ours = True
        try:
            pb.decode_topk(fb, 55)
        except pb.Error:
            ours = False
        assert ours == ref.topk_decode_ok(fb, 55)


def test_oracle_topk_mean_matches_reference_aggregate(port, ref):
    rng = np.random.default_rng(6)
    for n in (2, 3, 4):
        ln = 2000
        grads = [tie_heavy(rng, ln) if r % 2 else rng.standard_normal(ln).astype(np.float32) for r in range(n)]
        outs, byts = ref.topk_aggregate(grads, 0.05)
        sel = [port.topk_select(x, 0.05) for x in grads]
        mean = port.topk_mean([s[0] for s in sel], [s[1] for s in sel], ln)
        k = sel[0][0].size
        for r in range(n):
            assert np.array_equal(u32(outs[r]), u32(mean))
            assert byts[r] == (n - 1) * (26 + 8 * k)


# ------------------------------------------------------------------ GPU


@pytest.mark.gpu
@pytest.mark.parametrize("n,rate", [(1, 0.5), (7, 1.0), (100, 0.2), (4097, 0.01), (1_000_003, 0.01),
                                    (2_500_000, 0.3), (25_557_032, 0.01)])
def test_gpu_topk_select_bitexact(pb, port, cuda, n, rate):
    import torch

    rng = np.random.default_rng(n)
    cases = [rng.standard_normal(n).astype(np.float32)]
    if n < 5_000_000:
        cases.append(tie_heavy(rng, n))
    for g in cases:
        p = pb.topk_select(torch.from_numpy(g).cuda(), rate)
        idx, val = port.topk_select(g, rate)
        assert np.array_equal(p.indices.cpu().numpy().view(np.uint32), idx)
        assert np.array_equal(u32(p.values.cpu().numpy()), u32(val))
        d = pb.topk_densify(p).cpu().numpy()
        want = np.zeros(n, np.float32)
        want[idx] = val
        assert np.array_equal(u32(d), u32(want))


@pytest.mark.gpu
def test_gpu_topk_densify_rejects_out_of_range(pb, cuda):
    import torch

    p = pb.TopKPayload(torch.tensor([1, 9], dtype=torch.int32).cuda(), torch.tensor([1.0, 2.0]).cuda(), 9)
    with pytest.raises(pb.Error) as e:
        pb.topk_densify(p)
    assert e.value.code == pb.Errc.CorruptPayload


@pytest.mark.gpu
def test_gpu_topk_aggregate_single_rank(pb, port, cuda):
    import torch

    rng = np.random.default_rng(1)
    g = tie_heavy(rng, 300_001)
    r = pb.topk_allgather_aggregate(torch.from_numpy(g).cuda(), 0.05, 0, None)
    idx, val = port.topk_select(g, 0.05)
    assert r.stats.mode_used == pb.SyncMode.TopKAllGather
    assert np.array_equal(u32(r.tensor.cpu().numpy()), u32(port.topk_mean([idx], [val], g.size)))
