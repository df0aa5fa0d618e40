"""Ternary-on-packed aggregation (codec.cpp:40-75,
313-343; collective.cpp:311-368).

The reference draws from a sequential mt19937_64 stream; the product and the
oracle draw from a counter-based SplitMix64 stream of the same seed (one
independent draw per element on the GPU). Parity is therefore pinned three
ways:
* wherever no draw matters (|g_i| in {0, max}) the product, the oracle and
  the REFERENCE itself (oracle/_ref, mt19937_64) agree bit for bit --
  ternarize, the wire frame, and the whole SimCluster aggregate;
* everywhere, the GPU agrees bit for bit with the oracle restatement using
  the same counter draws (ternarize, decode checks, double-accumulated mean);
* the reference's statistical acceptance test (unbiasedness within 3
  standard errors, test_codec.cpp:109-125) holds for the counter draws.
"""
import struct

import numpy as np
import pytest

from conftest import u32

# ------------------------------------------------------------------ CPU


def saturated(rng, n, s=2.0, zero_frac=0.3):
    v = np.where(rng.random(n) < 0.5, s, -s).astype(np.float32)
    v[rng.random(n) < zero_frac] = 0.0
    return v


def test_oracle_ternarize_matches_reference_when_draws_do_not_matter(port, ref):
    rng = np.random.default_rng(3)
    for n in (1, 2, 3, 4, 5, 9, 64, 1001):
        v = saturated(rng, n, s=float(rng.integers(1, 9)) / 4)
        for seed in (0, 1, 123, 2**63 + 5):
            assert port.ternarize(v, seed)[0] == ref.ternarize(v, seed)[0]
            assert np.array_equal(port.ternarize(v, seed)[1], ref.ternarize(v, seed)[1])
    # test_codec.cpp:96-107
    s, b = port.ternarize(np.array([1.0, -1.0], np.float32), 123)
    assert s == 1.0 and b[0] == 0b1001
    s, b = port.ternarize(np.zeros(9, np.float32), 5)
    assert s == 0.0 and not b.any() and b.size == 3


def test_oracle_ternarize_scale_edge_cases(port, ref):
    v = np.array([0.5, np.nan, -3.0, 1.0], np.float32)  # NaN skipped by std::max
    assert port.ternarize(v, 1)[0] == ref.ternarize(v, 1)[0] == 3.0
    v = np.array([-0.0, 0.0], np.float32)
    assert port.ternarize(v, 1)[0] == ref.ternarize(v, 1)[0] == 0.0


def test_counter_draws_are_unbiased(port):
    """test_codec.cpp:109-125 restated for the counter-based draws."""
    g = np.array([0.5, -0.25, 1.0], np.float32)
    draws = 20_000  # the GPU test runs the reference's full 200k
    acc = np.zeros(3)
    for d in range(draws):
        s, b = port.ternarize(g, port.derive_seed(2024, d))
        pairs = (b[0] >> np.array([0, 2, 4])) & 3
        acc += s * np.where(pairs == 1, 1.0, np.where(pairs == 2, -1.0, 0.0))
    for i in range(3):
        mean = acc[i] / draws
        var = 1.0 * abs(g[i]) - g[i] * g[i]
        se = np.sqrt(max(var, 0.0) / draws)
        assert abs(mean - g[i]) <= 3.0 * se + 1e-12


def test_oracle_mean_matches_reference_aggregate_saturated(port, ref):
    """SimCluster ternary_allgather_aggregate (the reference, mt19937_64)
    against the oracle pipeline on inputs where no draw matters."""
    from oracle import words_from_bits

    rng = np.random.default_rng(9)
    for n, ln in ((2, 6), (3, 1000), (4, 777)):
        bits = rng.random(ln) < 0.6
        words = words_from_bits(bits)
        grads = [port.gse(saturated(rng, ln, s=float(r + 1)), words) for r in range(n)]
        seeds = [port.derive_seed(5, r) for r in range(n)]
        outs, modes, byts = ref.ternary_aggregate(grads, [words] * n, [1] * n, seeds, 0)
        assert modes == [2] * n
        tern = [port.ternarize(port.pack(g, words), sd) for g, sd in zip(grads, seeds)]
        mean = port.ternary_mean([t[0] for t in tern], [t[1] for t in tern], int(bits.sum()))
        want = port.unpack(mean, port.mask_digest(words, ln), words, ln)
        for r in range(n):
            assert np.array_equal(u32(outs[r]), u32(want)), (n, r)
            # ring all-gather of n-1 ternary frames (26 + 4 + ceil(nnz/4) bytes)
            assert byts[r] == (n - 1) * (30 + (int(bits.sum()) + 3) // 4)
    # test_collective.cpp:287-300
    v = np.array([2, -2, 2, -2, 2, -2], np.float32)
    outs, _, _ = ref.ternary_aggregate([v, v], [words_from_bits(np.ones(6, bool))] * 2, [1, 1],
                                       [port.derive_seed(5, r) for r in range(2)], 0)
    assert all(np.array_equal(o, v) for o in outs)


def test_reference_fallback_is_sum_over_n(port, ref):
    from oracle import words_from_bits

    rng = np.random.default_rng(11)
    n, ln = 3, 501
    words = words_from_bits(rng.random(ln) < 0.5)
    grads = [rng.standard_normal(ln).astype(np.float32) for _ in range(n)]
    outs, modes, byts = ref.ternary_aggregate(grads, [words] * n, [1, 0, 1], [1, 2, 3], 4)
    assert modes == [0] * n
    s = port.ring_allreduce(grads)[0]
    want = (s / np.float32(n)).astype(np.float32)  # sum / float(n), IEEE division
    assert all(np.array_equal(u32(o), u32(want)) for o in outs)


def test_host_ternary_frame_codec_matches_reference(pb, port, ref):
    """encode_ternary / decode_ternary (host wire layer) vs wire:: in the reference."""
    import torch

    rng = np.random.default_rng(5)
    for n in (1, 3, 8, 100, 1001):
        v = rng.standard_normal(n).astype(np.float32)
        s, b = ref.ternarize(v, 999)
        frame = ref.encode_ternary(s, b, n, 7, 0xABCD)
        assert len(frame) == 26 + 4 + (n + 3) // 4  # test_codec.cpp:310-315
        t = pb.TernaryGradient(s, n, torch.from_numpy(np.concatenate([b, np.zeros(16, np.uint8)])))
        assert pb.encode_ternary(t, 7, 0xABCD) == frame
        tt, dg = pb.decode_ternary(frame)
        assert dg == 0xABCD and tt.scale == s and tt.len == n and tt.sign_words() == bytes(b)
        # corrupt frames: the same accept / reject decision as the reference
        bad = []
        f = bytearray(frame)
        f[30] = 0xFF  # reserved 11 patterns (test_codec.cpp:333-336)
        bad.append(bytes(f))
        bad.append(frame[:26] + struct.pack("<f", -1.0) + frame[30:])
        bad.append(frame[:26] + struct.pack("<f", float("inf")) + frame[30:])
        bad.append(frame[:26] + struct.pack("<f", 0.0) + frame[30:])
        if n % 4:
            f = bytearray(frame)
            f[-1] |= 0x80  # bits past the payload length
            bad.append(bytes(f))
        bad.append(frame[:-1])  # truncated
        for fb in bad:
            ref_ok = True
            try:
                ref.decode_ternary(fb)
            except Exception:
                ref_ok = False
            ours_ok = True
            try:
                pb.decode_ternary(fb)
            except pb.Error as e:
                assert e.code in (pb.Errc.CorruptPayload,)
                ours_ok = False
            assert ours_ok == ref_ok, fb[26:40]


# ------------------------------------------------------------------ GPU


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 15, 16, 17, 1000, 65_537, 3_000_001])
def test_gpu_ternarize_bitexact_vs_oracle(pb, port, cuda, n):
    import torch

    rng = np.random.default_rng(n)
    v = rng.standard_normal(n).astype(np.float32)
    if n > 20:
        v[rng.integers(0, n, 5)] = 0.0
        v[3] = -0.0
        v[7] = np.nan
    for seed in (0, 77, 2**64 - 1):
        t = pb.ternarize(torch.from_numpy(v).cuda(), seed)
        s, b = port.ternarize(v, seed)
        assert t.scale == s
        got = t.signs.cpu().numpy()
        assert np.array_equal(got[: b.size], b)
        assert not got[b.size:pb.api.ternary_sign_bytes(n)].any()
        d = pb.deternarize(t).cpu().numpy()
        assert np.array_equal(u32(d), u32(ref_deternarize(s, b, n)))


def ref_deternarize(s, b, n):
    pairs = ((b[:, None] >> np.array([0, 2, 4, 6], dtype=np.uint8)) & 3).reshape(-1)[:n]
    return (np.float32(s) * np.where(pairs == 1, 1.0, np.where(pairs == 2, -1.0, 0.0)).astype(np.float32)
            ).astype(np.float32)


@pytest.mark.gpu
def test_gpu_deternarize_matches_reference_and_rejects_corrupt(pb, ref, cuda):
    import torch

    rng = np.random.default_rng(2)
    n = 4099
    s, b = ref.ternarize(rng.standard_normal(n).astype(np.float32), 31337)
    t = pb.TernaryGradient(s, n, torch.from_numpy(np.concatenate([b, np.zeros(16, np.uint8)])).cuda())
    d = pb.deternarize(t).cpu().numpy()
    assert np.array_equal(u32(d), u32(ref.deternarize(s, b, n)))
    assert set(np.unique(d)) <= {s, -s, 0.0}  # test_codec.cpp:127-136
    for bad_scale, patch in ((s, 0xFF), (-1.0, None), (float("inf"), None), (0.0, None)):
        bb = b.copy()
        if patch is not None:
            bb[0] = patch
        t = pb.TernaryGradient(bad_scale, n, torch.from_numpy(np.concatenate([bb, np.zeros(16, np.uint8)])).cuda())
        with pytest.raises(pb.Error) as e:
            pb.deternarize(t)
        assert e.value.code == pb.Errc.CorruptPayload


@pytest.mark.gpu
def test_gpu_ternarize_unbiased(pb, cuda):
    """test_codec.cpp:109-125 over 200k independent counter draws (positions)."""
    import torch

    g = np.tile(np.array([0.5, -0.25, 1.0], np.float32), 200_000)
    t = pb.ternarize(torch.from_numpy(g).cuda(), pb.api.lib.pact_abi_version() * 2024)
    d = pb.deternarize(t).cpu().numpy().reshape(-1, 3).astype(np.float64)
    draws = d.shape[0]
    for i, gi in enumerate((0.5, -0.25, 1.0)):
        mean = d[:, i].mean()
        se = np.sqrt(max(1.0 * abs(gi) - gi * gi, 0.0) / draws)
        assert abs(mean - gi) <= 3.0 * se + 1e-12


@pytest.mark.gpu
def test_gpu_ternary_aggregate_single_rank(pb, port, cuda):
    import torch

    from oracle import words_from_bits

    rng = np.random.default_rng(8)
    ln = 1_000_003
    bits = rng.random(ln) < 0.1
    words = words_from_bits(bits)
    m = pb.SparsityMask.from_words(torch.from_numpy(words.view(np.int64)).cuda(), ln)
    g = rng.standard_normal(ln).astype(np.float32)
    r = pb.ternary_allgather_aggregate(torch.from_numpy(g).cuda(), m, pb.TrackerStatus.Stable, 99, 3, None)
    assert r.stats.mode_used == pb.SyncMode.TernaryAllGather
    s, b = port.ternarize(port.pack(g, words), 99)
    want = port.unpack(port.ternary_mean([s], [b], int(bits.sum())), port.mask_digest(words, ln), words, ln)
    assert np.array_equal(u32(r.tensor.cpu().numpy()), u32(want))
    r = pb.ternary_allgather_aggregate(torch.from_numpy(g).cuda(), m, pb.TrackerStatus.Unstable, 99, 3, None)
    assert r.stats.mode_used == pb.SyncMode.FullAllReduce
    assert np.array_equal(u32(r.tensor.cpu().numpy()), u32(g))
