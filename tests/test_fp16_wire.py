"""binary16 wire: the reference's hand-rolled conversions
(codec.cpp:79-146), the F16Wire ring (collective.cpp:133-216, 261-267), and
the packed variant (masked_allreduce with the packed values on the binary16
ring; policy.wire = F16).

CPU: the oracle restatement against the reference itself -- every binary16
value, rounding boundaries, random float bit patterns, and SimCluster
fp16_allreduce for n = 2..5 (bit-exact, bytes_on_wire). GPU: the kernels
against the oracle on the same inputs."""
import numpy as np
import pytest

from conftest import u32


def float_cases(rng, n_random=1 << 20):
    halves = np.arange(1 << 16, dtype=np.uint32)
    # every binary16 value's float and the float neighbours around it and
    # around the midpoints (the rounding boundaries)
    h_as_f = np.zeros(1 << 16, np.float32)
    mant = halves & 0x3FF
    exp = (halves >> 10) & 0x1F
    sign = (halves & 0x8000) << 16
    normal = (exp > 0) & (exp < 31)
    bits = np.where(normal, sign | ((exp + 112) << 23) | (mant << 13), sign)
    h_as_f = bits.astype(np.uint32).view(np.float32)
    near = []
    for d in (-2, -1, 1, 2, 4095, 4096, 4097, -4095, -4096, -4097):
        near.append((bits.astype(np.int64) + d).clip(0, 0xFFFFFFFF).astype(np.uint32))
    rnd = rng.integers(0, 1 << 32, n_random, dtype=np.uint64).astype(np.uint32)
    special = np.array([0, 0x80000000, 0x7F800000, 0xFF800000, 0x7FC00000, 0xFFC00001, 0x7F800001,
                        0x477FE000, 0x477FEFFF, 0x477FF000, 0x47800000, 0x33000000, 0x33000001,
                        0x32FFFFFF, 0x387FC000, 0x38800000, 0x00000001, 0x7F7FFFFF], np.uint32)
    allb = np.concatenate([bits.astype(np.uint32)] + near + [rnd, special])
    return allb.view(np.float32), h_as_f


def test_conversions_match_reference(port, ref):
    rng = np.random.default_rng(1)
    f, _ = float_cases(rng)
    assert np.array_equal(port.float_to_half(f), ref.float_to_half(f))
    h = np.arange(1 << 16, dtype=np.uint16)
    assert np.array_equal(u32(port.half_to_float(h)), u32(ref.half_to_float(h)))
    # clamping contract (codec.hpp:55-57): beyond range and +-Inf -> +-65504
    big = np.array([65520.0, 1e30, np.inf, -np.inf, -7e4], np.float32)
    assert (port.half_to_float(port.float_to_half(big)) == np.array([65504, 65504, 65504, -65504, -65504],
                                                                    np.float32)).all()


@pytest.mark.parametrize("n", [2, 3, 4, 5])
def test_oracle_fp16_ring_matches_reference(port, ref, n):
    rng = np.random.default_rng(n)
    ln = 1009
    ins = [(rng.standard_normal(ln) * rng.choice([1e-6, 1.0, 3e4], ln)).astype(np.float32) for _ in range(n)]
    outs, byts = ref.fp16_allreduce(ins)
    mine = port.ring_allreduce_fp16(ins)
    for r in range(n):
        assert np.array_equal(u32(mine[r]), u32(outs[r]))
        assert byts[r] == port.ring_bytes(n, r, ln) // 2


# ------------------------------------------------------------------ GPU


@pytest.mark.gpu
def test_gpu_roundtrip_bitexact(pb, port, cuda):
    import torch

    rng = np.random.default_rng(2)
    f, h_as_f = float_cases(rng, 1 << 22)
    got = pb.fp16_roundtrip(torch.from_numpy(f).cuda()).cpu().numpy()
    want = port.half_to_float(port.float_to_half(f))
    assert np.array_equal(u32(got), u32(want))
    # every binary16 value is a fixed point
    got = pb.fp16_roundtrip(torch.from_numpy(h_as_f).cuda()).cpu().numpy()
    assert np.array_equal(u32(got), u32(port.half_to_float(port.float_to_half(h_as_f))))


@pytest.mark.gpu
def test_gpu_roundtrip_exhaustive_near_half_range(pb, port, cuda):
    """The wire encode is the hardware cvt.rn.f16.f32 with the reference's
    special-value rules patched on (f16wire.cu): every fp32 of both signs
    with a biased exponent in [96, 145] -- below the smallest subnormal's
    half through the clamp region, every mantissa -- plus every binary16
    pattern decoded, bit-exact against the reference's conversions."""
    import torch

    mant = np.arange(1 << 23, dtype=np.uint32)
    for sign in (0, 1):
        for e in list(range(96, 146)) + [0, 1, 200, 254, 255]:
            bits = (np.uint32(sign << 31) | np.uint32(e << 23) | mant).view(np.float32)
            got = pb.fp16_roundtrip(torch.from_numpy(bits).cuda()).cpu().numpy()
            want = port.half_to_float(port.float_to_half(bits))
            bad = np.nonzero(u32(got) != u32(want))[0]
            assert bad.size == 0, (sign, e, hex(int(u32(bits)[bad[0]])), hex(int(u32(got)[bad[0]])),
                                   hex(int(u32(want)[bad[0]])))
    h = np.arange(1 << 16, dtype=np.uint32)
    f = port.half_to_float(h.astype(np.uint16))
    got = pb.fp16_roundtrip(torch.from_numpy(f).cuda()).cpu().numpy()
    assert np.array_equal(u32(got), u32(port.half_to_float(port.float_to_half(f))))


@pytest.mark.gpu
def test_gpu_fp16_single_rank_and_packed_wire(pb, port, cuda):
    import torch

    from oracle import words_from_bits

    rng = np.random.default_rng(3)
    ln = 500_001
    g = (rng.standard_normal(ln) * 100).astype(np.float32)
    r = pb.fp16_allreduce(torch.from_numpy(g).cuda(), None)
    assert r.stats.mode_used == pb.SyncMode.Fp16AllReduce
    assert np.array_equal(u32(r.tensor.cpu().numpy()), u32(port.half_to_float(port.float_to_half(g))))
    bits = rng.random(ln) < 0.25
    words = words_from_bits(bits)
    m = pb.SparsityMask.from_words(torch.from_numpy(words.view(np.int64)).cuda(), ln)
    res = pb.masked_allreduce(torch.from_numpy(g).cuda(), m, pb.TrackerStatus.Stable, 1, None,
                              policy=pb.SyncPolicy(wire=pb.SyncPolicy.F16))
    packed = port.half_to_float(port.float_to_half(port.pack(g, words)))
    want = port.unpack(packed, port.mask_digest(words, ln), words, ln)
    assert res.stats.mode_used == pb.SyncMode.PackedAllReduce
    assert np.array_equal(u32(res.tensor.cpu().numpy()), u32(want))
