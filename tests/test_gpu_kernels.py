"""GPU parity of the sm_100a kernels against the CPU oracle, through the
C-ABI: bit-exact masks/thresholds/packed layouts (north_star), exact digests,
reference error contract, and size-independent properties at full BASELINE
sizes."""
import numpy as np
import pytest
import torch

from conftest import u32
from oracle import bits_from_words, words_from_bits

pytestmark = pytest.mark.gpu


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def expand_bits(words: torch.Tensor, n: int) -> torch.Tensor:
    """device words -> bool[n] (torch ops, test-side only)"""
    w = words.view(-1, 1)
    sh = torch.arange(64, device=words.device, dtype=torch.int64).view(1, 64)
    return ((w >> sh) & 1).view(-1)[:n].bool()


# ----------------------------------------------------------------- prune


def check_prune(pb, port, x, ratio, expect_path=None):
    n = x.size
    st = {}
    m = pb.magnitude_prune(dev(x), ratio, stats=st)
    ref = port.magnitude_prune(x, ratio)
    got = m.words_host()
    assert got.shape == ref.shape
    if not np.array_equal(got, ref):
        bad = np.nonzero(got != ref)[0]
        raise AssertionError(f"n={n} ratio={ratio} words differ at {bad[:5]} stats={st}")
    k = port.drop_count(ratio, n)
    assert m.nnz() == n - min(k, n)
    if 0 < k < n:
        T, c_lt = port.prune_threshold(x, k)
        assert st["threshold"] == T and st["c_lt"] == c_lt, (st, T, c_lt)
    if expect_path is not None:
        assert st["path"] == expect_path, st
    return m, st


def test_prune_golden_cases(pb, port, golden, cuda):
    j, a = golden
    for ex in j["prune_examples"]:
        m = pb.magnitude_prune(dev(np.array(ex["w"], np.float32)), ex["ratio"])
        assert [int(b) for b in bits_from_words(m.words_host(), len(ex["w"]))] == ex["keep"]
    for t, c in enumerate(j["prune_cases"]):
        m = pb.magnitude_prune(dev(a[f"prune_w_{t}"]), c["ratio"])
        assert np.array_equal(m.words_host(), a[f"prune_words_{t}"]), t
        assert m.nnz() == c["nnz"]
        assert m.digest() == c["digest"]


@pytest.mark.parametrize("n", [1, 2, 63, 64, 65, 4095, 4096, 4097, 12289, 100_003, 1_000_001])
def test_prune_ragged_lengths(pb, port, cuda, n):
    rng = np.random.default_rng(n)
    for ratio in (0.1, 0.5, 0.9, 0.99):
        check_prune(pb, port, rng.standard_normal(n).astype(np.float32), ratio)


def test_prune_tie_heavy(pb, port, cuda):
    from paper_2505_18563_b200 import synth

    rng = np.random.default_rng(1)
    for n in (5000, 300_000, 2_000_000):
        x = (rng.integers(-6, 7, n) * 0.25).astype(np.float32)
        x[rng.random(n) < 0.2] = -0.0  # +-0 tie at key 0
        for ratio in (0.3, 0.5, 0.8, 0.95):
            check_prune(pb, port, x, ratio)
    x = synth.synth_host(3_000_000, 77, synth.W_TIES, 2.0 ** -5)
    for ratio in (0.5, 0.9):
        check_prune(pb, port, x, ratio)


def test_prune_all_equal_and_zeros(pb, port, cuda):
    for n in (10, 5000, 200_000):
        check_prune(pb, port, np.full(n, 0.5, np.float32), 0.5)
        check_prune(pb, port, np.zeros(n, np.float32), 0.7)


def test_prune_ratio_bounds(pb, port, cuda):
    x = np.random.default_rng(2).standard_normal(10_000).astype(np.float32)
    m = pb.magnitude_prune(dev(x), 0.0)
    assert m.nnz() == 10_000
    for r in (1.0, -0.1):
        with pytest.raises(pb.Error) as e:
            pb.magnitude_prune(dev(x), r)
        assert e.value.code == pb.Errc.InvalidRatio


def test_prune_fallback_path(pb, port, cuda):
    """Adversarial input: every sampled position is 0 while the rest is large,
    so the sampled window misses and the full radix path must take over."""
    n = 1_000_000
    x = np.random.default_rng(3).uniform(1.0, 2.0, n).astype(np.float32)
    S = 16384
    pos = (np.arange(S, dtype=np.uint64) * np.uint64(n) + np.uint64(n // 2)) // np.uint64(S)
    x[pos.astype(np.int64)] = 0.0
    check_prune(pb, port, x, 0.5, expect_path=2)


def test_prune_sort_oracle_property(pb, cuda):
    """test_sparsity.cpp:49-69: 1000 gaussians at 0.8 keep 200, min kept >= max dropped."""
    rng = np.random.default_rng(17)
    for _ in range(20):
        x = rng.standard_normal(1000).astype(np.float32)
        m = pb.magnitude_prune(dev(x), 0.8)
        assert m.nnz() == 200
        keep = bits_from_words(m.words_host(), 1000)
        assert np.abs(x[keep]).min() >= np.abs(x[~keep]).max()


def test_prune_changed_flag_and_digest_cache(pb, port, cuda):
    rng = np.random.default_rng(4)
    x = rng.standard_normal(500_000).astype(np.float32)
    m = pb.magnitude_prune(dev(x), 0.9)
    d = m.digest()
    pb.magnitude_prune(dev(x), 0.9, out=m)
    assert not m.changed and m.digest() == d
    x[np.argmax(np.abs(x))] = 0.0  # the largest becomes the smallest -> mask moves
    pb.magnitude_prune(dev(x), 0.9, out=m)
    assert m.changed
    assert m.digest() == port.mask_digest(port.magnitude_prune(x, 0.9), x.size)


# ----------------------------------------------------------------- codec


def test_codec_golden(pb, golden, cuda):
    j, a = golden
    for t, c in enumerate(j["codec_cases"]):
        g = dev(a[f"codec_g_{t}"])
        m = pb.SparsityMask.from_words(dev(a[f"codec_words_{t}"].view(np.int64)), c["n"])
        assert m.digest() == c["digest"]
        p = pb.pack(g, m, t)
        assert p.mask_digest == c["digest"] and p.epoch == t
        assert np.array_equal(u32(p.values.cpu().numpy()), u32(a[f"codec_packed_{t}"]))
        u = pb.unpack(p, m)
        assert np.array_equal(u32(u.cpu().numpy()), u32(a[f"codec_unpacked_{t}"]))
        gse = pb.enforce_gradient_sparsity(g, m)
        assert np.array_equal(u32(gse.cpu().numpy()), u32(a[f"codec_unpacked_{t}"]))


@pytest.mark.parametrize("n", [1, 77, 4096, 4097, 65_537, 2_500_003])
@pytest.mark.parametrize("density", [0.0, 0.01, 0.2, 0.5, 1.0])
def test_pack_unpack_random(pb, port, cuda, n, density):
    rng = np.random.default_rng(n + int(density * 100))
    g = rng.standard_normal(n).astype(np.float32)
    g[rng.random(n) < 0.01] = -0.0
    bits = rng.random(n) < density
    w = words_from_bits(bits)
    m = pb.SparsityMask.from_words(dev(w.view(np.int64)), n)
    assert m.nnz() == int(bits.sum())
    p = pb.pack(dev(g), m, 1)
    ref = port.pack(g, w)
    assert np.array_equal(u32(p.values.cpu().numpy()), u32(ref))
    u = pb.unpack(p, m)
    assert np.array_equal(u32(u.cpu().numpy()), u32(port.gse(g, w)))


def test_unaligned_and_inplace(pb, port, cuda):
    """pointers off the 16-byte grid take the scalar path; GSE in place."""
    rng = np.random.default_rng(9)
    n = 100_001
    big = rng.standard_normal(n + 3).astype(np.float32)
    g_h = big[1:n + 1]
    bits = rng.random(n) < 0.3
    w = words_from_bits(bits)
    m = pb.SparsityMask.from_words(dev(w.view(np.int64)), n)
    gd = dev(big)[1:n + 1]
    p = pb.pack(gd, m, 0)
    assert np.array_equal(u32(p.values.cpu().numpy()), u32(port.pack(g_h, w)))
    out = torch.zeros(n + 1, device=cuda)[1:]
    pb.unpack(p, m, out=out)
    assert np.array_equal(u32(out.cpu().numpy()), u32(port.gse(g_h, w)))
    x = dev(g_h.copy())
    pb.enforce_gradient_sparsity(x, m, out=x)
    assert np.array_equal(u32(x.cpu().numpy()), u32(port.gse(g_h, w)))


@pytest.mark.parametrize("n", [1, 31, 1000, 1025, 65_537, 300_007])
def test_no_writes_outside_outputs(pb, port, cuda, n):
    """Bounds check without a sanitizer: pack / unpack / GSE / unpack_sgd /
    masked_allreduce write into buffers flanked by 64-float canaries (at
    16-byte-aligned and unaligned offsets); the canaries must survive and
    the payload must match the oracle."""
    import ctypes as C

    rng = np.random.default_rng(n)
    g_h = rng.standard_normal(n).astype(np.float32)
    bits = rng.random(n) < 0.37
    w = words_from_bits(bits)
    m = pb.SparsityMask.from_words(dev(w.view(np.int64)), n)
    nnz = int(bits.sum())
    canary = -12345.5
    for lead in (64, 65):  # aligned / unaligned payload start
        def framed(k):
            buf = torch.full((lead + k + 64,), canary, device=cuda)
            return buf, buf[lead:lead + k]

        def intact(buf, k):
            b = buf.cpu().numpy()
            return bool(np.all(b[:lead] == canary) and np.all(b[lead + k:] == canary))

        gd = dev(g_h)
        pbuf, packed = framed(max(nnz, 1))
        ctx = pb.Context.get()
        pb.api._call(pb.api.lib.pact_pack, ctx.handle, pb.api._ptr(gd), n, m.handle, pb.api._ptr(packed), 0,
                     C.c_uint64(2 ** 64 - 1), pb.api._stream())
        assert intact(pbuf, nnz), "pack wrote outside the packed vector"
        assert np.array_equal(u32(packed[:nnz].cpu().numpy()), u32(port.pack(g_h, w)))
        obuf, out = framed(n)
        pb.unpack(pb.PackedGradient(m.digest(), 0, packed[:nnz]), m, out=out)
        assert intact(obuf, n), "unpack wrote outside the output"
        assert np.array_equal(u32(out.cpu().numpy()), u32(port.gse(g_h, w)))
        ebuf, eout = framed(n)
        pb.enforce_gradient_sparsity(gd, m, out=eout)
        assert intact(ebuf, n), "GSE wrote outside the output"
        wbuf, wts = framed(n)
        wts.copy_(gd)
        pb.unpack_sgd(packed[:nnz], m, 0.5, 0.25, wts)
        assert intact(wbuf, n), "unpack_sgd wrote outside the weights"
        rbuf, rout = framed(n)
        pb.masked_allreduce(gd, m, pb.TrackerStatus.Stable, 0, None, out=rout)
        assert intact(rbuf, n), "masked_allreduce wrote outside the output"
        assert np.array_equal(u32(rout.cpu().numpy()), u32(port.gse(g_h, w)))


def test_codec_errors(pb, cuda):
    m = pb.SparsityMask.all_ones(2)
    p = pb.pack(dev(np.array([1.0, 2.0], np.float32)), m, 0)
    p.mask_digest ^= 1
    with pytest.raises(pb.Error) as e:
        pb.unpack(p, m)
    assert e.value.code == pb.Errc.MaskMismatch
    m3 = pb.SparsityMask.all_ones(3)
    with pytest.raises(pb.Error) as e:
        pb.unpack(pb.PackedGradient(m3.digest(), 0, dev(np.array([1.0, 2.0], np.float32))), m3)
    assert e.value.code == pb.Errc.CorruptPayload
    with pytest.raises(pb.Error) as e:
        pb.enforce_gradient_sparsity(dev(np.ones(1, np.float32)), pb.SparsityMask.all_ones(2))
    assert e.value.code == pb.Errc.ShapeMismatch
    with pytest.raises(pb.Error) as e:
        pb.pack(dev(np.ones(5, np.float32)), pb.SparsityMask.all_ones(4), 0)
    assert e.value.code == pb.Errc.ShapeMismatch
    z = pb.SparsityMask.all_zeros(4)  # empty payload over an all-zero mask
    u = pb.unpack(pb.PackedGradient(z.digest(), 0, torch.empty(0, device=cuda)), z)
    assert torch.all(u == 0)


def test_mask_constructors(pb, port, cuda):
    assert pb.SparsityMask.all_zeros(64).digest() == 0xA8C7F832281A39C5
    assert pb.SparsityMask.all_ones(11).digest() == 0xB57A47E34A2684D3
    assert pb.SparsityMask.all_ones(77).nnz() == 77
    m = pb.SparsityMask.all_zeros(130).with_bit(0, True).with_bit(64, True).with_bit(129, True)
    assert m.nnz() == 3 and m.test(0) and m.test(64) and m.test(129)
    m = m.with_bit(64, False)
    assert m.nnz() == 2
    # digest flips on every single-bit change (test_tensor.cpp:103-117, sampled)
    rng = np.random.default_rng(99)
    for _ in range(50):
        n = int(rng.integers(1, 512))
        bits = rng.random(n) < 0.5
        a = pb.SparsityMask.from_bits(bits)
        i = int(rng.integers(0, n))
        b = a.with_bit(i, not bits[i])
        assert a.digest() != b.digest()
        assert a.digest() == port.mask_digest(words_from_bits(bits), n)


@pytest.mark.parametrize("n", [1, 64, 4096 * 64, 16384 * 128 + 5, 33_554_432 + 64 * 300 + 7, 170_000_000])
def test_digest_sizes(pb, port, cuda, n):
    """crosses segment (16384 elements) and group (2M elements) boundaries"""
    rng = np.random.default_rng(n % 1000)
    nw = (n + 63) // 64
    w = rng.integers(0, 2**63, nw, dtype=np.uint64) ^ rng.integers(0, 2, nw, dtype=np.uint64) << np.uint64(63)
    if n % 64:
        w[-1] &= np.uint64((1 << (n % 64)) - 1)
    m = pb.SparsityMask.from_words(dev(w.view(np.int64)), n)
    assert m.digest() == port.mask_digest(w, n)
    assert m.nnz() == port.mask_nnz(w, n)


def test_single_gpu_masked_allreduce(pb, port, cuda):
    rng = np.random.default_rng(12)
    n = 1_234_567
    g = rng.standard_normal(n).astype(np.float32)
    bits = rng.random(n) < 0.2
    w = words_from_bits(bits)
    m = pb.SparsityMask.from_words(dev(w.view(np.int64)), n)
    r = pb.masked_allreduce(dev(g), m, pb.TrackerStatus.Stable, 5, None)
    assert r.stats.mode_used == pb.SyncMode.PackedAllReduce and r.stats.bytes_on_wire == 0
    assert np.array_equal(u32(r.tensor.cpu().numpy()), u32(port.gse(g, w)))
    r = pb.masked_allreduce(dev(g), m, pb.TrackerStatus.Unstable, 5, None)
    assert r.stats.mode_used == pb.SyncMode.FullAllReduce
    assert np.array_equal(u32(r.tensor.cpu().numpy()), u32(g))
    pol = pb.SyncPolicy(density_threshold=0.1)
    r = pb.masked_allreduce(dev(g), m, pb.TrackerStatus.Stable, 5, None, policy=pol)
    assert r.stats.mode_used == pb.SyncMode.FullAllReduce and r.stats.fallback_reason == 3
    pol = pb.SyncPolicy(scale=0.5)
    r = pb.masked_allreduce(dev(g), m, pb.TrackerStatus.Stable, 5, None, policy=pol)
    assert np.array_equal(u32(r.tensor.cpu().numpy()), u32(port.to_mean(port.gse(g, w), 2)))
    with pytest.raises(pb.Error) as e:
        pb.masked_allreduce(dev(g[:-1]), m, pb.TrackerStatus.Stable, 5, None)
    assert e.value.code == pb.Errc.ShapeMismatch
    # host-buffer (e2e) entry point
    gh = torch.from_numpy(g).pin_memory()
    oh = torch.empty(n, dtype=torch.float32).pin_memory()
    st = pb.masked_allreduce_host(gh, m, pb.TrackerStatus.Stable, 5, None, oh)
    assert st.mode_used == pb.SyncMode.PackedAllReduce
    assert np.array_equal(u32(oh.numpy()), u32(port.gse(g, w)))
    # pipelined segments (len > 8 MiB) on every mode of the host entry point
    n2 = 5_000_011
    g2 = rng.standard_normal(n2).astype(np.float32)
    w2 = words_from_bits(rng.random(n2) < 0.3)
    m2 = pb.SparsityMask.from_words(dev(w2.view(np.int64)), n2)
    gh2 = torch.from_numpy(g2).pin_memory()
    oh2 = torch.empty(n2, dtype=torch.float32).pin_memory()
    for status, pol, want in (
            (pb.TrackerStatus.Stable, pb.SyncPolicy(scale=0.5), port.to_mean(port.gse(g2, w2), 2)),
            (pb.TrackerStatus.Unstable, None, g2),
            (pb.TrackerStatus.Unstable, pb.SyncPolicy(scale=0.25, gse_dense=True), port.to_mean(port.gse(g2, w2), 4))):
        st = pb.masked_allreduce_host(gh2, m2, status, 6, None, oh2, policy=pol)
        assert st.buckets > 1
        assert np.array_equal(u32(oh2.numpy()), u32(want)), (status, pol)


def test_dense_fallback_gse(pb, port, cuda):
    """SyncPolicy.gse_dense: an unmasked gradient aggregated on the dense
    path equals GSE-then-aggregate (trainer.cpp:369-377), like the packed one."""
    rng = np.random.default_rng(21)
    n = 777_777
    g = rng.standard_normal(n).astype(np.float32)
    bits = rng.random(n) < 0.3
    w = words_from_bits(bits)
    m = pb.SparsityMask.from_words(dev(w.view(np.int64)), n)
    want = u32(port.to_mean(port.gse(g, w), 4))
    for status in (pb.TrackerStatus.Unstable, pb.TrackerStatus.Stable):
        pol = pb.SyncPolicy(scale=0.25, gse_dense=True)
        gd = dev(g)
        r = pb.masked_allreduce(gd, m, status, 1, None, policy=pol, out=gd)  # in place, like DDP
        assert np.array_equal(u32(r.tensor.cpu().numpy()), want), status


def test_calibrate_density_single_gpu(pb, cuda):
    """pact_calibrate_density on one GPU: well-formed timings; with nothing
    to exchange the dense path (a copy) beats pack + unpack at every density,
    so the measured crossover sits below the sparsest probe."""
    cal = pb.calibrate_density(1 << 21, None, densities=[0.1, 0.5, 0.9])
    assert len(cal.t_packed) == 3 and all(t > 0 for t in cal.t_packed) and cal.t_dense > 0
    assert 0.0 < cal.threshold <= 1.0
    if cal.t_packed[0] >= cal.t_dense:
        assert cal.threshold == pytest.approx(0.05)
    with pytest.raises(pb.Error):
        pb.calibrate_density(1 << 20, None, densities=[0.5, 0.2])


@pytest.mark.parametrize("src_len", [1, 64, 1000, 4096 * 3 + 17, 2_000_003])
def test_mask_gather(pb, cuda, src_len):
    """pact_mask_gather == numpy bit slicing/concatenation (DDP bucket masks)."""
    rng = np.random.default_rng(src_len)
    bits = rng.random(src_len) < 0.37
    src = pb.SparsityMask.from_words(dev(words_from_bits(bits).view(np.int64)), src_len)
    for trial in range(6):
        nseg = int(rng.integers(1, 40))
        segs = []
        for _ in range(nseg):
            b = int(rng.integers(0, src_len))
            ln = int(rng.integers(0, src_len - b + 1)) if trial % 2 else int(rng.integers(0, min(200, src_len - b) + 1))
            segs.append((b, ln))
        want = np.concatenate([bits[b:b + ln] for b, ln in segs]) if segs else np.zeros(0, bool)
        m = pb.api.mask_gather(src, segs)
        assert m.size() == want.size and m.nnz() == int(want.sum())
        assert np.array_equal(m.words_host(), words_from_bits(want)), (trial, segs[:3])
        if want.size:
            assert m.digest() == pb.SparsityMask.from_bits(want).digest()
    with pytest.raises(pb.Error) as e:
        pb.api.mask_gather(src, [(src_len - 1, 2)])
    assert e.value.code == pb.Errc.ShapeMismatch
    with pytest.raises(pb.Error) as e:
        pb.api.mask_gather(src, [(0, 1)], out=pb.SparsityMask(2))
    assert e.value.code == pb.Errc.ShapeMismatch


def test_unpack_sgd_matches_trainer(pb, port, cuda):
    rng = np.random.default_rng(13)
    n = 300_001
    s = rng.standard_normal(n).astype(np.float32)
    wts = rng.standard_normal(n).astype(np.float32)
    bits = rng.random(n) < 0.4
    w = words_from_bits(bits)
    m = pb.SparsityMask.from_words(dev(w.view(np.int64)), n)
    p = pb.pack(dev(s), m, 0)
    wd = dev(wts.copy())
    gout = torch.empty(n, device=cuda)
    pb.unpack_sgd(p.values, m, 1.0 / 8, 0.05, wd, gout)
    mean = port.to_mean(port.gse(s, w), 8)
    assert np.array_equal(u32(gout.cpu().numpy()), u32(mean))
    assert np.array_equal(u32(wd.cpu().numpy()), u32(port.sgd_step(wts, mean, 0.05, w)))


# ------------------------------------------------- full BASELINE sizes


def test_prune_resnet50_full_size_bitexact(pb, port, cuda):
    """C2: ResNet-50 shape (25,557,032) at 80%: words bit-exact vs the oracle."""
    from paper_2505_18563_b200 import synth

    shape = synth.model_shape("resnet50")
    for recipe in (synth.W_REAL, synth.W_TIES):
        wd = synth.weights_device(shape, 21, recipe)
        m = pb.magnitude_prune(wd, 0.8)
        assert m.nnz() == 5_111_404
        ref = port.magnitude_prune(wd.cpu().numpy(), 0.8)
        assert np.array_equal(m.words_host(), ref)
        assert m.digest() == port.mask_digest(ref, shape.total)


# Exact kept counts of SURVEY 8 (drop_count, sparsity.cpp:33-40)
FULL_NNZ = {("resnet18", 0.9): 1_168_951, ("resnet50", 0.8): 5_111_404, ("vgg19", 0.95): 7_183_350,
            ("bert-base", 0.5): 54_741_110, ("bert-base", 0.8): 21_896_436, ("bert-base", 0.9): 10_948_216,
            ("bert-base", 0.95): 5_474_103, ("bert-base", 0.99): 1_094_811, ("gpt2-medium", 0.9): 35_482_290}
C4_SWEEP = (0.5, 0.6, 0.7, 0.8, 0.9, 0.95, 0.99)


def _check_full(pb, port, wd, ratio, n, tag):
    m = pb.magnitude_prune(wd, ratio)
    ref = port.magnitude_prune(wd.cpu().numpy(), ratio)
    assert m.nnz() == n - port.drop_count(ratio, n), tag
    assert np.array_equal(m.words_host(), ref), tag
    assert m.digest() == port.mask_digest(ref, n), tag
    return m, ref


@pytest.mark.parametrize("model,ratios", [("resnet18", (0.9,)), ("vgg19", (0.95,)), ("bert-base", C4_SWEEP),
                                          ("gpt2-medium", (0.9,))])
def test_prune_full_size_bitexact(pb, port, cuda, model, ratios):
    """C1 (global), C3, C4 at every sweep ratio, C5: words, nnz and digest
    bit-exact against the oracle's restatement of sparsity.cpp:44-59 at the
    exact BASELINE sizes, both weight recipes (W_TIES: ~40 exact repeats per
    magnitude at 355M, so the tie ranks decide bits)."""
    from paper_2505_18563_b200 import synth

    shape = synth.model_shape(model)
    n = shape.total
    for recipe in (synth.W_REAL, synth.W_TIES):
        wd = synth.weights_device(shape, 41 + recipe, recipe)
        for ratio in ratios:
            m, _ = _check_full(pb, port, wd, ratio, n, (model, recipe, ratio))
            if (model, ratio) in FULL_NNZ:
                assert m.nnz() == FULL_NNZ[(model, ratio)]
            del m
        del wd
        torch.cuda.empty_cache()


def _perturb(kind, w, keep, rng, synth, step):
    """Re-prune schedules (SURVEY A.9 and moves of the threshold both ways)."""
    n = w.size
    if kind == "same":
        return w
    if kind == "up":  # 40 dropped elements just below T become large: T moves up
        drop = np.nonzero(~keep)[0]
        j = drop[np.argsort(np.abs(w[drop]), kind="stable")[-40:]]
        w = w.copy()
        w[j] = np.float32(4.0) * np.sign(w[j] + np.float32(1e-30))
        return w
    if kind in ("down", "down3k"):  # kept elements just above T become tiny: T moves down
        kept = np.nonzero(keep)[0]
        j = kept[np.argsort(np.abs(w[kept]), kind="stable")[:40 if kind == "down" else 3000]]
        w = w.copy()
        w[j] = np.float32(2.0 ** -40)
        return w
    if kind == "a9":  # w <- GSE(w) + delta: kept entries drift, pruned ones get fresh tiny noise
        jit = synth.synth_host(n, 1000 + step, synth.W_REAL, 2.0 ** -16)
        drift = synth.synth_host(n, 2000 + step, synth.W_REAL, 2.0 ** -12)
        return np.where(keep, w + drift, np.float32(0.0)).astype(np.float32) + jit
    if kind == "a9ties":  # the same with the noise on 2^10 levels: ties at the threshold
        jit = synth.synth_host(n, 3000 + step, synth.W_REAL, 2.0 ** -16)
        jit = (np.round(jit.astype(np.float64) * 2.0 ** 26) * 2.0 ** -26).astype(np.float32)
        return np.where(keep, w, np.float32(0.0)).astype(np.float32) + jit
    if kind == "new":  # unrelated weights: the window misses
        return synth.synth_host(n, 4000 + step, synth.W_REAL, 0.25)
    raise ValueError(kind)


SCHEDULE = ["same", "up", "down", "same", "a9", "a9", "a9", "same", "up", "a9ties", "a9ties", "down3k",
            "a9ties", "down", "new", "same"]


@pytest.mark.parametrize("n", [3_000_017, 200_003])
def test_reprune_sequence_paths(pb, port, cuda, n):
    """Per-step re-pruning (C5's mask regeneration) through every prune path:
    temporal reuse (3), a moved threshold resolved from the bitmap pass's
    window candidates (4, both directions, ties straddling r), the sampled
    path (1). Words and digest bit-exact at every step; `changed` never
    misses a change."""
    from paper_2505_18563_b200 import synth

    for recipe in (synth.W_REAL, synth.W_TIES):
        rng = np.random.default_rng(n + recipe)
        w = synth.synth_host(n, 77 + recipe, recipe, 0.25)
        m = pb.SparsityMask(n)
        prev, paths = None, []
        for t, kind in enumerate(["same"] + SCHEDULE):
            if prev is not None:
                w = _perturb(kind, w, bits_from_words(prev, n), rng, synth, t)
            st = {}
            pb.magnitude_prune(dev(w), 0.9, out=m, stats=st)
            ref = port.magnitude_prune(w, 0.9)
            got = m.words_host()
            assert np.array_equal(got, ref), (recipe, t, kind, st, np.nonzero(got != ref)[0][:5])
            assert m.nnz() == n - port.drop_count(0.9, n)
            if prev is not None and not m.changed:
                assert np.array_equal(ref, prev), (recipe, t, kind, "change missed")
            assert m.digest() == port.mask_digest(ref, n), (recipe, t, kind)
            paths.append((kind, st["path"]))
            prev = ref
        got_paths = [p for _, p in paths]
        assert got_paths.count(3) >= 3, paths
        assert got_paths.count(4) >= 4, paths


def test_bitmap_cpasync_variant(cuda):
    """prune_bitmap_kernel ships in two load variants: the default moves each
    chunk with two cp.async.bulk copies into a linear stage (UBLKCP), the
    PACT_BITMAP_CPASYNC=1 one with per-lane cp.async into a swizzled stage.
    The re-prune schedule above runs bit-exact through the latter too."""
    import os
    import subprocess
    import sys

    env = dict(os.environ, PACT_BITMAP_CPASYNC="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        f"{os.path.abspath(__file__)}::test_reprune_sequence_paths"],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "2 passed" in r.stdout, r.stdout[-1000:]


def test_unpack_bulk_store_variant(cuda):
    """The opt-in unpack variant that stores whole chunks with one 4 KiB
    cp.async.bulk (PACT_UNPACK_BULK=1) is bit-exact through the codec tests
    (golden, random densities, unaligned / in place, canaries, scaling)."""
    import os
    import subprocess
    import sys

    env = dict(os.environ, PACT_UNPACK_BULK="1")
    sel = " or ".join(["test_codec_golden", "test_pack_unpack_random", "test_unaligned_and_inplace",
                       "test_no_writes_outside_outputs", "test_single_gpu_masked_allreduce",
                       "test_full_size_pack_properties"])
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.abspath(__file__), "-k", sel],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout, r.stdout[-1000:]


def test_c5_reprune_a9_full_size(pb, port, cuda):
    """C5 (GPT-2-medium, 354,823,168) per-step re-pruning at 0.9 with the A.9
    recipe (w <- GSE(w) + delta), plus threshold moves both ways: words
    bit-exact against the oracle at every step."""
    from paper_2505_18563_b200 import synth

    shape = synth.model_shape("gpt2-medium")
    n = shape.total
    w = synth.weights_host(shape, 51, synth.W_TIES)
    m = pb.SparsityMask(n)
    prev = None
    rng = np.random.default_rng(5)
    paths = []
    for t, kind in enumerate(["same", "same", "a9", "a9", "up", "down"]):
        if prev is not None:
            w = _perturb(kind, w, bits_from_words(prev, n), rng, synth, t)
        st = {}
        pb.magnitude_prune(dev(w), 0.9, out=m, stats=st)
        ref = port.magnitude_prune(w, 0.9)
        assert np.array_equal(m.words_host(), ref), (t, kind, st)
        assert m.nnz() == 35_482_290
        assert m.digest() == port.mask_digest(ref, n)
        paths.append(st["path"])
        prev = ref
    assert 3 in paths and 4 in paths, paths


@pytest.mark.parametrize("model,ratio,nnz", [("vgg19", 0.95, 7_183_350), ("gpt2-medium", 0.9, 35_482_290)])
def test_full_size_pack_properties(pb, cuda, model, ratio, nnz):
    """C3/C5 sizes: pack -> unpack == GSE and the packed checksum == the
    checksum of the GSE'd gradient (size-independent properties)."""
    from paper_2505_18563_b200 import synth

    shape = synth.model_shape(model)
    wd = synth.weights_device(shape, 31, synth.W_TIES)
    st = {}
    m = pb.magnitude_prune(wd, ratio, stats=st)
    assert m.nnz() == nnz
    keep = expand_bits(m.words(), shape.total)
    key = wd.view(torch.int32) & 0x7FFFFFFF
    assert int(key[keep].min()) >= st["threshold"] >= int(key[~keep].max())
    del key
    g = torch.empty_like(wd)
    pb.synth_fill(g, 5, synth.G_FULL)
    del wd
    p = pb.pack(g, m, 0)
    assert p.values.numel() == nnz
    ref_sum = torch.where(keep, g, torch.zeros((), device=g.device)).double().sum()
    assert float(p.values.double().sum()) == float(ref_sum)
    u = pb.unpack(p, m)
    assert torch.equal(u, torch.where(keep, g, torch.zeros((), device=g.device)))


# ------------------------------------------------- per-layer prune (D1)


def test_per_layer_prune_random_segments(pb, port, cuda):
    rng = np.random.default_rng(21)
    for t in range(12):
        n = int(rng.integers(2000, 400_000))
        nseg = int(rng.integers(1, 40))
        cuts = np.unique(np.concatenate([[0, n], rng.integers(1, n, nseg - 1)]))
        if t % 3 == 0:  # tie heavy with signed zeros and 1-element layers
            x = (rng.integers(-4, 5, n) * 0.5).astype(np.float32)
            x[rng.random(n) < 0.1] = -0.0
            cuts = np.unique(np.concatenate([cuts, cuts[1:-1] + 1]))
            cuts = cuts[cuts <= n]
        else:
            x = (rng.standard_normal(n) * np.exp2(rng.integers(-6, 3, n))).astype(np.float32)
        for ratio in (0.0, 0.5, 0.9, 0.99):
            m = pb.magnitude_prune_per_layer(dev(x), [int(c) for c in cuts], ratio)
            ref = port.magnitude_prune_segmented(x, cuts, ratio)
            assert np.array_equal(m.words_host(), ref), (t, ratio)
            assert m.nnz() == port.mask_nnz(ref, n)


def test_per_layer_prune_model_shapes(pb, port, cuda):
    from paper_2505_18563_b200 import synth

    shape = synth.model_shape("resnet18")
    offs = shape.offsets()
    for recipe in (synth.W_TIES, synth.W_REAL):
        wd = synth.weights_device(shape, 9, recipe)
        m = pb.magnitude_prune_per_layer(wd, offs, 0.9)
        ref = port.magnitude_prune_segmented(wd.cpu().numpy(), np.array(offs, np.uint64), 0.9)
        assert np.array_equal(m.words_host(), ref)
        assert m.digest() == port.mask_digest(ref, shape.total)


def test_per_layer_reprune_sequence(pb, port, cuda):
    """Per-layer re-pruning into the same mask (temporal reuse: one bitmap
    pass at every layer's previous threshold, verified per layer, else the
    full path): words bit-exact against the oracle's per-slice rule at every
    step of a schedule that keeps, moves (both ways) and scrambles the
    thresholds, with tie-heavy weights, and across a ratio change and a
    changed layer table (the cache is keyed on both)."""
    from paper_2505_18563_b200 import synth

    shape = synth.model_shape("resnet18")
    n = shape.total
    offs = shape.offsets()
    cuts = np.array(offs, np.uint64)
    for recipe in (synth.W_REAL, synth.W_TIES):
        rng = np.random.default_rng(7 + recipe)
        w = synth.weights_host(shape, 17 + recipe, recipe)
        m = pb.SparsityMask(n)
        prev = None
        sizes = np.diff(np.array(offs))
        small = [i for i in range(len(sizes)) if 4096 <= sizes[i] <= n // 16]
        for t, kind in enumerate(["same", "same", "layer", "same", "layer", "up", "a9", "a9ties", "down", "same",
                                  "new", "same"]):
            if kind == "layer":  # one layer's weights re-drawn: only its threshold moves (partial re-select)
                i = small[(t * 7) % len(small)]
                w = w.copy()
                w[offs[i]:offs[i + 1]] = rng.standard_normal(sizes[i]).astype(np.float32) * np.float32(0.05)
            elif prev is not None:
                w = _perturb(kind, w, bits_from_words(prev, n), rng, synth, t)
            pb.magnitude_prune_per_layer(dev(w), offs, 0.9, out=m)
            ref = port.magnitude_prune_segmented(w, cuts, 0.9)
            assert np.array_equal(m.words_host(), ref), (recipe, t, kind)
            assert m.nnz() == port.mask_nnz(ref, n)
            if prev is not None and not m.changed:  # an unchanged mask keeps its digest
                assert np.array_equal(ref, prev), (recipe, t, kind, "change missed")
            assert m.digest() == port.mask_digest(ref, n)
            prev = ref
        for ratio, table in ((0.8, offs), (0.8, [0, 5000] + [o for o in offs[1:] if o > 5000])):
            pb.magnitude_prune_per_layer(dev(w), table, ratio, out=m)
            pb.magnitude_prune_per_layer(dev(w), table, ratio, out=m)  # the reuse of the new key
            ref = port.magnitude_prune_segmented(w, np.array(table, np.uint64), ratio)
            assert np.array_equal(m.words_host(), ref), (recipe, ratio, len(table))


@pytest.mark.parametrize("model", ["gpt2-medium", "bert-base"])
def test_per_layer_prune_full_size(pb, port, cuda, model):
    """Per-layer mode (north_star (1)) at C5 / C4 size: every
    layer's own k-th threshold, words bit-exact against the oracle applied to
    each layer slice, both weight recipes."""
    from paper_2505_18563_b200 import synth

    shape = synth.model_shape(model)
    offs = shape.offsets()
    for recipe in (synth.W_REAL, synth.W_TIES):
        wd = synth.weights_device(shape, 61 + recipe, recipe)
        m = pb.magnitude_prune_per_layer(wd, offs, 0.9)
        ref = port.magnitude_prune_segmented(wd.cpu().numpy(), np.array(offs, np.uint64), 0.9)
        assert np.array_equal(m.words_host(), ref), (model, recipe)
        assert m.nnz() == port.mask_nnz(ref, shape.total)
        del wd, m
        torch.cuda.empty_cache()


def test_per_layer_prune_errors(pb, cuda):
    x = dev(np.ones(100, np.float32))
    for bad in ([0, 50], [0, 50, 50, 100], [1, 100]):
        with pytest.raises(pb.Error) as e:
            pb.magnitude_prune_per_layer(x, bad, 0.5)
        assert e.value.code == pb.Errc.InvalidView
    with pytest.raises(pb.Error) as e:
        pb.magnitude_prune_per_layer(x, [0, 100], 1.0)
    assert e.value.code == pb.Errc.InvalidRatio


def test_max_len_prune_pack_unpack(pb, port, cuda):
    """len = PACT_MAX_LEN = 2^31 - 1 (8 GiB of fp32, larger than GPT-2-XL's
    1.56B; an odd length, so a ragged last word and chunk): words and digest
    bit-exact against the oracle at 0.9, then pack -> unpack == GSE. One past
    the limit is refused with a shape error."""
    from paper_2505_18563_b200 import synth

    n = (1 << 31) - 1
    wd = torch.empty(n, dtype=torch.float32, device="cuda")
    pb.synth_fill(wd, 91, synth.W_TIES, 0.25)
    m, _ = _check_full(pb, port, wd, 0.9, n, "max_len")
    keep = expand_bits(m.words(), n)
    g = wd  # reuse the buffer: the gradient
    pb.synth_fill(g, 7, synth.G_FULL)
    p = pb.pack(g, m, 0)
    assert p.values.numel() == m.nnz()
    u = pb.unpack(p, m)
    assert torch.equal(u, torch.where(keep, g, torch.zeros((), device=g.device)))
    del u, p, keep, g, wd, m
    torch.cuda.empty_cache()
    with pytest.raises(pb.Error) as ei:
        pb.SparsityMask(n + 1)
    assert ei.value.code == pb.Errc.ShapeMismatch
