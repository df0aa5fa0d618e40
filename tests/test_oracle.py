"""Pin the CPU restatement (oracle/pact_oracle.c) against the reference's own
known answers and against fixtures produced by the reference itself
(tests/golden/, generated from oracle/_ref by tests/golden/make_golden.py),
plus a live cross-check against oracle/_ref where it is built."""
import numpy as np
import pytest

from conftest import u32
from oracle import words_from_bits


def test_digest_goldens(port, golden):
    j, a = golden
    assert port.mask_digest(np.zeros(1, np.uint64), 64) == 0xA8C7F832281A39C5  # test_tensor.cpp:91
    assert port.mask_digest(np.zeros(1, np.uint64), 64) == j["digest_all_zeros_64"]
    assert port.mask_digest(words_from_bits(np.ones(11, bool)), 11) == j["digest_all_ones_11"]
    assert port.mask_digest(np.zeros(0, np.uint64), 0) == j["digest_empty"]
    for t, c in enumerate(j["digest_cases"]):
        w = a[f"dig_words_{t}"]
        assert port.mask_digest(w, c["n"]) == c["digest"]
        assert port.mask_nnz(w, c["n"]) == c["nnz"]


def test_fnv_bytes(port):
    assert port.fnv1a64(b"") == 0xCBF29CE484222325
    assert port.fnv1a64(b"\0" * 8) == 0xA8C7F832281A39C5


def test_prune_examples(port, golden):
    j, a = golden
    for ex in j["prune_examples"]:
        w = port.magnitude_prune(np.array(ex["w"], np.float32), ex["ratio"])
        bits = [(int(w[0]) >> i) & 1 for i in range(len(ex["w"]))]
        assert bits == ex["keep"]


def test_prune_cases_match_reference(port, golden):
    j, a = golden
    for t, c in enumerate(j["prune_cases"]):
        w = port.magnitude_prune(a[f"prune_w_{t}"], c["ratio"])
        assert np.array_equal(w, a[f"prune_words_{t}"]), t
        assert port.mask_nnz(w, c["n"]) == c["nnz"]
        assert port.mask_digest(w, c["n"]) == c["digest"]


def test_prune_rejects_bad_ratio(port):
    import oracle.oracle as oo

    for r in (1.0, -0.1, 2.0):
        with pytest.raises(oo.OracleError) as e:
            port.magnitude_prune(np.ones(3, np.float32), r)
        assert e.value.code == 3  # InvalidRatio


def test_drop_count_table(port, golden):
    j, _ = golden
    for e in j["drop_counts"]:
        assert port.drop_count(e["ratio"], e["len"]) == e["k"]


def test_prune_threshold_consistent(port, golden):
    j, a = golden
    for t, c in enumerate(j["prune_cases"][:30]):
        x = a[f"prune_w_{t}"]
        k = port.drop_count(c["ratio"], c["n"])
        T, c_lt = port.prune_threshold(x, k)
        keys = x.view(np.uint32) & 0x7FFFFFFF
        if k:
            assert (keys < T).sum() == c_lt
            assert c_lt < k <= c_lt + (keys == T).sum()


def test_codec_cases(port, golden):
    j, a = golden
    for t, c in enumerate(j["codec_cases"]):
        g, w = a[f"codec_g_{t}"], a[f"codec_words_{t}"]
        p = port.pack(g, w)
        assert np.array_equal(u32(p), u32(a[f"codec_packed_{t}"]))
        u = port.unpack(p, c["digest"], w, c["n"])
        assert np.array_equal(u32(u), u32(a[f"codec_unpacked_{t}"]))
        assert np.array_equal(u32(port.gse(g, w)), u32(u))


def test_unpack_errors(port):
    import oracle.oracle as oo

    w = words_from_bits(np.ones(2, bool))
    d = port.mask_digest(w, 2)
    with pytest.raises(oo.OracleError) as e:
        port.unpack(np.ones(2, np.float32), d ^ 1, w, 2)
    assert e.value.code == 7  # MaskMismatch
    with pytest.raises(oo.OracleError) as e:
        port.unpack(np.ones(1, np.float32), d, w, 2)
    assert e.value.code == 8  # CorruptPayload


def test_header(port, golden):
    j, _ = golden
    assert port.encode_header(1, 0x01020304, 0x1122334455667788, 5).hex() == j["header_packed"]
    assert port.encode_header(0, 7, 0xDEADBEEFCAFEF00D, 123456789).hex() == j["header_full"]


def test_ring_fold_order(port, golden):
    j, a = golden
    for c in j["ring_cases"]:
        key = f"ring_{c['n']}_{c['len']}"
        xs = list(a[key + "_in"])
        outs = port.ring_allreduce(xs)
        for o in outs:
            assert np.array_equal(u32(o), u32(a[key + "_out"])), key
        assert [port.ring_bytes(c["n"], p, c["len"]) for p in range(c["n"])] == c["bytes"]
    o = port.ring_allreduce([np.array([1e8], np.float32), np.array([-1e8], np.float32), np.array([1.0], np.float32)])
    assert [float(o[0][0])] == j["ring_fold_probe_n3"]


def test_masked_allreduce_cases(port, golden):
    j, a = golden
    for c in j["masked_cases"]:
        nm = c["name"]
        grads = list(a[f"masked_{nm}_grads"])
        masks = list(a[f"masked_{nm}_masks"])
        outs, modes, byts = port.masked_allreduce(grads, masks, c["stable"], c["epoch"], c["advertised"])
        assert modes == c["modes"], nm
        assert byts == c["bytes"], nm
        for o, e in zip(outs, a[f"masked_{nm}_outs"]):
            assert np.array_equal(u32(o), u32(e)), nm


def test_acceptance5_byte_ratios(port, golden):
    j, _ = golden
    for c in j["acceptance5"]:
        pbytes = 26 + port.ring_bytes(2, 0, c["nnz"])
        assert pbytes == c["packed_bytes"]
        assert port.ring_bytes(2, 0, 1_000_000) == c["full_bytes"]
        assert abs(c["ratio_bytes"] - (1 - c["ratio"])) < 0.01


def test_tracker_and_decide(port, golden):
    j, a = golden
    import ctypes as C

    t = (C.c_uint8 * 64)()
    port.L.orc_tracker_init.argtypes = [C.c_void_p, C.c_uint32]
    port.L.orc_tracker_init(t, 3)
    masks = [a[f"tracker_mask_{i}"] for i in range(4)]
    digests = [port.mask_digest(m, 32) for m in masks]
    port.L.orc_tracker_observe.argtypes = [C.c_void_p, C.c_uint64]
    got = [port.L.orc_tracker_observe(t, digests[s]) for s in j["tracker_seq"]["seq"]]
    assert got == j["tracker_seq"]["status"]
    for k, v in j["decide_sync_mode"].items():
        r, s = map(int, k.split("_"))
        assert port.decide_sync_mode(r, s) == v


def test_sgd_and_mean(port):
    s = np.array([1.0, 3.0, -2.5, 7.0], np.float32)
    m = port.to_mean(s, 3)
    assert np.array_equal(u32(m), u32(s * np.float32(1.0 / 3.0)))
    w = words_from_bits(np.array([1, 0, 1, 1], bool))
    p = port.sgd_step(np.array([1, 2, 3, 4], np.float32), m, 0.1, w)
    exp = np.array([1, 2, 3, 4], np.float32) - np.float32(0.1) * m
    exp[1] = 0.0
    assert np.array_equal(u32(p), u32(exp))


def test_port_vs_reference_live(port, ref):
    rng = np.random.default_rng(7)
    for t in range(80):
        n = int(rng.integers(1, 4000))
        x = (rng.integers(-20, 21, n) * 0.5).astype(np.float32) if t % 2 else rng.standard_normal(n).astype(np.float32)
        r = float(np.float32(rng.choice([0.0, 0.25, 0.5, 0.9, 0.99])))
        assert np.array_equal(port.magnitude_prune(x, r), ref.magnitude_prune(x, r)[0])
    for n in (2, 3, 5, 8):
        xs = [rng.standard_normal(999).astype(np.float32) for _ in range(n)]
        a, _ = ref.ring_allreduce(xs)
        b = port.ring_allreduce(xs)
        assert all(np.array_equal(u32(p), u32(q)) for p, q in zip(a, b))
