"""CPU tests of the product library: it loads without a GPU, exports every
symbol include/pact_c.h declares, and its host-side scalar logic (drop count,
wire header, tracker, vote rule, byte accounting) matches the oracle and the
reference fixtures. No compute kernel is called here."""
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "pact_c.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pact_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(pb):
    from paper_2505_18563_b200 import _lib

    syms = declared_symbols()
    assert len(syms) >= 35
    for s in syms:
        assert hasattr(_lib.lib, s), s
        assert s in _lib.SIGNATURES, f"{s} not bound in _lib.SIGNATURES"


def test_library_is_sm100a(pb):
    import subprocess

    from paper_2505_18563_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_abi_version_and_status_names(pb):
    from paper_2505_18563_b200._lib import lib

    assert lib.pact_abi_version() == 1
    assert lib.pact_status_name(3) == b"InvalidRatio"
    assert lib.pact_status_name(7) == b"MaskMismatch"
    assert lib.pact_status_name(14) == b"BadTopology"


def test_drop_count_matches_oracle(pb, port, golden):
    j, _ = golden
    for e in j["drop_counts"]:
        assert pb.drop_count(e["ratio"], e["len"]) == e["k"]
    rng = np.random.default_rng(3)
    for _ in range(2000):
        n = int(rng.integers(0, 1 << 30))
        r = float(np.float32(rng.random()))
        assert pb.drop_count(r, n) == port.drop_count(r, n)
    for r in (1.0, -0.1, float("nan")):
        with pytest.raises(pb.Error) as e:
            pb.drop_count(r, 10)
        assert e.value.code == pb.Errc.InvalidRatio


def test_header_roundtrip_and_errors(pb, golden):
    j, _ = golden
    h = pb.FrameHeader(pb.PayloadKind.Packed, 0x01020304, 0x1122334455667788, 5)
    b = pb.encode_header(h)
    assert b.hex() == j["header_packed"]
    assert pb.decode_header(b) == h
    assert pb.encode_header(pb.FrameHeader(pb.PayloadKind.Full, 7, 0xDEADBEEFCAFEF00D, 123456789)).hex() == j["header_full"]
    for bad in (b[:25], b"XACT" + b[4:], b[:4] + b"\x02" + b[5:], b[:5] + b"\x05" + b[6:]):
        with pytest.raises(pb.Error) as e:
            pb.decode_header(bad)
        assert e.value.code == pb.Errc.CorruptPayload


def test_tracker_matches_reference_sequence(pb, port, golden):
    j, a = golden
    masks = [a[f"tracker_mask_{i}"] for i in range(4)]
    digests = [port.mask_digest(m, 32) for m in masks]
    t = pb.MaskTracker(j["tracker_seq"]["K"])
    got = [int(t.observe_digest(digests[s]) == pb.TrackerStatus.Stable) for s in j["tracker_seq"]["seq"]]
    assert got == j["tracker_seq"]["status"]
    t = pb.MaskTracker(3)
    assert [t.observe_digest(5) == pb.TrackerStatus.Stable for _ in range(5)] == [False, False, False, True, True]
    t = pb.MaskTracker(0)  # 0 promoted to 1 (sparsity.hpp:41)
    assert [t.observe_digest(1) == pb.TrackerStatus.Stable for _ in range(2)] == [False, True]
    t = pb.MaskTracker(2)
    for _ in range(10):  # alternating digests never stabilise (test_sparsity.cpp:214-222)
        assert t.observe_digest(1) == pb.TrackerStatus.Unstable
        assert t.observe_digest(2) == pb.TrackerStatus.Unstable


def test_decide_sync_mode(pb, golden):
    j, _ = golden
    for k, v in j["decide_sync_mode"].items():
        r, s = map(int, k.split("_"))
        st = pb.TrackerStatus.Stable if s else pb.TrackerStatus.Unstable
        assert int(pb.decide_sync_mode(pb.SyncMode(r), st)) == v


def test_vote_rule(pb):
    mine = pb.FrameHeader(pb.PayloadKind.Packed, 3, 0xABC, 100)
    f = pb.encode_header(mine)
    assert pb.vote_decide([f, f, f], mine, True)
    assert not pb.vote_decide([f, f, f], mine, False)  # own tracker unstable
    other = pb.encode_header(pb.FrameHeader(pb.PayloadKind.Full, 3, 0xABC, 100))
    assert not pb.vote_decide([f, other, f], mine, True)
    assert not pb.vote_decide([f, pb.encode_header(pb.FrameHeader(pb.PayloadKind.Packed, 3, 0xABD, 100))], mine, True)
    assert not pb.vote_decide([f, pb.encode_header(pb.FrameHeader(pb.PayloadKind.Packed, 3, 0xABC, 99))], mine, True)
    # epoch is not part of the rule (collective.cpp:288-289)
    assert pb.vote_decide([f, pb.encode_header(pb.FrameHeader(pb.PayloadKind.Packed, 9, 0xABC, 100))], mine, True)
    with pytest.raises(pb.Error):
        pb.vote_decide([f, b"PACX" + f[4:]], mine, True)


def test_byte_accounting_matches_reference(pb, port, golden):
    j, _ = golden
    for c in j["ring_cases"]:
        assert [pb.ring_bytes(c["n"], p, c["len"]) for p in range(c["n"])] == c["bytes"]
    for c in j["masked_cases"]:
        n = c["n"]
        count = c["len"]
        if c["modes"][0]:
            count = int(port.mask_nnz(golden[1][f"masked_{c['name']}_masks"][0], c["len"]))
        assert [pb.masked_bytes(n, p, count) for p in range(n)] == c["bytes"]
    for c in j["acceptance5"]:
        assert pb.masked_bytes(2, 0, c["nnz"]) == c["packed_bytes"]
        assert pb.ring_bytes(2, 0, 1_000_000) == c["full_bytes"]
    rng = np.random.default_rng(5)
    for _ in range(300):
        n = int(rng.integers(2, 9))
        cnt = int(rng.integers(0, 100000))
        p = int(rng.integers(0, n))
        assert pb.ring_bytes(n, p, cnt) == port.ring_bytes(n, p, cnt)


def test_no_gpu_means_loud_failure(pb):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(pb.Error) as e:
        pb.Context(0)
    assert e.value.status == 103  # PACT_E_NO_DEVICE: no silent CPU path
