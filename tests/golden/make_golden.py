"""Generate tests/golden/ fixtures by running the REFERENCE itself.

Every value here comes from oracle/_ref/libpactref.so, i.e. the reference's
own tensor/sparsity/codec/collective sources compiled in place (see
oracle/Makefile), driven through oracle/ref_shim.cpp. The reference's own
known-answer constants (test_*.cpp) are asserted while generating, so the
fixtures are pinned twice. Run from the repo root:

    python tests/golden/make_golden.py

Outputs: tests/golden/golden.json (scalars, small vectors) and
tests/golden/golden.npz (arrays).
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from oracle import words_from_bits  # noqa: E402


def main() -> None:
    R = oracle.ref()
    J: dict = {}
    A: dict = {}
    rng = np.random.default_rng(20250518)

    # --- digests (test_tensor.cpp:89-92, pact_main.cpp:43-49)
    nnz, dig = R.mask_info(words_from_bits(np.zeros(64, bool)), 64)
    assert dig == 0xA8C7F832281A39C5
    J["digest_all_zeros_64"] = dig
    _, J["digest_all_ones_11"] = R.mask_info(words_from_bits(np.ones(11, bool)), 11)
    _, J["digest_empty"] = R.mask_info(np.zeros(0, np.uint64), 0)
    dig_cases = []
    for t in range(40):
        n = int(rng.integers(1, 700))
        bits = rng.random(n) < rng.random()
        w = words_from_bits(bits)
        nnz, d = R.mask_info(w, n)
        dig_cases.append({"n": n, "nnz": nnz, "digest": d})
        A[f"dig_words_{t}"] = w
    J["digest_cases"] = dig_cases

    # --- prune known answers (test_sparsity.cpp:13-47)
    w, nnz, _ = R.magnitude_prune(np.array([0.1, -0.5, 0.3, 0.0], np.float32), 0.5)
    assert nnz == 2 and [(int(w[0]) >> i) & 1 for i in range(4)] == [0, 1, 1, 0]
    w, nnz, _ = R.magnitude_prune(np.array([0.5, -0.5, 0.5, 0.5], np.float32), 0.5)
    assert [(int(w[0]) >> i) & 1 for i in range(4)] == [0, 0, 1, 1]
    J["prune_examples"] = [
        {"w": [0.1, -0.5, 0.3, 0.0], "ratio": 0.5, "keep": [0, 1, 1, 0]},
        {"w": [0.5, -0.5, 0.5, 0.5], "ratio": 0.5, "keep": [0, 0, 1, 1]},
        {"w": [0.1, 0.2, 0.3], "ratio": 0.0, "keep": [1, 1, 1]},
    ]
    # random prune cases incl. heavy ties, +-0.0, ragged lengths
    pc = []
    for t in range(60):
        n = int(rng.integers(1, 5000))
        kind = t % 4
        if kind == 0:
            x = rng.standard_normal(n).astype(np.float32)
        elif kind == 1:  # heavy ties on a coarse grid, signed zeros
            x = (rng.integers(-8, 9, n) * 0.125).astype(np.float32)
            x[rng.random(n) < 0.1] = -0.0
        elif kind == 2:
            x = (rng.integers(-3, 4, n)).astype(np.float32)
        else:
            x = (rng.standard_normal(n) * np.exp2(rng.integers(-20, 5, n))).astype(np.float32)
        ratio = float(np.float32(rng.choice([0.0, 0.1, 0.3, 0.5, 0.7, 0.8, 0.9, 0.95, 0.99])))
        words, nnz, dig = R.magnitude_prune(x, ratio)
        pc.append({"n": n, "ratio": ratio, "nnz": nnz, "digest": dig})
        A[f"prune_w_{t}"] = x
        A[f"prune_words_{t}"] = words
    J["prune_cases"] = pc
    # sort-oracle property case (test_sparsity.cpp:49-69): 1000 gaussians @0.8 -> nnz 200
    x = rng.standard_normal(1000).astype(np.float32)
    words, nnz, _ = R.magnitude_prune(x, 0.8)
    assert nnz == 200

    # --- drop_count at the BASELINE config sizes
    dc = []
    for n, r in [(11689512, 0.9), (11700000, 0.9), (25557032, 0.8), (143667240, 0.95),
                 (109482240, 0.5), (109482240, 0.8), (109482240, 0.9), (109482240, 0.95),
                 (109482240, 0.99), (354823168, 0.9), (25600000, 0.8), (1000, 0.7)]:
        dc.append({"len": n, "ratio": r, "k": n - 0})  # filled below
    # k via the reference: prune an all-distinct ramp of that length is too big;
    # use the closed form the reference computes (sparsity.cpp:38-39) and pin
    # it against the survey's table values
    import math

    for e in dc:
        e["k"] = int(math.floor(float(np.float32(e["ratio"])) * e["len"] + e["len"] * 1e-7))
    table = {11689512: 10520561, 25557032: 20445628, 143667240: 136483890, 354823168: 319340878}
    for e in dc:
        if e["len"] in table and e["ratio"] in (0.9, 0.8, 0.95) and (e["len"], e["ratio"]) in (
                (11689512, 0.9), (25557032, 0.8), (143667240, 0.95), (354823168, 0.9)):
            assert e["k"] == table[e["len"]], e
    J["drop_counts"] = dc

    # --- pack / unpack (test_codec.cpp:31-94)
    cc = []
    for t in range(40):
        n = int(rng.integers(1, 3000))
        g = rng.standard_normal(n).astype(np.float32)
        g[rng.random(n) < 0.05] = -0.0
        bits = rng.random(n) < rng.random()
        words = words_from_bits(bits)
        packed, dig = R.pack(g, words, t)
        un = R.unpack(packed, dig, words, n)
        gse = R.gse(g, words)
        assert np.array_equal(un.view(np.uint32), gse.view(np.uint32))
        cc.append({"n": n, "count": int(packed.size), "digest": dig})
        A[f"codec_g_{t}"] = g
        A[f"codec_words_{t}"] = words
        A[f"codec_packed_{t}"] = packed
        A[f"codec_unpacked_{t}"] = un
    J["codec_cases"] = cc

    # --- header bytes (test_codec.cpp:247-274)
    hb = R.encode_header(1, 0x01020304, 0x1122334455667788, 5)
    assert hb[:4] == b"PACT" and hb[4] == 1 and hb[5] == 1 and hb[6] == 0x04 and hb[10] == 0x88
    J["header_packed"] = hb.hex()
    J["header_full"] = R.encode_header(0, 7, 0xDEADBEEFCAFEF00D, 123456789).hex()

    # --- ring allreduce fold order (test_collective.cpp:46-99)
    rc = []
    for n in (2, 3, 4, 8):
        for ln in (1, 3, 37, 4096):
            xs = [(rng.standard_normal(ln) * np.exp2(rng.integers(-10, 10, ln))).astype(np.float32) for _ in range(n)]
            outs, byts = R.ring_allreduce(xs)
            for o in outs[1:]:
                assert np.array_equal(o.view(np.uint32), outs[0].view(np.uint32))
            key = f"ring_{n}_{ln}"
            A[key + "_in"] = np.stack(xs)
            A[key + "_out"] = outs[0]
            rc.append({"n": n, "len": ln, "bytes": byts})
    outs, _ = R.ring_allreduce([np.array([1e8], np.float32), np.array([-1e8], np.float32), np.array([1.0], np.float32)])
    J["ring_fold_probe_n3"] = [float(outs[0][0])]
    J["ring_cases"] = rc

    # --- masked allreduce (test_collective.cpp:210-285, acceptance 5/10)
    mc = []

    def masked_case(name, grads, masks, stable, epoch, advertised=None):
        outs, modes, byts = R.masked_allreduce(grads, masks, stable, epoch, advertised)
        A[f"masked_{name}_grads"] = np.stack(grads)
        A[f"masked_{name}_masks"] = np.stack(masks)
        A[f"masked_{name}_outs"] = np.stack(outs)
        mc.append({"name": name, "n": len(grads), "len": int(grads[0].size), "stable": list(map(int, stable)),
                   "epoch": epoch, "advertised": advertised, "modes": modes, "bytes": byts})

    ln = 5000
    bits = rng.random(ln) < 0.3
    mw = words_from_bits(bits)
    for n in (2, 3, 4):
        gs = [np.where(bits, rng.standard_normal(ln), 0).astype(np.float32) for _ in range(n)]
        masked_case(f"stable_n{n}", gs, [mw] * n, [1] * n, 3)
        masked_case(f"unstable_n{n}", gs, [mw] * n, [1] * (n - 1) + [0], 3)
    gs = [rng.standard_normal(ln).astype(np.float32) for _ in range(4)]
    bad = bits.copy()
    bad[6] = not bad[6]
    masked_case("divergent_n4", gs, [mw, mw, words_from_bits(bad), mw], [1] * 4, 7)
    _, d0 = R.mask_info(mw, ln)
    masked_case("fault_n3", gs[:3], [mw] * 3, [1] * 3, 2, [d0, d0 ^ 0x5A5A5A5A5A5A5A5A, d0])
    J["masked_cases"] = mc

    # acceptance 5 byte proportionality at 1e6 (acceptance_main.cpp:249-276)
    ln = 1_000_000
    a5 = []
    for ratio in (0.5, 0.8, 0.9):
        x = rng.standard_normal(ln).astype(np.float32)
        words, nnz, _ = R.magnitude_prune(x, ratio)
        gs = [R.gse(rng.standard_normal(ln).astype(np.float32), words) for _ in range(2)]
        _, _, pb = R.masked_allreduce(gs, [words, words], [1, 1], 0)
        _, fb = R.full_allreduce(gs)
        a5.append({"ratio": ratio, "nnz": nnz, "packed_bytes": pb[0], "full_bytes": fb[0],
                   "ratio_bytes": pb[0] / fb[0]})
    J["acceptance5"] = a5

    # tracker sequences (test_sparsity.cpp:204-236)
    masks = [words_from_bits(rng.random(32) < 0.5) for _ in range(4)]
    seq = [int(s) for s in rng.integers(0, 4, 40)]
    J["tracker_seq"] = {"K": 3, "seq": seq, "status": R.tracker_sequence(3, masks, [32] * 4, seq)}
    for i, m in enumerate(masks):
        A[f"tracker_mask_{i}"] = m
    J["tracker_repeat"] = R.tracker_sequence(3, masks[:1], [32], [0, 0, 0, 0, 0])
    J["decide_sync_mode"] = {f"{r}_{s}": R.decide_sync_mode(r, s) for r in range(5) for s in (0, 1)}

    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(J, f, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **A)
    print("wrote", len(J), "json keys,", len(A), "arrays")


if __name__ == "__main__":
    main()
