"""ctypes front-end for the two oracle libraries (TEST INFRASTRUCTURE ONLY)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from functools import lru_cache

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_port", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libpactref.so")

_f32p = C.POINTER(C.c_float)
_u64p = C.POINTER(C.c_uint64)
_u8p = C.POINTER(C.c_uint8)


def build(force: bool = False) -> None:
    """Compile the oracle libraries (port always; ref when /root/reference exists)."""
    if force or not os.path.exists(PORT_SO) or (
        os.path.isdir("/root/reference/proj") and not os.path.exists(REF_SO)
    ):
        subprocess.run(["make", "-s", "-C", HERE], check=True)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def _f(a: np.ndarray):
    return a.ctypes.data_as(_f32p)


def _u(a: np.ndarray):
    return a.ctypes.data_as(_u64p)


def _ptr_array(arrs, ctype):
    arr_t = C.POINTER(ctype) * len(arrs)
    return arr_t(*[a.ctypes.data_as(C.POINTER(ctype)) for a in arrs])


def word_count(n: int) -> int:
    return (n + 63) // 64


def words_from_bits(keep) -> np.ndarray:
    """Reference word layout (tensor.hpp:93): bit i at words[i>>6] bit (i&63)."""
    keep = np.asarray(keep, dtype=bool)
    n = keep.size
    padded = np.zeros(word_count(n) * 64, dtype=bool)
    padded[:n] = keep
    return np.packbits(padded.reshape(-1, 8), axis=1, bitorder="little").reshape(-1).view(np.uint64).copy()


def bits_from_words(words: np.ndarray, n: int) -> np.ndarray:
    b = np.unpackbits(np.ascontiguousarray(words).view(np.uint8), bitorder="little")
    return b[:n].astype(bool)


class OracleError(Exception):
    def __init__(self, code: int):
        super().__init__(f"oracle status {code}")
        self.code = code


def _check(st: int):
    if st:
        raise OracleError(st)


class Port:
    """The C restatement (oracle/pact_oracle.c)."""

    def __init__(self):
        L = C.CDLL(PORT_SO)
        self.L = L
        L.orc_splitmix64.restype = C.c_uint64
        L.orc_splitmix64.argtypes = [C.c_uint64]
        L.orc_derive_seed.restype = C.c_uint64
        L.orc_derive_seed.argtypes = [C.c_uint64] * 4
        L.orc_fnv1a64.restype = C.c_uint64
        L.orc_fnv1a64.argtypes = [C.c_void_p, C.c_size_t]
        L.orc_mask_nnz.restype = C.c_uint64
        L.orc_mask_nnz.argtypes = [_u64p, C.c_size_t]
        L.orc_mask_digest.restype = C.c_uint64
        L.orc_mask_digest.argtypes = [_u64p, C.c_size_t]
        L.orc_drop_count.argtypes = [C.c_float, C.c_uint64, _u64p]
        L.orc_magnitude_prune.argtypes = [_f32p, C.c_size_t, C.c_float, _u64p]
        L.orc_magnitude_prune_segmented.argtypes = [_f32p, C.c_size_t, _u64p, C.c_size_t, C.c_float, _u64p]
        L.orc_prune_threshold.argtypes = [_f32p, C.c_size_t, C.c_uint64, C.POINTER(C.c_uint32), _u64p]
        L.orc_gse.argtypes = [_f32p, _u64p, C.c_size_t, _f32p]
        L.orc_pack.argtypes = [_f32p, _u64p, C.c_size_t, _f32p, _u64p]
        L.orc_unpack.argtypes = [_f32p, C.c_uint64, C.c_uint64, _u64p, C.c_size_t, _f32p]
        L.orc_ring_allreduce.argtypes = [C.c_int, C.c_void_p, C.c_size_t, C.c_void_p]
        L.orc_ring_bytes.restype = C.c_uint64
        L.orc_ring_bytes.argtypes = [C.c_int, C.c_int, C.c_uint64]
        L.orc_masked_allreduce.argtypes = [
            C.c_int, C.c_void_p, C.c_void_p, _u64p, C.c_void_p, C.POINTER(C.c_int),
            C.c_uint32, C.c_size_t, C.c_void_p, C.POINTER(C.c_int), _u64p,
        ]
        L.orc_decide_sync_mode.argtypes = [C.c_int, C.c_int]
        L.orc_to_mean.argtypes = [_f32p, C.c_size_t, C.c_int, _f32p]
        L.orc_sgd_step.argtypes = [_f32p, _f32p, C.c_size_t, C.c_float, C.c_void_p]
        L.orc_encode_header.argtypes = [C.c_void_p, _u8p]
        L.orc_decode_header.argtypes = [_u8p, C.c_size_t, C.c_void_p]
        L.orc_topk_select.argtypes = [_f32p, C.c_size_t, C.c_float, C.POINTER(C.c_uint32), _f32p, _u64p]
        L.orc_topk_mean.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_size_t, _f32p]
        L.orc_float_to_half.argtypes = [_f32p, C.c_size_t, C.POINTER(C.c_uint16)]
        L.orc_half_to_float.argtypes = [C.POINTER(C.c_uint16), C.c_size_t, _f32p]
        L.orc_ring_allreduce_fp16.argtypes = [C.c_int, C.c_void_p, C.c_size_t, C.c_void_p]
        L.orc_ternarize_ctr.argtypes = [_f32p, C.c_size_t, C.c_uint64, C.POINTER(C.c_float), _u8p]
        L.orc_ternary_check.argtypes = [C.c_float, _u8p, C.c_size_t]
        L.orc_ternary_mean.argtypes = [C.c_int, _f32p, C.c_void_p, C.c_size_t, _f32p]

    # -- scalar / mask helpers
    def splitmix64(self, x: int) -> int:
        return self.L.orc_splitmix64(x)

    def derive_seed(self, base, a, b=0, c=0) -> int:
        return self.L.orc_derive_seed(base, a, b, c)

    def fnv1a64(self, data: bytes) -> int:
        buf = C.create_string_buffer(data, len(data))
        return self.L.orc_fnv1a64(buf, len(data))

    def mask_nnz(self, words, n) -> int:
        words = np.ascontiguousarray(words, dtype=np.uint64)
        return self.L.orc_mask_nnz(_u(words), n)

    def mask_digest(self, words, n) -> int:
        words = np.ascontiguousarray(words, dtype=np.uint64)
        return self.L.orc_mask_digest(_u(words), n)

    def drop_count(self, ratio: float, n: int) -> int:
        k = C.c_uint64()
        _check(self.L.orc_drop_count(ratio, n, C.byref(k)))
        return k.value

    def magnitude_prune(self, w: np.ndarray, ratio: float) -> np.ndarray:
        w = np.ascontiguousarray(w, dtype=np.float32)
        words = np.zeros(max(1, word_count(w.size)), dtype=np.uint64)
        _check(self.L.orc_magnitude_prune(_f(w), w.size, ratio, _u(words)))
        return words[: word_count(w.size)]

    def magnitude_prune_segmented(self, w, seg_offsets, ratio) -> np.ndarray:
        w = np.ascontiguousarray(w, dtype=np.float32)
        seg = np.ascontiguousarray(seg_offsets, dtype=np.uint64)
        words = np.zeros(max(1, word_count(w.size)), dtype=np.uint64)
        _check(self.L.orc_magnitude_prune_segmented(_f(w), w.size, _u(seg), seg.size - 1, ratio, _u(words)))
        return words[: word_count(w.size)]

    def prune_threshold(self, w, k):
        w = np.ascontiguousarray(w, dtype=np.float32)
        T = C.c_uint32()
        c = C.c_uint64()
        _check(self.L.orc_prune_threshold(_f(w), w.size, k, C.byref(T), C.byref(c)))
        return T.value, c.value

    def gse(self, g, words):
        g = np.ascontiguousarray(g, dtype=np.float32)
        words = np.ascontiguousarray(words, dtype=np.uint64)
        out = np.empty_like(g)
        _check(self.L.orc_gse(_f(g), _u(words), g.size, _f(out)))
        return out

    def pack(self, g, words):
        g = np.ascontiguousarray(g, dtype=np.float32)
        words = np.ascontiguousarray(words, dtype=np.uint64)
        out = np.empty(max(1, g.size), dtype=np.float32)
        cnt = C.c_uint64()
        _check(self.L.orc_pack(_f(g), _u(words), g.size, _f(out), C.byref(cnt)))
        return out[: cnt.value].copy()

    def unpack(self, packed, digest, words, n):
        packed = np.ascontiguousarray(packed, dtype=np.float32)
        words = np.ascontiguousarray(words, dtype=np.uint64)
        out = np.empty(max(1, n), dtype=np.float32)
        _check(self.L.orc_unpack(_f(packed), packed.size, digest, _u(words), n, _f(out)))
        return out[:n]

    def ring_allreduce(self, inputs):
        inputs = [np.ascontiguousarray(x, dtype=np.float32) for x in inputs]
        outs = [np.empty_like(inputs[0]) for _ in inputs]
        self.L.orc_ring_allreduce(
            len(inputs), C.cast(_ptr_array(inputs, C.c_float), C.c_void_p), inputs[0].size,
            C.cast(_ptr_array(outs, C.c_float), C.c_void_p),
        )
        return outs

    def ring_bytes(self, n, position, count) -> int:
        return self.L.orc_ring_bytes(n, position, count)

    def masked_allreduce(self, grads, masks, stable, epoch, advertised=None):
        n = len(grads)
        ln = grads[0].size
        grads = [np.ascontiguousarray(x, dtype=np.float32) for x in grads]
        masks = [np.ascontiguousarray(m, dtype=np.uint64) for m in masks]
        digests = np.array([self.mask_digest(m, ln) for m in masks], dtype=np.uint64)
        adv = None if advertised is None else np.array(advertised, dtype=np.uint64)
        outs = [np.empty_like(grads[0]) for _ in range(n)]
        st = (C.c_int * n)(*[int(bool(s)) for s in stable])
        modes = (C.c_int * n)()
        byts = np.zeros(n, dtype=np.uint64)
        _check(self.L.orc_masked_allreduce(
            n, C.cast(_ptr_array(grads, C.c_float), C.c_void_p),
            C.cast(_ptr_array(masks, C.c_uint64), C.c_void_p), _u(digests),
            None if adv is None else C.cast(_u(adv), C.c_void_p), st, epoch, ln,
            C.cast(_ptr_array(outs, C.c_float), C.c_void_p), modes, _u(byts),
        ))
        return outs, list(modes), [int(b) for b in byts]

    def decide_sync_mode(self, requested: int, stable: bool) -> int:
        return self.L.orc_decide_sync_mode(requested, int(bool(stable)))

    def to_mean(self, s, n):
        s = np.ascontiguousarray(s, dtype=np.float32)
        out = np.empty_like(s)
        self.L.orc_to_mean(_f(s), s.size, n, _f(out))
        return out

    def sgd_step(self, params, mean_grad, lr, words=None):
        p = np.ascontiguousarray(params, dtype=np.float32).copy()
        g = np.ascontiguousarray(mean_grad, dtype=np.float32)
        w = None if words is None else np.ascontiguousarray(words, dtype=np.uint64)
        self.L.orc_sgd_step(_f(p), _f(g), p.size, lr, None if w is None else C.cast(_u(w), C.c_void_p))
        return p

    # -- TopK
    def topk_select(self, g, rate):
        g = np.ascontiguousarray(g, dtype=np.float32)
        idx = np.empty(max(1, g.size), dtype=np.uint32)
        val = np.empty(max(1, g.size), dtype=np.float32)
        k = C.c_uint64()
        _check(self.L.orc_topk_select(_f(g), g.size, rate, idx.ctypes.data_as(C.POINTER(C.c_uint32)), _f(val),
                                      C.byref(k)))
        return idx[: k.value].copy(), val[: k.value].copy()

    def topk_mean(self, idxs, vals, length):
        n = len(idxs)
        idxs = [np.ascontiguousarray(i if i.size else np.zeros(1, np.uint32), dtype=np.uint32) for i in idxs]
        vals = [np.ascontiguousarray(v if v.size else np.zeros(1, np.float32), dtype=np.float32) for v in vals]
        k = min(i.size for i in idxs)
        out = np.empty(max(1, length), dtype=np.float32)
        _check(self.L.orc_topk_mean(n, C.cast(_ptr_array(idxs, C.c_uint32), C.c_void_p),
                                    C.cast(_ptr_array(vals, C.c_float), C.c_void_p), k, length, _f(out)))
        return out[:length]

    # -- binary16 wire
    def float_to_half(self, x):
        x = np.ascontiguousarray(x, dtype=np.float32)
        out = np.empty(max(1, x.size), dtype=np.uint16)
        self.L.orc_float_to_half(_f(x), x.size, out.ctypes.data_as(C.POINTER(C.c_uint16)))
        return out[: x.size]

    def half_to_float(self, h):
        h = np.ascontiguousarray(h, dtype=np.uint16)
        out = np.empty(max(1, h.size), dtype=np.float32)
        self.L.orc_half_to_float(h.ctypes.data_as(C.POINTER(C.c_uint16)), h.size, _f(out))
        return out[: h.size]

    def ring_allreduce_fp16(self, inputs):
        inputs = [np.ascontiguousarray(x, dtype=np.float32) for x in inputs]
        outs = [np.empty_like(inputs[0]) for _ in inputs]
        self.L.orc_ring_allreduce_fp16(
            len(inputs), C.cast(_ptr_array(inputs, C.c_float), C.c_void_p), inputs[0].size,
            C.cast(_ptr_array(outs, C.c_float), C.c_void_p))
        return outs

    # -- ternary
    def ternarize(self, v, seed):
        v = np.ascontiguousarray(v, dtype=np.float32)
        sc = C.c_float()
        b = np.zeros(max(1, (v.size + 3) // 4), dtype=np.uint8)
        self.L.orc_ternarize_ctr(_f(v), v.size, seed & 0xFFFFFFFFFFFFFFFF, C.byref(sc),
                                 b.ctypes.data_as(_u8p))
        return sc.value, b[: (v.size + 3) // 4].copy()

    def ternary_mean(self, scales, sign_bytes, count):
        n = len(scales)
        sc = np.ascontiguousarray(scales, dtype=np.float32)
        bs = [np.ascontiguousarray(b if len(b) else np.zeros(1, np.uint8), dtype=np.uint8) for b in sign_bytes]
        out = np.empty(max(1, count), dtype=np.float32)
        _check(self.L.orc_ternary_mean(n, _f(sc), C.cast(_ptr_array(bs, C.c_uint8), C.c_void_p), count, _f(out)))
        return out[:count]

    def encode_header(self, kind, epoch, digest, count) -> bytes:
        class H(C.Structure):
            _fields_ = [("kind", C.c_uint8), ("epoch", C.c_uint32), ("mask_digest", C.c_uint64),
                        ("value_count", C.c_uint64)]
        h = H(kind, epoch, digest, count)
        out = (C.c_uint8 * 26)()
        self.L.orc_encode_header(C.byref(h), out)
        return bytes(out)


class Ref:
    """The reference's own code (oracle/_ref/libpactref.so)."""

    def __init__(self):
        L = C.CDLL(REF_SO)
        self.L = L
        L.ref_magnitude_prune.argtypes = [_f32p, C.c_size_t, C.c_float, _u64p, _u64p, _u64p]
        L.ref_mask_from_words.argtypes = [_u64p, C.c_size_t, _u64p, _u64p]
        L.ref_gse.argtypes = [_f32p, _u64p, C.c_size_t, C.c_size_t, _f32p]
        L.ref_pack.argtypes = [_f32p, _u64p, C.c_size_t, C.c_size_t, C.c_uint32, _f32p, _u64p, _u64p]
        L.ref_unpack.argtypes = [_f32p, C.c_uint64, C.c_uint64, _u64p, C.c_size_t, _f32p]
        L.ref_encode_header.argtypes = [C.c_uint8, C.c_uint32, C.c_uint64, C.c_uint64, _u8p]
        L.ref_decode_header.argtypes = [_u8p, C.c_size_t, _u8p, C.POINTER(C.c_uint32), _u64p, _u64p]
        L.ref_tracker_sequence.argtypes = [C.c_uint32, C.c_void_p, C.c_void_p, C.POINTER(C.c_int),
                                           C.c_size_t, C.POINTER(C.c_int)]
        L.ref_decide_sync_mode.argtypes = [C.c_int, C.c_int]
        L.ref_ring_allreduce.argtypes = [C.c_int, C.c_void_p, C.c_size_t, C.c_void_p, _u64p]
        L.ref_full_allreduce.argtypes = [C.c_int, C.c_void_p, C.c_size_t, C.c_void_p, _u64p]
        L.ref_masked_allreduce.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_int),
                                           C.c_void_p, C.c_uint32, C.c_size_t, C.c_void_p,
                                           C.POINTER(C.c_int), _u64p]
        L.ref_topk_select.argtypes = [_f32p, C.c_size_t, C.c_float, C.POINTER(C.c_uint32), _f32p, _u64p]
        L.ref_topk_densify.argtypes = [C.POINTER(C.c_uint32), _f32p, C.c_size_t, C.c_size_t, _f32p]
        L.ref_topk_decode_check.argtypes = [_u8p, C.c_size_t, C.c_size_t, _u64p]
        L.ref_topk_aggregate.argtypes = [C.c_int, C.c_void_p, C.c_size_t, C.c_float, C.c_uint32, C.c_void_p,
                                         _u64p]
        L.ref_float_to_half.argtypes = [_f32p, C.c_size_t, C.POINTER(C.c_uint16)]
        L.ref_half_to_float.argtypes = [C.POINTER(C.c_uint16), C.c_size_t, _f32p]
        L.ref_fp16_allreduce.argtypes = [C.c_int, C.c_void_p, C.c_size_t, C.c_void_p, _u64p]
        L.ref_ternarize.argtypes = [_f32p, C.c_size_t, C.c_uint64, C.POINTER(C.c_float), _u8p]
        L.ref_deternarize.argtypes = [C.c_float, _u8p, C.c_size_t, _f32p]
        L.ref_decode_ternary.argtypes = [_u8p, C.c_size_t, C.POINTER(C.c_float), _u64p, _u64p, _u8p]
        L.ref_encode_ternary.argtypes = [C.c_float, _u8p, C.c_size_t, C.c_uint32, C.c_uint64, _u8p,
                                         C.POINTER(C.c_size_t)]
        L.ref_ternary_aggregate.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_int), _u64p,
                                            C.c_uint32, C.c_size_t, C.c_void_p, C.POINTER(C.c_int), _u64p]
        L.ref_bench_create.restype = C.c_void_p
        L.ref_bench_create.argtypes = [C.c_int, C.c_void_p, _u64p, C.c_size_t, C.c_int]
        L.ref_bench_destroy.argtypes = [C.c_void_p]
        L.ref_bench_masked.restype = C.c_double
        L.ref_bench_masked.argtypes = [C.c_void_p, C.c_uint32]
        L.ref_bench_pack_unpack.restype = C.c_double
        L.ref_bench_pack_unpack.argtypes = [C.c_void_p, C.c_uint32]
        L.ref_bench_prune.restype = C.c_double
        L.ref_bench_prune.argtypes = [_f32p, C.c_size_t, C.c_float]

    def magnitude_prune(self, w, ratio):
        w = np.ascontiguousarray(w, dtype=np.float32)
        words = np.zeros(max(1, word_count(w.size)), dtype=np.uint64)
        nnz = C.c_uint64()
        dig = C.c_uint64()
        _check(self.L.ref_magnitude_prune(_f(w), w.size, ratio, _u(words), C.byref(nnz), C.byref(dig)))
        return words[: word_count(w.size)], nnz.value, dig.value

    def mask_info(self, words, n):
        words = np.ascontiguousarray(words, dtype=np.uint64)
        if words.size == 0:
            words = np.zeros(1, dtype=np.uint64)
        nnz = C.c_uint64()
        dig = C.c_uint64()
        _check(self.L.ref_mask_from_words(_u(words), n, C.byref(nnz), C.byref(dig)))
        return nnz.value, dig.value

    def gse(self, g, words, mask_len=None):
        g = np.ascontiguousarray(g, dtype=np.float32)
        words = np.ascontiguousarray(words, dtype=np.uint64)
        out = np.empty(max(1, g.size), dtype=np.float32)
        _check(self.L.ref_gse(_f(g), _u(words), g.size, g.size if mask_len is None else mask_len, _f(out)))
        return out[: g.size]

    def pack(self, g, words, epoch=0, mask_len=None):
        g = np.ascontiguousarray(g, dtype=np.float32)
        words = np.ascontiguousarray(words, dtype=np.uint64)
        out = np.empty(max(1, g.size), dtype=np.float32)
        cnt = C.c_uint64()
        dig = C.c_uint64()
        _check(self.L.ref_pack(_f(g), _u(words), g.size, g.size if mask_len is None else mask_len,
                               epoch, _f(out), C.byref(cnt), C.byref(dig)))
        return out[: cnt.value].copy(), dig.value

    def unpack(self, packed, digest, words, n):
        packed = np.ascontiguousarray(packed, dtype=np.float32)
        if packed.size == 0:
            packed_buf = np.zeros(1, dtype=np.float32)
        else:
            packed_buf = packed
        words = np.ascontiguousarray(words, dtype=np.uint64)
        out = np.empty(max(1, n), dtype=np.float32)
        _check(self.L.ref_unpack(_f(packed_buf), packed.size, digest, _u(words), n, _f(out)))
        return out[:n]

    def encode_header(self, kind, epoch, digest, count) -> bytes:
        out = (C.c_uint8 * 26)()
        _check(self.L.ref_encode_header(kind, epoch, digest, count, out))
        return bytes(out)

    def decode_header(self, frame: bytes):
        buf = (C.c_uint8 * max(1, len(frame))).from_buffer_copy(frame + b"\0" * (1 - min(1, len(frame))))
        kind = C.c_uint8()
        ep = C.c_uint32()
        dig = C.c_uint64()
        cnt = C.c_uint64()
        _check(self.L.ref_decode_header(buf, len(frame), C.byref(kind), C.byref(ep), C.byref(dig), C.byref(cnt)))
        return kind.value, ep.value, dig.value, cnt.value

    def tracker_sequence(self, threshold, masks, lens, seq):
        masks = [np.ascontiguousarray(m, dtype=np.uint64) for m in masks]
        lens_a = np.array(lens, dtype=np.uint64)
        seq_a = (C.c_int * len(seq))(*seq)
        out = (C.c_int * len(seq))()
        _check(self.L.ref_tracker_sequence(threshold, C.cast(_ptr_array(masks, C.c_uint64), C.c_void_p),
                                           C.cast(_u(lens_a), C.c_void_p), seq_a, len(seq), out))
        return list(out)

    def decide_sync_mode(self, requested, stable):
        return self.L.ref_decide_sync_mode(requested, int(bool(stable)))

    def _coll(self, fn, inputs):
        inputs = [np.ascontiguousarray(x, dtype=np.float32) for x in inputs]
        outs = [np.empty_like(inputs[0]) for _ in inputs]
        byts = np.zeros(len(inputs), dtype=np.uint64)
        _check(fn(len(inputs), C.cast(_ptr_array(inputs, C.c_float), C.c_void_p), inputs[0].size,
                  C.cast(_ptr_array(outs, C.c_float), C.c_void_p), _u(byts)))
        return outs, [int(b) for b in byts]

    def ring_allreduce(self, inputs):
        return self._coll(self.L.ref_ring_allreduce, inputs)

    def full_allreduce(self, inputs):
        return self._coll(self.L.ref_full_allreduce, inputs)

    def masked_allreduce(self, grads, masks, stable, epoch, advertised=None):
        n = len(grads)
        ln = grads[0].size
        grads = [np.ascontiguousarray(x, dtype=np.float32) for x in grads]
        masks = [np.ascontiguousarray(m, dtype=np.uint64) for m in masks]
        adv = None if advertised is None else np.array(advertised, dtype=np.uint64)
        outs = [np.empty_like(grads[0]) for _ in range(n)]
        st = (C.c_int * n)(*[int(bool(s)) for s in stable])
        modes = (C.c_int * n)()
        byts = np.zeros(n, dtype=np.uint64)
        _check(self.L.ref_masked_allreduce(
            n, C.cast(_ptr_array(grads, C.c_float), C.c_void_p),
            C.cast(_ptr_array(masks, C.c_uint64), C.c_void_p), st,
            None if adv is None else C.cast(_u(adv), C.c_void_p), epoch, ln,
            C.cast(_ptr_array(outs, C.c_float), C.c_void_p), modes, _u(byts)))
        return outs, list(modes), [int(b) for b in byts]

    # -- TopK
    def topk_select(self, g, rate):
        g = np.ascontiguousarray(g, dtype=np.float32)
        idx = np.empty(max(1, g.size), dtype=np.uint32)
        val = np.empty(max(1, g.size), dtype=np.float32)
        k = C.c_uint64()
        _check(self.L.ref_topk_select(_f(g), g.size, rate, idx.ctypes.data_as(C.POINTER(C.c_uint32)), _f(val),
                                      C.byref(k)))
        return idx[: k.value].copy(), val[: k.value].copy()

    def topk_densify(self, idx, val, length):
        idx = np.ascontiguousarray(idx if len(idx) else np.zeros(1, np.uint32), dtype=np.uint32)
        val = np.ascontiguousarray(val if len(val) else np.zeros(1, np.float32), dtype=np.float32)
        out = np.empty(max(1, length), dtype=np.float32)
        _check(self.L.ref_topk_densify(idx.ctypes.data_as(C.POINTER(C.c_uint32)), _f(val), len(idx), length,
                                       _f(out)))
        return out[:length]

    def topk_decode_ok(self, frame: bytes, original_len: int) -> bool:
        buf = (C.c_uint8 * max(1, len(frame))).from_buffer_copy(frame or b"\0")
        k = C.c_uint64()
        return self.L.ref_topk_decode_check(buf, len(frame), original_len, C.byref(k)) == 0

    def topk_aggregate(self, grads, rate, epoch=0):
        grads = [np.ascontiguousarray(x, dtype=np.float32) for x in grads]
        outs = [np.empty_like(grads[0]) for _ in grads]
        byts = np.zeros(len(grads), dtype=np.uint64)
        _check(self.L.ref_topk_aggregate(len(grads), C.cast(_ptr_array(grads, C.c_float), C.c_void_p),
                                         grads[0].size, rate, epoch, C.cast(_ptr_array(outs, C.c_float), C.c_void_p),
                                         _u(byts)))
        return outs, [int(b) for b in byts]

    # -- binary16
    def float_to_half(self, x):
        x = np.ascontiguousarray(x, dtype=np.float32)
        out = np.empty(max(1, x.size), dtype=np.uint16)
        self.L.ref_float_to_half(_f(x), x.size, out.ctypes.data_as(C.POINTER(C.c_uint16)))
        return out[: x.size]

    def half_to_float(self, h):
        h = np.ascontiguousarray(h, dtype=np.uint16)
        out = np.empty(max(1, h.size), dtype=np.float32)
        self.L.ref_half_to_float(h.ctypes.data_as(C.POINTER(C.c_uint16)), h.size, _f(out))
        return out[: h.size]

    def fp16_allreduce(self, inputs):
        return self._coll(self.L.ref_fp16_allreduce, inputs)

    # -- ternary: the reference's own mt19937_64 ternarize
    def ternarize(self, v, seed):
        v = np.ascontiguousarray(v, dtype=np.float32)
        sc = C.c_float()
        b = np.zeros(max(1, (v.size + 3) // 4), dtype=np.uint8)
        _check(self.L.ref_ternarize(_f(v), v.size, seed & 0xFFFFFFFFFFFFFFFF, C.byref(sc), b.ctypes.data_as(_u8p)))
        return sc.value, b[: (v.size + 3) // 4].copy()

    def deternarize(self, scale, sign_bytes, n):
        b = np.ascontiguousarray(sign_bytes if len(sign_bytes) else np.zeros(1, np.uint8), dtype=np.uint8)
        out = np.empty(max(1, n), dtype=np.float32)
        _check(self.L.ref_deternarize(scale, b.ctypes.data_as(_u8p), n, _f(out)))
        return out[:n]

    def encode_ternary(self, scale, sign_bytes, n, epoch, digest) -> bytes:
        b = np.ascontiguousarray(sign_bytes if len(sign_bytes) else np.zeros(1, np.uint8), dtype=np.uint8)
        out = (C.c_uint8 * (30 + (n + 3) // 4))()
        nb = C.c_size_t()
        _check(self.L.ref_encode_ternary(scale, b.ctypes.data_as(_u8p), n, epoch, digest, out, C.byref(nb)))
        return bytes(out)[: nb.value]

    def decode_ternary(self, frame: bytes):
        """-> (scale, len, digest, sign bytes); raises OracleError(8) on a corrupt frame"""
        buf = (C.c_uint8 * max(1, len(frame))).from_buffer_copy(frame or b"\0")
        sc, ln, dg = C.c_float(), C.c_uint64(), C.c_uint64()
        out = (C.c_uint8 * max(1, len(frame)))()
        _check(self.L.ref_decode_ternary(buf, len(frame), C.byref(sc), C.byref(ln), C.byref(dg), out))
        return sc.value, ln.value, dg.value, bytes(out)[: (ln.value + 3) // 4]

    def ternary_aggregate(self, grads, masks, stable, seeds, epoch):
        n = len(grads)
        ln = grads[0].size
        grads = [np.ascontiguousarray(x, dtype=np.float32) for x in grads]
        masks = [np.ascontiguousarray(m, dtype=np.uint64) for m in masks]
        outs = [np.empty_like(grads[0]) for _ in range(n)]
        st = (C.c_int * n)(*[int(bool(x)) for x in stable])
        sd = np.array([x & 0xFFFFFFFFFFFFFFFF for x in seeds], dtype=np.uint64)
        modes = (C.c_int * n)()
        byts = np.zeros(n, dtype=np.uint64)
        _check(self.L.ref_ternary_aggregate(
            n, C.cast(_ptr_array(grads, C.c_float), C.c_void_p),
            C.cast(_ptr_array(masks, C.c_uint64), C.c_void_p), st, _u(sd), epoch, ln,
            C.cast(_ptr_array(outs, C.c_float), C.c_void_p), modes, _u(byts)))
        return outs, list(modes), [int(b) for b in byts]

    # -- CPU baseline timing
    def bench_create(self, grads, words, slices=0):
        grads = [np.ascontiguousarray(x, dtype=np.float32) for x in grads]
        words = np.ascontiguousarray(words, dtype=np.uint64)
        self._keep = (grads, words)
        return self.L.ref_bench_create(len(grads), C.cast(_ptr_array(grads, C.c_float), C.c_void_p),
                                       _u(words), grads[0].size, slices)

    def bench_destroy(self, h):
        self.L.ref_bench_destroy(h)
        self._keep = None

    def bench_masked(self, h, epoch=0) -> float:
        return self.L.ref_bench_masked(h, epoch)

    def bench_pack_unpack(self, h, epoch=0) -> float:
        return self.L.ref_bench_pack_unpack(h, epoch)

    def bench_prune(self, w, ratio) -> float:
        w = np.ascontiguousarray(w, dtype=np.float32)
        return self.L.ref_bench_prune(_f(w), w.size, ratio)


@lru_cache(maxsize=1)
def port() -> Port:
    build()
    return Port()


@lru_cache(maxsize=1)
def ref() -> Ref:
    build()
    if not ref_available():
        raise RuntimeError("oracle/_ref/libpactref.so not built (reference sources absent)")
    return Ref()
