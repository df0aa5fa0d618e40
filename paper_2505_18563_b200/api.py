"""Python host mirror of the reference operator API for the hot path.

Same names, argument meaning and error behaviour as the reference C++ API
(/root/reference/proj/include/pact/{tensor,sparsity,codec,collective}.hpp),
but tensors are CUDA fp32 ``torch.Tensor``s and every computation runs in
the sm_100a kernels behind include/pact_c.h. torch is used only for device
memory, streams and torch.distributed plumbing.

Deviations, all deliberate:
  * ``FlatTensor`` is a 1-D CUDA float32 torch.Tensor.
  * ``masked_allreduce`` / ``full_allreduce`` take a :class:`Comm` backed by
    NCCL (one process per GPU) instead of a ring ``Transport``; passing
    ``comm=None`` runs the single-GPU path (pack -> unpack, no exchange),
    which the reference cannot express (it rejects n < 2).
  * ``SyncStats.seconds`` is measured device time, not a virtual clock;
    ``bytes_on_wire`` keeps the reference's ring accounting exactly.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import torch

from . import _lib
from ._lib import check, lib

# ------------------------------------------------------------------ errors


class Errc(enum.IntEnum):  # error.hpp:10-26, same order
    DuplicateParam = 0
    InvalidView = 1
    InvalidRatio = 2
    InvalidRate = 3
    NumericalFailure = 4
    ShapeMismatch = 5
    MaskMismatch = 6
    CorruptPayload = 7
    LinkError = 8
    UndefinedMetric = 9
    MissingFile = 10
    ParseError = 11
    UnknownKey = 12
    BadTopology = 13
    RunFailure = 14


class Error(RuntimeError):
    """error.hpp:51-62. ``code`` is an :class:`Errc` (None for CUDA/NCCL
    failures, whose C status is in ``status``)."""

    def __init__(self, code: Optional[Errc], what: str, status: int = 0):
        super().__init__(what)
        self.code = code
        self.status = status


def _call(fn, *args):
    st = fn(*args)
    if st != 0:
        msg = lib.pact_last_error().decode(errors="replace")
        code = Errc(st - 1) if 1 <= st <= 15 else None
        raise Error(code, msg, st)


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)
_cur_dev = getattr(torch._C, "_cuda_getDevice", None)


def _stream() -> C.c_void_p:
    # the raw handle of torch's current stream without building a Stream
    # object (this sits between the prune's readback and the next launch)
    if _raw_stream is not None and _cur_dev is not None:
        return C.c_void_p(_raw_stream(_cur_dev()))
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t: Optional[torch.Tensor]) -> C.c_void_p:
    return C.c_void_p(t.data_ptr() if t is not None else 0)


def _as_grad(x: torch.Tensor, name: str = "tensor") -> torch.Tensor:
    if not isinstance(x, torch.Tensor) or not x.is_cuda or x.dtype != torch.float32:
        raise TypeError(f"{name} must be a CUDA float32 tensor")
    return x.contiguous().view(-1)


# ---------------------------------------------------------------- context


class Context:
    """One pact_ctx per CUDA device (workspace, streams)."""

    _by_device: dict = {}

    def __init__(self, device: int):
        h = C.c_void_p()
        _call(lib.pact_ctx_create, device, C.byref(h))
        self.handle = h
        self.device = device

    @classmethod
    def get(cls, device: Optional[int] = None) -> "Context":
        if device is None:
            device = torch.cuda.current_device()
        if device not in cls._by_device:
            cls._by_device[device] = Context(device)
        return cls._by_device[device]

    def kernel_launches(self) -> int:
        return int(lib.pact_ctx_kernel_launches(self.handle))


# ------------------------------------------------------------------ masks


class _CudaArray:
    """__cuda_array_interface__ shim so torch can view library-owned memory."""

    def __init__(self, ptr: int, n: int, typestr: str, owner):
        self.__cuda_array_interface__ = {
            "shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3, "strides": None,
        }
        self._owner = owner


class SparsityMask:
    """tensor.hpp:78-106, device resident. Words use the reference layout
    (bit i at words[i>>6] bit i&63, tail bits zero)."""

    def __init__(self, length: int, ctx: Optional[Context] = None):
        self.ctx = ctx or Context.get()
        h = C.c_void_p()
        _call(lib.pact_mask_create, self.ctx.handle, int(length), C.byref(h))
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            lib.pact_mask_destroy(h)
            self.handle = None

    # -- constructors (tensor.cpp:87-105)
    @staticmethod
    def all_ones(length: int) -> "SparsityMask":
        m = SparsityMask(length)
        _call(lib.pact_mask_fill, m.handle, 1, _stream())
        return m

    @staticmethod
    def all_zeros(length: int) -> "SparsityMask":
        m = SparsityMask(length)
        _call(lib.pact_mask_fill, m.handle, 0, _stream())
        return m

    @staticmethod
    def from_words(words: torch.Tensor, length: int) -> "SparsityMask":
        m = SparsityMask(length)
        w = words.to(device=f"cuda:{m.ctx.device}", dtype=torch.int64).contiguous().view(-1)
        if w.numel() != (length + 63) // 64:
            raise Error(Errc.ShapeMismatch, f"{w.numel()} words for {length} bits")
        _call(lib.pact_mask_set_words, m.handle, _ptr(w), _stream())
        return m

    @staticmethod
    def from_bits(bits) -> "SparsityMask":
        b = torch.as_tensor(bits, dtype=torch.bool).view(-1).cpu()
        n = b.numel()
        padded = torch.zeros(((n + 63) // 64) * 64, dtype=torch.bool)
        padded[:n] = b
        import numpy as np

        words = np.packbits(padded.numpy().reshape(-1, 8), axis=1, bitorder="little").reshape(-1).view(np.int64)
        return SparsityMask.from_words(torch.from_numpy(words.copy()), n)

    # -- accessors
    def _info(self) -> _lib.MaskInfo:
        info = _lib.MaskInfo()
        _call(lib.pact_mask_info_get, self.handle, C.byref(info))
        return info

    def size(self) -> int:
        return int(self._info().len)

    def nnz(self) -> int:
        return int(self._info().nnz)

    def digest(self) -> int:
        d = C.c_uint64()
        _call(lib.pact_mask_digest, self.handle, _stream(), C.byref(d))
        return int(d.value)

    @property
    def changed(self) -> bool:
        return bool(self._info().changed)

    def words(self) -> torch.Tensor:
        """Zero-copy int64 view of the device words (valid while self lives)."""
        info = self._info()
        n = (int(info.len) + 63) // 64
        return torch.as_tensor(_CudaArray(int(info.words or 0), n, "<i8", self), device=f"cuda:{self.ctx.device}")

    def tile_offsets(self) -> torch.Tensor:
        info = self._info()
        return torch.as_tensor(_CudaArray(int(info.tile_off), int(info.ntiles) + 1, "<u4", self),
                               device=f"cuda:{self.ctx.device}")

    def words_host(self):
        return self.words().cpu().numpy().view("uint64").copy()

    def test(self, i: int) -> bool:
        w = int(self.words()[i >> 6].item()) & 0xFFFFFFFFFFFFFFFF
        return bool((w >> (i & 63)) & 1)

    def with_bit(self, i: int, keep: bool) -> "SparsityMask":  # tensor.cpp:107-115
        w = self.words().clone()
        word = int(w[i >> 6].item()) & 0xFFFFFFFFFFFFFFFF
        word = word | (1 << (i & 63)) if keep else word & ~(1 << (i & 63))
        if word >= 1 << 63:
            word -= 1 << 64
        w[i >> 6] = word
        return SparsityMask.from_words(w, self.size())

    def __eq__(self, other) -> bool:
        return isinstance(other, SparsityMask) and self.size() == other.size() and bool(
            torch.equal(self.words(), other.words()))

    __hash__ = None


def mask_digest(mask: SparsityMask) -> int:  # tensor.hpp:110
    return mask.digest()


def mask_gather(src: SparsityMask, segments: Sequence[Tuple[int, int]],
                out: Optional[SparsityMask] = None) -> SparsityMask:
    """Concatenate bit ranges (begin, length) of `src` into one mask: the mask
    of a DDP bucket whose parameters sit at those offsets of the flattened
    model (BucketView/flatten, tensor.hpp:54-74)."""
    total = sum(int(n) for _, n in segments)
    m = out if out is not None else SparsityMask(total, src.ctx)
    nseg = len(segments)
    begins = (C.c_uint64 * max(1, nseg))(*[int(b) for b, _ in segments])
    lens = (C.c_uint64 * max(1, nseg))(*[int(n) for _, n in segments])
    _call(lib.pact_mask_gather, src.handle, nseg, begins, lens, m.handle, _stream())
    return m


# ------------------------------------------------------------------ prune


@dataclass
class PruneConfig:  # sparsity.hpp:24-31 (magnitude method only)
    ratio: float = 0.0

    def validate(self) -> None:
        if not (0.0 <= self.ratio < 1.0):
            raise Error(Errc.InvalidRatio, f"prune ratio {self.ratio} outside [0, 1)")


def drop_count(ratio: float, length: int) -> int:  # sparsity.cpp:33-40
    k = C.c_uint64()
    _call(lib.pact_drop_count, C.c_float(ratio), int(length), C.byref(k))
    return int(k.value)


def magnitude_prune(weights: torch.Tensor, ratio: float, out: Optional[SparsityMask] = None,
                    stats: Optional[dict] = None) -> SparsityMask:
    """sparsity.cpp:44-59: keep all but the k smallest |w| (ties drop the lower
    index first). ``out`` reuses a mask (its ``changed`` flag then reports
    whether the words moved, which feeds the tracker without a digest)."""
    w = _as_grad(weights, "weights")
    m = out if out is not None else SparsityMask(w.numel())
    ps = _lib.PruneStats()
    _call(lib.pact_prune_magnitude, m.ctx.handle, _ptr(w), w.numel(), C.c_float(ratio), m.handle,
          _stream(), C.byref(ps))
    if stats is not None:
        stats.update(k=ps.k, threshold=ps.threshold, c_lt=ps.c_lt, path=ps.path, candidates=ps.candidates)
    return m


def magnitude_prune_per_layer(weights: torch.Tensor, seg_offsets: Sequence[int], ratio: float,
                              out: Optional[SparsityMask] = None) -> SparsityMask:
    """Per-layer mode (north_star): the reference rule applied to
    every [seg[s], seg[s+1]) slice with k_s = drop_count(ratio, len_s)."""
    w = _as_grad(weights, "weights")
    m = out if out is not None else SparsityMask(w.numel())
    seg = (C.c_uint64 * len(seg_offsets))(*[int(x) for x in seg_offsets])
    _call(lib.pact_prune_magnitude_segmented, m.ctx.handle, _ptr(w), w.numel(), seg,
          len(seg_offsets) - 1, C.c_float(ratio), m.handle, _stream())
    return m


def build_prune_mask(weights: torch.Tensor, cfg: PruneConfig) -> SparsityMask:  # sparsity.cpp:121-128
    cfg.validate()
    return magnitude_prune(weights, cfg.ratio)


def enforce_gradient_sparsity(grad: torch.Tensor, mask: SparsityMask, out: Optional[torch.Tensor] = None
                              ) -> torch.Tensor:
    """sparsity.cpp:112-119 (out may be grad for the in-place variant)."""
    g = _as_grad(grad, "grad")
    o = torch.empty_like(g) if out is None else out
    _call(lib.pact_gse, mask.ctx.handle, _ptr(g), g.numel(), mask.handle, _ptr(o), _stream())
    return o


class TrackerStatus(enum.Enum):  # sparsity.hpp:33
    Stable = 0
    Unstable = 1


class MaskTracker:
    """sparsity.hpp:37-54 / sparsity.cpp:17-25 (host state machine)."""

    def __init__(self, stability_threshold: int = 3):
        self._t = _lib.Tracker()
        lib.pact_tracker_init(C.byref(self._t), int(stability_threshold))

    def observe(self, mask: SparsityMask) -> TrackerStatus:
        return self.observe_digest(mask.digest())

    def observe_digest(self, digest: int) -> TrackerStatus:
        s = lib.pact_tracker_observe(C.byref(self._t), int(digest) & 0xFFFFFFFFFFFFFFFF)
        return TrackerStatus.Stable if s else TrackerStatus.Unstable

    def status(self) -> TrackerStatus:
        return TrackerStatus.Stable if lib.pact_tracker_status(C.byref(self._t)) else TrackerStatus.Unstable

    def stable_count(self) -> int:
        return int(self._t.stable_count)

    def last_digest(self) -> Optional[int]:
        return int(self._t.last_digest) if self._t.has_last else None


def tracker_observe(tracker: MaskTracker, mask: SparsityMask) -> TrackerStatus:
    return tracker.observe(mask)


# ------------------------------------------------------------------ codec


@dataclass
class PackedGradient:  # codec.hpp:19-23
    mask_digest: int = 0
    epoch: int = 0
    values: Optional[torch.Tensor] = None


def pack(grad: torch.Tensor, mask: SparsityMask, epoch: int) -> PackedGradient:  # codec.cpp:14-25
    g = _as_grad(grad, "grad")
    if g.numel() != mask.size():
        raise Error(Errc.ShapeMismatch, f"gradient length {g.numel()} != mask length {mask.size()}")
    vals = torch.empty(max(1, mask.nnz()), dtype=torch.float32, device=g.device)[: mask.nnz()]
    _call(lib.pact_pack, mask.ctx.handle, _ptr(g), g.numel(), mask.handle, _ptr(vals), 0,
          C.c_uint64(0xFFFFFFFFFFFFFFFF), _stream())
    return PackedGradient(mask.digest(), int(epoch), vals)


def unpack(packed: PackedGradient, mask: SparsityMask, scale: float = 1.0,
           out: Optional[torch.Tensor] = None) -> torch.Tensor:  # codec.cpp:27-38
    vals = packed.values if packed.values is not None else torch.empty(0, device="cuda")
    o = torch.empty(mask.size(), dtype=torch.float32, device=f"cuda:{mask.ctx.device}") if out is None else out
    _call(lib.pact_unpack, mask.ctx.handle, _ptr(vals), vals.numel(),
          C.c_uint64(int(packed.mask_digest) & 0xFFFFFFFFFFFFFFFF), 1, mask.handle,
          C.c_float(scale), _ptr(o), 0, C.c_uint64(0xFFFFFFFFFFFFFFFF), _stream())
    return o


def unpack_sgd(packed_values: torch.Tensor, mask: SparsityMask, scale: float, lr: float,
               weights: torch.Tensor, grad_out: Optional[torch.Tensor] = None) -> None:
    """Fused unpack + to_mean + masked SGD step (trainer.cpp:202-214, 268-273)."""
    _call(lib.pact_unpack_sgd, mask.ctx.handle, _ptr(packed_values), packed_values.numel(),
          mask.handle, C.c_float(scale), C.c_float(lr), _ptr(grad_out), _ptr(weights), _stream())


@dataclass
class TernaryGradient:  # codec.hpp:32-40
    """Device ternary payload: ``scale`` (host float, also ``scale_dev``) and
    ``signs`` (device uint8, pact_ternary_sign_bytes(len) bytes whose first
    ceil(len/4) are the reference's ``sign_words``)."""
    scale: float = 0.0
    len: int = 0
    signs: Optional[torch.Tensor] = None
    scale_dev: Optional[torch.Tensor] = None

    def sign_words(self) -> bytes:
        return bytes(self.signs[: (self.len + 3) // 4].cpu().numpy().tobytes()) if self.len else b""

    def sign_at(self, i: int) -> int:  # codec.cpp:40-48
        pair = (self.sign_words()[i >> 2] >> (2 * (i & 3))) & 3
        if pair == 3:
            raise Error(Errc.CorruptPayload, "reserved ternary sign pattern 11")
        return (0, 1, -1)[pair]


def ternary_sign_bytes(count: int) -> int:
    return int(lib.pact_ternary_sign_bytes(int(count)))


def ternarize(grad: torch.Tensor, seed: int) -> TernaryGradient:  # codec.cpp:50-68
    """Stochastic ternarization on the GPU; draws from a counter-based
    SplitMix64 stream of ``seed`` (the reference's mt19937_64 stream is
    sequential; the distribution and every draw-independent result match)."""
    g = _as_grad(grad, "grad")
    signs = torch.empty(max(16, ternary_sign_bytes(g.numel())), dtype=torch.uint8, device=g.device)
    sc = torch.empty(1, dtype=torch.float32, device=g.device)
    _call(lib.pact_ternarize, Context.get(g.device.index).handle, _ptr(g), g.numel(),
          C.c_uint64(int(seed) & 0xFFFFFFFFFFFFFFFF), _ptr(sc), _ptr(signs), _stream())
    return TernaryGradient(float(sc.item()), g.numel(), signs, sc)


def deternarize(t: TernaryGradient, out: Optional[torch.Tensor] = None) -> torch.Tensor:  # codec.cpp:70-75
    dev = t.signs.device if t.signs is not None else torch.device("cuda", torch.cuda.current_device())
    o = torch.empty(t.len, dtype=torch.float32, device=dev) if out is None else out
    sc = t.scale_dev if t.scale_dev is not None else torch.tensor([t.scale], dtype=torch.float32, device=dev)
    signs = t.signs if t.signs is not None else torch.zeros(16, dtype=torch.uint8, device=dev)
    _call(lib.pact_deternarize, Context.get(dev.index).handle, _ptr(sc), _ptr(signs), t.len, _ptr(o),
          _stream())
    return o


@dataclass
class TopKPayload:  # codec.hpp:60-66 (device tensors)
    indices: Optional[torch.Tensor] = None  # int32 view of the u32 indices, strictly increasing
    values: Optional[torch.Tensor] = None
    original_len: int = 0


def topk_count(length: int, rate: float) -> int:  # codec.cpp:148-155
    k = C.c_uint64()
    _call(lib.pact_topk_count, int(length), C.c_float(rate), C.byref(k))
    return int(k.value)


def topk_select(grad: torch.Tensor, rate: float) -> TopKPayload:  # codec.cpp:147-172
    g = _as_grad(grad, "grad")
    k = topk_count(g.numel(), rate)
    idx = torch.empty(max(1, k), dtype=torch.int32, device=g.device)
    val = torch.empty(max(1, k), dtype=torch.float32, device=g.device)
    kk = C.c_uint64()
    _call(lib.pact_topk_select, Context.get(g.device.index).handle, _ptr(g), g.numel(), C.c_float(rate),
          _ptr(idx), _ptr(val), C.byref(kk), _stream())
    return TopKPayload(idx[:k], val[:k], g.numel())


def topk_densify(p: TopKPayload, out: Optional[torch.Tensor] = None) -> torch.Tensor:  # codec.cpp:174-182
    dev = p.values.device if p.values is not None else torch.device("cuda", torch.cuda.current_device())
    o = torch.empty(p.original_len, dtype=torch.float32, device=dev) if out is None else out
    k = p.indices.numel() if p.indices is not None else 0
    _call(lib.pact_topk_densify, Context.get(dev.index).handle, _ptr(p.indices), _ptr(p.values), k,
          p.original_len, _ptr(o), _stream())
    return o


class PayloadKind(enum.IntEnum):  # codec.hpp:80-86
    Full = 0
    Packed = 1
    Ternary = 2
    Fp16 = 3
    TopK = 4


@dataclass
class FrameHeader:  # codec.hpp:93-98
    kind: PayloadKind = PayloadKind.Full
    epoch: int = 0
    mask_digest: int = 0
    value_count: int = 0


def encode_header(h: FrameHeader) -> bytes:  # codec.cpp:257-259
    ch = _lib.FrameHeader(int(h.kind), h.epoch, h.mask_digest & 0xFFFFFFFFFFFFFFFF, h.value_count)
    out = (C.c_uint8 * 26)()
    _call(lib.pact_header_encode, C.byref(ch), out)
    return bytes(out)


def decode_header(frame: bytes) -> FrameHeader:  # codec.cpp:261-275
    buf = (C.c_uint8 * max(1, len(frame))).from_buffer_copy(bytes(frame) or b"\0")
    ch = _lib.FrameHeader()
    _call(lib.pact_header_decode, buf, len(frame), C.byref(ch))
    return FrameHeader(PayloadKind(ch.kind), ch.epoch, ch.mask_digest, ch.value_count)


def encode_ternary(t: TernaryGradient, epoch: int, mask_digest: int) -> bytes:  # codec.cpp:313-318
    import struct

    return (encode_header(FrameHeader(PayloadKind.Ternary, epoch, mask_digest, t.len))
            + struct.pack("<f", t.scale) + t.sign_words())


def decode_ternary(frame: bytes) -> Tuple[TernaryGradient, int]:  # codec.cpp:320-343
    """Host decode with the reference's checks; returns (ternary with HOST
    sign bytes in ``signs`` as a CPU uint8 tensor, mask digest)."""
    import math
    import struct

    h = decode_header(frame)
    if h.kind != PayloadKind.Ternary:
        raise Error(Errc.CorruptPayload, "not a ternary frame")
    words = (h.value_count + 3) // 4
    if len(frame) < 26 + 4 + words:
        raise Error(Errc.CorruptPayload, "frame truncated")
    scale = struct.unpack_from("<f", frame, 26)[0]
    if not (scale >= 0.0) or not math.isfinite(scale):
        raise Error(Errc.CorruptPayload, "negative or non-finite ternary scale")
    sw = bytes(frame[30:30 + words])
    import numpy as np

    b = np.frombuffer(sw, dtype=np.uint8)
    pairs = ((b[:, None] >> np.array([0, 2, 4, 6], dtype=np.uint8)) & 3).reshape(-1)
    if (pairs[: h.value_count] == 3).any():
        raise Error(Errc.CorruptPayload, "reserved ternary sign pattern 11")
    if pairs[h.value_count:].any():
        raise Error(Errc.CorruptPayload, "sign bits past payload length")
    if scale == 0.0 and pairs.any():
        raise Error(Errc.CorruptPayload, "zero scale with non-zero signs")
    return TernaryGradient(scale, int(h.value_count), torch.from_numpy(b.copy())), int(h.mask_digest)


def encode_topk(p: TopKPayload, epoch: int) -> bytes:  # codec.cpp:345-350
    idx = p.indices.cpu().numpy().astype("<u4").tobytes()
    val = p.values.cpu().numpy().astype("<f4").tobytes()
    return encode_header(FrameHeader(PayloadKind.TopK, epoch, 0, p.indices.numel())) + idx + val


def decode_topk(frame: bytes, original_len: int) -> TopKPayload:  # codec.cpp:352-369
    """Host decode with the reference's checks (range, strictly increasing)."""
    import numpy as np

    h = decode_header(frame)
    if h.kind != PayloadKind.TopK:
        raise Error(Errc.CorruptPayload, "not a topk frame")
    k = int(h.value_count)
    if len(frame) < 26 + 8 * k:
        raise Error(Errc.CorruptPayload, "frame truncated")
    idx = np.frombuffer(frame, dtype="<u4", count=k, offset=26).copy()
    val = np.frombuffer(frame, dtype="<f4", count=k, offset=26 + 4 * k).copy()
    if k and (idx >= original_len).any():
        raise Error(Errc.CorruptPayload, "topk index out of range")
    if k > 1 and not (np.diff(idx.astype(np.int64)) > 0).all():
        raise Error(Errc.CorruptPayload, "topk indices not strictly increasing")
    return TopKPayload(torch.from_numpy(idx.view(np.int32)), torch.from_numpy(val), int(original_len))


# -------------------------------------------------------------- collective


class SyncMode(enum.IntEnum):  # collective.hpp:58-64
    FullAllReduce = 0
    PackedAllReduce = 1
    TernaryAllGather = 2
    TopKAllGather = 3
    Fp16AllReduce = 4


def decide_sync_mode(requested: SyncMode, tracker: TrackerStatus) -> SyncMode:  # collective.cpp:62-67
    return SyncMode(lib.pact_decide_sync_mode(int(requested), int(tracker == TrackerStatus.Stable)))


def vote_decide(frames: Sequence[bytes], mine: FrameHeader, stable: bool) -> bool:
    """collective.cpp:285-293 unanimity rule (host scalar logic)."""
    blob = b"".join(frames)
    buf = (C.c_uint8 * max(1, len(blob))).from_buffer_copy(blob or b"\0")
    ch = _lib.FrameHeader(int(mine.kind), mine.epoch, mine.mask_digest & 0xFFFFFFFFFFFFFFFF, mine.value_count)
    agree = C.c_int()
    _call(lib.pact_vote_decide, buf, len(frames), C.byref(ch), int(bool(stable)), C.byref(agree))
    return bool(agree.value)


def ring_bytes(n: int, position: int, count: int) -> int:
    return int(lib.pact_ring_bytes(n, position, count))


def masked_bytes(n: int, position: int, count: int) -> int:
    return int(lib.pact_masked_bytes(n, position, count))


@dataclass
class SyncStats:  # collective.hpp:73-77
    bytes_on_wire: int = 0
    seconds: float = 0.0
    mode_used: SyncMode = SyncMode.FullAllReduce
    buckets: int = 0
    value_count: int = 0
    fallback_reason: int = 0
    transport: int = 0               # 0 none (1 GPU), 1 NCCL, 2 NVLink P2P
    t_pack: float = 0.0              # device seconds per stage (policy.time_stages)
    t_exchange: float = 0.0
    t_unpack: float = 0.0


@dataclass
class AggregateResult:  # collective.hpp:130-133
    tensor: Optional[torch.Tensor] = None
    stats: SyncStats = field(default_factory=SyncStats)


@dataclass
class SyncPolicy:
    """Adaptive knobs. Defaults == reference policy."""

    AUTO, NCCL, P2P = 0, 1, 2

    density_threshold: float = 0.0   # fall back to dense above this agreed density (0: never)
    bucket_bytes: int = 0            # packed bytes per overlapped bucket (0: auto, see pact_c.h)
    scale: float = 1.0               # fused into unpack (1/n gives the mean)
    time_stages: bool = False
    transport: int = 0               # 0 auto, 1 NCCL allreduce, 2 NVLink P2P (bit-exact fold order)
    wire: int = 0                    # packed payload: 0 fp32 (reference), 1 binary16 ring (F16Wire)
    gse_dense: bool = False          # gradient not yet masked: the dense fallback applies GSE first

    F32, F16 = 0, 1

    def c(self) -> _lib.PolicyC:
        return _lib.PolicyC(self.density_threshold, self.bucket_bytes, self.scale, int(self.time_stages),
                            int(self.transport), int(self.wire), int(self.gse_dense))


def _stats(s: _lib.SyncStatsC) -> SyncStats:
    return SyncStats(int(s.bytes_on_wire), float(s.seconds), SyncMode(s.mode_used), int(s.buckets),
                     int(s.value_count), int(s.fallback_reason), int(s.transport), float(s.t_pack),
                     float(s.t_exchange), float(s.t_unpack))


class Comm:
    """NCCL-backed worker endpoint (collective.hpp:89-116), one per GPU."""

    def __init__(self, rank: int, world_size: int, unique_id: bytes, ctx: Optional[Context] = None):
        self.ctx = ctx or Context.get()
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        h = C.c_void_p()
        _call(lib.pact_comm_create, self.ctx.handle, buf, int(world_size), int(rank), C.byref(h))
        self.handle = h

    @staticmethod
    def unique_id() -> bytes:
        out = (C.c_uint8 * 128)()
        _call(lib.pact_comm_unique_id, out)
        return bytes(out)

    @staticmethod
    def from_process_group(group=None, ctx: Optional[Context] = None) -> "Comm":
        """Rendezvous over an initialised torch.distributed group (gloo or nccl)."""
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return Comm(rank, world, obj[0], ctx)

    def rank(self) -> int:
        return int(lib.pact_comm_rank(self.handle))

    def world_size(self) -> int:
        return int(lib.pact_comm_size(self.handle))

    def check(self, timeout_ms: int = 0) -> None:
        """Wait for this rank's collectives on the current stream with a
        deadline; raises Error(LinkError) when a peer is lost (reference
        SimCluster::poison, collective.cpp:430-458). timeout_ms <= 0:
        PACT_LINK_TIMEOUT_MS (default 30 s)."""
        _call(lib.pact_comm_check, self.handle, _stream(), int(timeout_ms))

    @property
    def failed(self) -> bool:
        return bool(lib.pact_comm_failed(self.handle))

    def close(self) -> None:
        if getattr(self, "handle", None) is not None and self.handle.value:
            lib.pact_comm_destroy(self.handle)
            self.handle = None


def ring_allreduce(local: torch.Tensor, comm: Comm, out: Optional[torch.Tensor] = None,
                   exact: bool = False) -> torch.Tensor:
    """collective.cpp:165-216 (SUM). exact=False: NCCL chooses the reduction
    order; exact=True: the reference's own fold order over NVLink peer memory
    (pact_ring_allreduce), bit-identical to the reference ring on every rank,
    with the reference's length agreement (ShapeMismatch)."""
    g = _as_grad(local, "local")
    o = torch.empty_like(g) if out is None else out
    if exact:
        _call(lib.pact_ring_allreduce, comm.handle, _ptr(g), _ptr(o), g.numel(), _stream())
    else:
        _call(lib.pact_allreduce_sum, comm.handle, _ptr(g), _ptr(o), g.numel(), _stream())
    return o


def allgather(payload: bytes, comm: Comm) -> list:
    """collective.cpp:222-247 for equal-size frames; result indexed by rank."""
    n = comm.world_size()
    src = (C.c_uint8 * max(1, len(payload))).from_buffer_copy(payload or b"\0")
    dst = (C.c_uint8 * max(1, len(payload) * n))()
    _call(lib.pact_allgather_frames, comm.handle, src, len(payload), dst, _stream())
    raw = bytes(dst)
    return [raw[i * len(payload):(i + 1) * len(payload)] for i in range(n)]


def full_allreduce(grad: torch.Tensor, comm: Comm, scale: float = 1.0,
                   out: Optional[torch.Tensor] = None) -> AggregateResult:  # collective.cpp:253-259
    g = _as_grad(grad, "grad")
    o = torch.empty_like(g) if out is None else out
    st = _lib.SyncStatsC()
    _call(lib.pact_full_allreduce, comm.handle, _ptr(g), _ptr(o), g.numel(), C.c_float(scale),
          C.byref(st), _stream())
    return AggregateResult(o, _stats(st))


def masked_allreduce(grad: torch.Tensor, mask: SparsityMask, tracker: TrackerStatus, epoch: int,
                     comm: Optional[Comm], advertised_digest: Optional[int] = None,
                     policy: Optional[SyncPolicy] = None,
                     out: Optional[torch.Tensor] = None) -> AggregateResult:
    """collective.cpp:269-309: vote, then pack -> sum-allreduce -> unpack on a
    unanimous stable vote, else a dense sum-allreduce. Returns the SUM
    (times policy.scale)."""
    g = _as_grad(grad, "grad")
    o = torch.empty_like(g) if out is None else out
    st = _lib.SyncStatsC()
    pol = (policy or SyncPolicy()).c()
    adv = None
    if advertised_digest is not None:
        adv = C.c_uint64(int(advertised_digest) & 0xFFFFFFFFFFFFFFFF)
    _call(lib.pact_masked_allreduce, comm.handle if comm is not None else None, mask.ctx.handle,
          _ptr(g), g.numel(), mask.handle, int(tracker == TrackerStatus.Stable), int(epoch),
          C.byref(adv) if adv is not None else None, C.byref(pol), _ptr(o), C.byref(st), _stream())
    return AggregateResult(o, _stats(st))


@dataclass
class DensityCalibration:
    """pact_calibrate_density: the measured dense/sparse crossover."""
    threshold: float              # feed to SyncPolicy.density_threshold (1.0: packing always wins)
    densities: List[float]
    t_packed: List[float]         # seconds per masked_allreduce at each probe density (max over ranks)
    t_dense: float                # seconds per dense masked_allreduce (max over ranks)


def calibrate_density(length: int, comm: Optional[Comm], policy: Optional[SyncPolicy] = None,
                      densities: Optional[Sequence[float]] = None,
                      ctx: Optional["Context"] = None) -> DensityCalibration:
    """The adaptive policy's crossover density, measured on this communicator
    for gradients of `length` elements (north_star (4)). Collective:
    call on every rank with the same arguments."""
    ctx = ctx or (comm.ctx if comm is not None else Context.get())
    ds = list(densities) if densities is not None else [0.01, 0.02, 0.05, 0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7,
                                                         0.8, 0.9, 0.95]
    dv = (C.c_double * len(ds))(*ds)
    tp = (C.c_double * len(ds))()
    td, thr = C.c_double(), C.c_double()
    pol = (policy or SyncPolicy()).c()
    _call(lib.pact_calibrate_density, comm.handle if comm is not None else None, ctx.handle, int(length),
          C.byref(pol), dv, len(ds), tp, C.byref(td), C.byref(thr), _stream())
    return DensityCalibration(thr.value, ds, list(tp), td.value)


def masked_allreduce_host(grad_host: torch.Tensor, mask: SparsityMask, tracker: TrackerStatus,
                          epoch: int, comm: Optional[Comm], out_host: torch.Tensor,
                          policy: Optional[SyncPolicy] = None) -> SyncStats:
    """The same call on HOST (ideally pinned) fp32 buffers: H2D, device path, D2H."""
    st = _lib.SyncStatsC()
    pol = (policy or SyncPolicy()).c()
    _call(lib.pact_masked_allreduce_host, comm.handle if comm is not None else None, mask.ctx.handle,
          _ptr(grad_host), grad_host.numel(), mask.handle, int(tracker == TrackerStatus.Stable),
          int(epoch), None, C.byref(pol), _ptr(out_host), C.byref(st), _stream())
    return _stats(st)


def topk_allgather_aggregate(grad: torch.Tensor, rate: float, epoch: int, comm: Optional[Comm],
                             out: Optional[torch.Tensor] = None) -> AggregateResult:  # collective.cpp:370-390
    """All-gather of every rank's TopK payload, double-accumulated densify,
    float(acc / n). Returns the MEAN."""
    g = _as_grad(grad, "grad")
    o = torch.empty_like(g) if out is None else out
    st = _lib.SyncStatsC()
    ctx = comm.ctx if comm is not None else Context.get(g.device.index)
    _call(lib.pact_topk_allgather_aggregate, comm.handle if comm is not None else None, ctx.handle, _ptr(g),
          g.numel(), C.c_float(rate), int(epoch), _ptr(o), C.byref(st), _stream())
    return AggregateResult(o, _stats(st))


def fp16_roundtrip(grad: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:  # codec.cpp:142-146
    g = _as_grad(grad, "grad")
    o = torch.empty_like(g) if out is None else out
    _call(lib.pact_fp16_roundtrip, Context.get(g.device.index).handle, _ptr(g), _ptr(o), g.numel(), _stream())
    return o


def fp16_allreduce(grad: torch.Tensor, comm: Optional[Comm],
                   out: Optional[torch.Tensor] = None) -> AggregateResult:  # collective.cpp:261-267
    """Dense ring all-reduce with binary16 chunks re-rounded at every hop
    (F16Wire, collective.cpp:133-163), bit-identical to the reference ring."""
    g = _as_grad(grad, "grad")
    o = torch.empty_like(g) if out is None else out
    st = _lib.SyncStatsC()
    ctx = comm.ctx if comm is not None else Context.get(g.device.index)
    _call(lib.pact_fp16_allreduce, comm.handle if comm is not None else None, ctx.handle, _ptr(g), _ptr(o),
          g.numel(), C.byref(st), _stream())
    return AggregateResult(o, _stats(st))


def ternary_allgather_aggregate(grad: torch.Tensor, mask: SparsityMask, tracker: TrackerStatus, seed: int,
                                epoch: int, comm: Optional[Comm],
                                out: Optional[torch.Tensor] = None) -> AggregateResult:
    """collective.cpp:311-368: pack -> ternarize -> all-gather -> mean ->
    unpack on a unanimous stable vote, else dense all-reduce / n. Returns
    the MEAN."""
    g = _as_grad(grad, "grad")
    o = torch.empty_like(g) if out is None else out
    st = _lib.SyncStatsC()
    _call(lib.pact_ternary_allgather_aggregate, comm.handle if comm is not None else None, mask.ctx.handle,
          _ptr(g), g.numel(), mask.handle, int(tracker == TrackerStatus.Stable),
          C.c_uint64(int(seed) & 0xFFFFFFFFFFFFFFFF), int(epoch), _ptr(o), C.byref(st), _stream())
    return AggregateResult(o, _stats(st))


def synth_fill(x: torch.Tensor, seed: int, recipe: int, scale: float = 1.0, index_base: int = 0) -> torch.Tensor:
    """Device-side synthetic data; host twin in synth.py."""
    ctx = Context.get(x.device.index)
    _call(lib.pact_synth_fill, ctx.handle, _ptr(x), x.numel(), C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF),
          C.c_uint64(index_base), int(recipe), C.c_float(scale), _stream())
    return x
