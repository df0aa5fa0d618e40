"""ctypes binding of the C-ABI (include/pact_c.h) -- the only way the Python
host mirror reaches the GPU. There is no CPU fallback: if the native library
is missing, importing this module raises."""
from __future__ import annotations

import ctypes as C
import os

from ._build import LIB

if not os.path.exists(LIB):
    raise ImportError(
        f"native library {LIB} is missing; build it with "
        "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)"
    )

_L = C.CDLL(LIB)

u8p = C.POINTER(C.c_uint8)
u64p = C.POINTER(C.c_uint64)
vp = C.c_void_p


class FrameHeader(C.Structure):
    _fields_ = [("kind", C.c_uint8), ("epoch", C.c_uint32), ("mask_digest", C.c_uint64),
                ("value_count", C.c_uint64)]


class Tracker(C.Structure):
    _fields_ = [("threshold", C.c_uint32), ("stable_count", C.c_uint32), ("has_last", C.c_int),
                ("last_digest", C.c_uint64)]


class SyncStatsC(C.Structure):
    _fields_ = [("bytes_on_wire", C.c_uint64), ("seconds", C.c_double), ("mode_used", C.c_int),
                ("buckets", C.c_int), ("value_count", C.c_uint64), ("fallback_reason", C.c_int),
                ("transport", C.c_int), ("t_pack", C.c_double), ("t_exchange", C.c_double),
                ("t_unpack", C.c_double)]


class PolicyC(C.Structure):
    _fields_ = [("density_threshold", C.c_double), ("bucket_bytes", C.c_uint64),
                ("scale", C.c_float), ("time_stages", C.c_int), ("transport", C.c_int),
                ("wire", C.c_int), ("gse_dense", C.c_int)]


class MaskInfo(C.Structure):
    _fields_ = [("len", C.c_uint64), ("nnz", C.c_uint64), ("digest", C.c_uint64),
                ("digest_valid", C.c_int), ("changed", C.c_int), ("ntiles", C.c_uint64),
                ("words", C.c_void_p), ("tile_off", C.c_void_p)]


class PruneStats(C.Structure):
    _fields_ = [("k", C.c_uint64), ("threshold", C.c_uint32), ("c_lt", C.c_uint64),
                ("path", C.c_int), ("candidates", C.c_uint64)]


# name -> (restype, argtypes); every symbol declared in include/pact_c.h
SIGNATURES = {
    "pact_status_name": (C.c_char_p, [C.c_int]),
    "pact_last_error": (C.c_char_p, []),
    "pact_abi_version": (C.c_int, []),
    "pact_drop_count": (C.c_int, [C.c_float, C.c_uint64, u64p]),
    "pact_header_encode": (C.c_int, [C.POINTER(FrameHeader), u8p]),
    "pact_header_decode": (C.c_int, [u8p, C.c_size_t, C.POINTER(FrameHeader)]),
    "pact_tracker_init": (None, [C.POINTER(Tracker), C.c_uint32]),
    "pact_tracker_observe": (C.c_int, [C.POINTER(Tracker), C.c_uint64]),
    "pact_tracker_status": (C.c_int, [C.POINTER(Tracker)]),
    "pact_decide_sync_mode": (C.c_int, [C.c_int, C.c_int]),
    "pact_vote_decide": (C.c_int, [u8p, C.c_int, C.POINTER(FrameHeader), C.c_int, C.POINTER(C.c_int)]),
    "pact_ring_bytes": (C.c_uint64, [C.c_int, C.c_int, C.c_uint64]),
    "pact_masked_bytes": (C.c_uint64, [C.c_int, C.c_int, C.c_uint64]),
    "pact_ctx_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
    "pact_ctx_destroy": (C.c_int, [vp]),
    "pact_ctx_kernel_launches": (C.c_uint64, [vp]),
    "pact_mask_create": (C.c_int, [vp, C.c_uint64, C.POINTER(vp)]),
    "pact_mask_destroy": (C.c_int, [vp]),
    "pact_mask_info_get": (C.c_int, [vp, C.POINTER(MaskInfo)]),
    "pact_mask_fill": (C.c_int, [vp, C.c_int, vp]),
    "pact_mask_set_words": (C.c_int, [vp, vp, vp]),
    "pact_mask_digest": (C.c_int, [vp, vp, u64p]),
    "pact_mask_gather": (C.c_int, [vp, C.c_uint64, u64p, u64p, vp, vp]),
    "pact_prune_magnitude": (C.c_int, [vp, vp, C.c_uint64, C.c_float, vp, vp, C.POINTER(PruneStats)]),
    "pact_prune_magnitude_segmented": (C.c_int, [vp, vp, C.c_uint64, u64p, C.c_uint64, C.c_float, vp, vp]),
    "pact_gse": (C.c_int, [vp, vp, C.c_uint64, vp, vp, vp]),
    "pact_pack": (C.c_int, [vp, vp, C.c_uint64, vp, vp, C.c_uint64, C.c_uint64, vp]),
    "pact_debug_pack_push": (C.c_int, [vp, vp, C.c_uint64, vp, vp, vp, vp]),
    "pact_unpack": (C.c_int, [vp, vp, C.c_uint64, C.c_uint64, C.c_int, vp, C.c_float, vp,
                              C.c_uint64, C.c_uint64, vp]),
    "pact_unpack_sgd": (C.c_int, [vp, vp, C.c_uint64, vp, C.c_float, C.c_float, vp, vp, vp]),
    "pact_synth_fill": (C.c_int, [vp, vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, C.c_float, vp]),
    "pact_comm_unique_id": (C.c_int, [u8p]),
    "pact_comm_create": (C.c_int, [vp, u8p, C.c_int, C.c_int, C.POINTER(vp)]),
    "pact_comm_destroy": (C.c_int, [vp]),
    "pact_comm_rank": (C.c_int, [vp]),
    "pact_comm_size": (C.c_int, [vp]),
    "pact_allreduce_sum": (C.c_int, [vp, vp, vp, C.c_uint64, vp]),
    "pact_ring_allreduce": (C.c_int, [vp, vp, vp, C.c_uint64, vp]),
    "pact_comm_check": (C.c_int, [vp, vp, C.c_int]),
    "pact_comm_failed": (C.c_int, [vp]),
    "pact_allgather_frames": (C.c_int, [vp, u8p, C.c_size_t, u8p, vp]),
    "pact_full_allreduce": (C.c_int, [vp, vp, vp, C.c_uint64, C.c_float, C.POINTER(SyncStatsC), vp]),
    "pact_masked_allreduce": (C.c_int, [vp, vp, vp, C.c_uint64, vp, C.c_int, C.c_uint32, u64p,
                                        C.POINTER(PolicyC), vp, C.POINTER(SyncStatsC), vp]),
    "pact_calibrate_density": (C.c_int, [vp, vp, C.c_uint64, C.POINTER(PolicyC), C.POINTER(C.c_double), C.c_int,
                                         C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double), vp]),
    "pact_topk_count": (C.c_int, [C.c_uint64, C.c_float, u64p]),
    "pact_topk_select": (C.c_int, [vp, vp, C.c_uint64, C.c_float, vp, vp, u64p, vp]),
    "pact_topk_densify": (C.c_int, [vp, vp, vp, C.c_uint64, C.c_uint64, vp, vp]),
    "pact_topk_allgather_aggregate": (C.c_int, [vp, vp, vp, C.c_uint64, C.c_float, C.c_uint32, vp,
                                                C.POINTER(SyncStatsC), vp]),
    "pact_fp16_roundtrip": (C.c_int, [vp, vp, vp, C.c_uint64, vp]),
    "pact_fp16_allreduce": (C.c_int, [vp, vp, vp, vp, C.c_uint64, C.POINTER(SyncStatsC), vp]),
    "pact_ternary_sign_bytes": (C.c_uint64, [C.c_uint64]),
    "pact_ternarize": (C.c_int, [vp, vp, C.c_uint64, C.c_uint64, vp, vp, vp]),
    "pact_deternarize": (C.c_int, [vp, vp, vp, C.c_uint64, vp, vp]),
    "pact_ternary_allgather_aggregate": (C.c_int, [vp, vp, vp, C.c_uint64, vp, C.c_int, C.c_uint64,
                                                   C.c_uint32, vp, C.POINTER(SyncStatsC), vp]),
    "pact_masked_allreduce_host": (C.c_int, [vp, vp, vp, C.c_uint64, vp, C.c_int, C.c_uint32, u64p,
                                             C.POINTER(PolicyC), vp, C.POINTER(SyncStatsC), vp]),
}

for _name, (_res, _args) in SIGNATURES.items():
    _fn = getattr(_L, _name)
    _fn.restype = _res
    _fn.argtypes = _args

lib = _L
PATH = LIB


class PactError(RuntimeError):
    """Raised for a non-zero pact_status; `.status` is the C code."""

    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status


def check(status: int) -> None:
    if status != 0:
        msg = _L.pact_last_error().decode(errors="replace")
        raise PactError(status, msg or _L.pact_status_name(status).decode())
