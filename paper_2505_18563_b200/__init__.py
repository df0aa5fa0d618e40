"""B200-native PacTrain gradient-sync hot path.

magnitude prune -> mask bitmap -> pack -> NCCL allreduce -> unpack, with the
reference's adaptive dense/sparse policy, behind the C-ABI in
include/pact_c.h (sm_100a kernels in csrc/). This package is the Python host
mirror of the reference operator API; see api.py for the names.
"""
from .api import (  # noqa: F401
    AggregateResult,
    Comm,
    Context,
    Errc,
    Error,
    FrameHeader,
    MaskTracker,
    PackedGradient,
    PayloadKind,
    PruneConfig,
    SparsityMask,
    SyncMode,
    SyncPolicy,
    SyncStats,
    TernaryGradient,
    TrackerStatus,
    allgather,
    build_prune_mask,
    decide_sync_mode,
    decode_header,
    decode_ternary,
    deternarize,
    drop_count,
    encode_header,
    encode_ternary,
    enforce_gradient_sparsity,
    fp16_allreduce,
    fp16_roundtrip,
    full_allreduce,
    magnitude_prune,
    magnitude_prune_per_layer,
    mask_gather,
    mask_digest,
    masked_allreduce,
    masked_allreduce_host,
    masked_bytes,
    pack,
    ring_allreduce,
    ring_bytes,
    synth_fill,
    ternarize,
    ternary_allgather_aggregate,
    tracker_observe,
    unpack,
    unpack_sgd,
    vote_decide,
)

__all__ = [n for n in dir() if not n.startswith("_")]
