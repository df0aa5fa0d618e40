"""PyTorch DDP communication hook over the C-ABI.

PacTrain's integration point is a DDP comm hook (PAPER.md: the compressed
all-reduce replaces DDP's bucket all-reduce; the Mask Tracker maps DDP's
flattened buckets to parameter masks). This module is that adapter: the
per-step work of the reference trainer (trainer.cpp:369-377) expressed at
DDP bucket granularity:

* the model's trainable parameters are flattened in ``module.parameters()``
  order (the reference's ``flatten``, tensor.cpp:49-79) and one global mask
  is built over them (``prune``: build_prune_mask, trainer.cpp:340-352);
* each DDP bucket gets the sub-mask of its parameters, gathered on the
  device (``pact_mask_gather``) and cached until the mask or DDP's bucket
  assignment changes;
* per step the tracker observes the global mask once (trainer.cpp:373-376),
  and every bucket runs ``masked_allreduce`` (vote -> pack -> exchange ->
  unpack, or the dense fallback) with the mean (1/n) fused into the unpack,
  i.e. ``aggregate_step``'s ``to_mean`` (trainer.cpp:268-273). The bucket's
  gradient is not pre-masked: the packed path reads only kept values and
  writes +0 elsewhere, and the dense fallback applies GSE first
  (``SyncPolicy.gse_dense``), so the result equals GSE-then-aggregate;
* before a mask exists (dense warm-up) buckets take ``full_allreduce``.

The hook returns an already-completed future: every operation is enqueued on
the current CUDA stream, which is the stream DDP consumes the result on.
"""
import dataclasses
from collections import Counter
from typing import Dict, List, Optional, Sequence, Tuple

import torch
import torch.distributed as dist

from .api import (Comm, Errc, Error, MaskTracker, SparsityMask, SyncMode, SyncPolicy, SyncStats,
                  TrackerStatus, enforce_gradient_sparsity, full_allreduce, magnitude_prune,
                  magnitude_prune_per_layer, mask_gather, masked_allreduce)


def flat_layout(params: Sequence[torch.Tensor]) -> Tuple[Dict[int, Tuple[int, int]], int]:
    """id(param) -> (offset, numel) in the flattened parameter vector."""
    out, off = {}, 0
    for p in params:
        out[id(p)] = (off, p.numel())
        off += p.numel()
    return out, off


def bucket_segments(layout: Dict[int, Tuple[int, int]], bucket) -> List[Tuple[int, int]]:
    """(flat offset, length) of every parameter of a DDP GradBucket, in bucket
    buffer order. The per-parameter gradients must tile the bucket buffer
    contiguously (DDP's bucket views); anything else is a ShapeMismatch."""
    buf = bucket.buffer()
    base = buf.storage_offset()
    segs, expected = [], 0
    for p, g in zip(bucket.parameters(), bucket.gradients()):
        if id(p) not in layout:
            raise Error(Errc.ShapeMismatch, "bucket parameter is not part of the hook's flattened model")
        at = g.storage_offset() - base
        if at != expected:
            raise Error(Errc.ShapeMismatch, f"bucket gradient view at {at}, expected {expected}")
        off, n = layout[id(p)]
        if n != g.numel():
            raise Error(Errc.ShapeMismatch, "bucket gradient size differs from its parameter")
        if segs and segs[-1][0] + segs[-1][1] == off:
            segs[-1] = (segs[-1][0], segs[-1][1] + n)  # merge adjacent runs
        else:
            segs.append((off, n))
        expected += n
    if expected != buf.numel():
        raise Error(Errc.ShapeMismatch, f"bucket views cover {expected} of {buf.numel()} elements")
    return segs


class PactHookState:
    """State of :func:`pact_hook` (one per DDP model and rank)."""

    def __init__(self, module: torch.nn.Module, process_group=None, stability_threshold: int = 3,
                 policy: Optional[SyncPolicy] = None, comm: Optional[Comm] = None,
                 auto_density: bool = False):
        self.params = [p for p in module.parameters() if p.requires_grad]
        self.layout, self.length = flat_layout(self.params)
        self.group = process_group
        self.world = dist.get_world_size(process_group) if dist.is_initialized() else 1
        self._comm = comm
        self.tracker = MaskTracker(stability_threshold)
        self.policy = policy or SyncPolicy()
        self.mask: Optional[SparsityMask] = None
        self.epoch = 0
        self.step = 0
        self._observed_step = -1
        self._status = TrackerStatus.Unstable
        self._version = 0
        self._bucket_masks: Dict[int, Tuple[int, Tuple[Tuple[int, int], ...], SparsityMask]] = {}
        self.last_stats: Dict[int, SyncStats] = {}
        self.mode_counts: Counter = Counter()
        # adaptive policy (north_star (4)): the dense/sparse crossover measured
        # once per bucket length on this communicator (collective: DDP calls
        # the hook for the same buckets in the same order on every rank)
        self.auto_density = auto_density
        self.density_thresholds: Dict[int, float] = {}

    def density_threshold(self, length: int) -> float:
        # pact_calibrate_density needs len >= 1024: tiny buckets keep the
        # policy's static threshold (identical on every rank: no collective)
        if not self.auto_density or self.comm() is None or length < 1024:
            return self.policy.density_threshold
        if length not in self.density_thresholds:
            from .api import calibrate_density
            self.density_thresholds[length] = calibrate_density(length, self.comm(), policy=self.policy).threshold
        return self.density_thresholds[length]

    # -- communicator (created on first use: needs the GPU and the group)
    def comm(self) -> Optional[Comm]:
        if self._comm is None and self.world > 1:
            self._comm = Comm.from_process_group(self.group)
        return self._comm

    # -- the flattened model (tensor.cpp:49-79)
    def flat_weights(self) -> torch.Tensor:
        return torch.cat([p.detach().reshape(-1).float() for p in self.params])

    def layer_offsets(self) -> List[int]:
        offs = [0]
        for p in self.params:
            offs.append(offs[-1] + p.numel())
        return offs

    def _scatter_flat(self, flat: torch.Tensor) -> None:
        with torch.no_grad():
            for p in self.params:
                off, n = self.layout[id(p)]
                p.copy_(flat[off:off + n].view_as(p))

    # -- mask lifecycle
    def prune(self, ratio: float, per_layer: bool = False) -> SparsityMask:
        """trainer.cpp:340-352: mask from the flattened weights (global
        threshold, or per layer), then the pruned weights are zeroed. Every
        rank must hold the same weights (DDP broadcasts them at wrap time)."""
        flat = self.flat_weights()
        if per_layer:
            mask = magnitude_prune_per_layer(flat, self.layer_offsets(), ratio)
        else:
            mask = magnitude_prune(flat, ratio)
        self.set_mask(mask)
        self.enforce_weights()
        return mask

    def set_mask(self, mask: Optional[SparsityMask]) -> None:
        if mask is not None and mask.size() != self.length:
            raise Error(Errc.ShapeMismatch, f"mask of {mask.size()} bits for {self.length} parameters")
        self.mask = mask
        self._version += 1
        self._bucket_masks.clear()

    def enforce_weights(self) -> None:
        """sgd_step's masked-weight rule (trainer.cpp:202-214): weights at
        cleared bits are forced to +0.0f. Call after ``optimizer.step()``."""
        if self.mask is None:
            return
        flat = self.flat_weights()
        enforce_gradient_sparsity(flat, self.mask, out=flat)
        self._scatter_flat(flat)

    def bucket_mask(self, bucket) -> SparsityMask:
        segs = tuple(bucket_segments(self.layout, bucket))
        hit = self._bucket_masks.get(bucket.index())
        if hit is not None and hit[0] == self._version and hit[1] == segs:
            return hit[2]
        m = mask_gather(self.mask, segs)
        self._bucket_masks[bucket.index()] = (self._version, segs, m)
        return m

    def _observe(self) -> TrackerStatus:
        if self._observed_step != self.step:  # once per step, like the trainer
            self._status = (self.tracker.observe(self.mask) if self.mask is not None
                            else TrackerStatus.Unstable)
            self._observed_step = self.step
        return self._status


def pact_hook(state: PactHookState, bucket: dist.GradBucket) -> torch.futures.Future[torch.Tensor]:
    """DDP comm hook: the bucket's MEAN gradient via PacTrain's masked
    all-reduce (``model.register_comm_hook(state, pact_hook)``)."""
    buf = bucket.buffer()
    if buf.dtype != torch.float32:
        raise Error(Errc.ShapeMismatch, f"pact_hook needs fp32 gradients, got {buf.dtype}")
    status = state._observe()
    comm = state.comm()
    inv_n = 1.0 / float(state.world)
    if state.mask is None:
        if comm is not None:
            r = full_allreduce(buf, comm, scale=inv_n, out=buf)
            stats = r.stats
        else:
            stats = SyncStats(0, 0.0, SyncMode.FullAllReduce)
    else:
        pol = dataclasses.replace(state.policy, scale=inv_n, gse_dense=True,
                                  density_threshold=state.density_threshold(buf.numel()))
        r = masked_allreduce(buf, state.bucket_mask(bucket), status, state.epoch, comm, policy=pol, out=buf)
        stats = r.stats
    state.last_stats[bucket.index()] = stats
    state.mode_counts[stats.mode_used] += 1
    if bucket.is_last():
        state.step += 1
    fut = torch.futures.Future(devices=[buf.device])
    fut.set_result(buf)
    return fut
