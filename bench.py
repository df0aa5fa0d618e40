"""Benchmark of the PacTrain gradient-sync hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ours|reference]

Metric (BASELINE.json): dense-equivalent gradient-sync GB/s
    = 4 * len bytes of fp32 gradient / t_step      (per rank)
where a step is one pass of the hot path over one synthetic gradient:
magnitude re-prune of the current weights (config c5, the default: GPT-2-
medium shape, 354,823,168 elements, 90%) -> vote -> pack -> exchange ->
unpack (N > 1), or prune -> pack -> unpack (N = 1, no exchange).
Between timed steps (untimed) the weights evolve per SURVEY A.9: w <- GSE(w)
+ delta on the kept entries, fresh regrowth noise on the pruned ones, so every
step re-derives the mask from new weights. `value` is per rank (every rank
syncs a full model-sized gradient; weak scaling), `value_job` = N x value.
Inputs are HBM resident; the L2 is flushed before every timed step; timing
is CUDA events on the launching stream, max over ranks. `e2e` is the same
step through the host-buffer C-ABI call (pinned H2D of the gradient, D2H of
the result inside the timed region).

Multi-GPU: launched by the driver under torch.distributed.run, one process per
GPU; torch.distributed (nccl) carries the barrier / max-over-ranks plumbing and
the NCCL unique id; the collective itself is the library's own NCCL comm.

--impl reference times the reference's own CPU implementation (oracle/_ref,
compiled from /root/reference by oracle/Makefile) on the host cores, on rank 0;
that process never maps the product library (asserted).
"""
from __future__ import annotations

import argparse
import gc
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (model shape, prune ratio, re-prune per step, bucket bytes; 0 = the library's auto)
    "c1": ("resnet18", 0.9, False, 0),
    "c2": ("resnet50", 0.8, False, 0),
    "c3": ("vgg19", 0.95, False, 0),
    "c4": ("bert-base", 0.5, False, 0),
    "c5": ("gpt2-medium", 0.9, True, 0),
}
L2_FLUSH_BYTES = 512 << 20
HOST_GATE_CYCLES = 2_000_000  # ~1 ms at 1.965 GHz


def _synth_module():
    """synth.py loaded by file path: importing the package would map the
    product library, which the reference arm must not do."""
    import importlib.util

    spec = importlib.util.spec_from_file_location("_pact_synth_bench",
                                                  os.path.join(ROOT, "paper_2505_18563_b200", "synth.py"))
    m = importlib.util.module_from_spec(spec)
    sys.modules[spec.name] = m  # dataclasses look their module up
    spec.loader.exec_module(m)
    return m


def _assert_no_product_lib():
    try:
        with open("/proc/self/maps") as f:
            maps = f.read()
    except OSError:
        return
    assert "libpact_b200" not in maps, "the reference arm mapped the product library"


def workload_name(cfg, model, ratio, reprune):
    return (f"{cfg}:{model} fp32 grads, {int(round(ratio * 100))}% magnitude-pruned mask"
            + (", re-pruned every step" if reprune else ""))


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def nvlink_bytes(device: int):
    """This GPU's cumulative NVLink data bytes (tx, rx) from the NVML field
    counters -- hardware counters read without kernel replay, so they work
    across ranks (ncu cannot profile a multi-rank exchange). Tries the
    per-link byte counters first, then the aggregate KiB throughput fields;
    None when neither is available."""
    try:
        import pynvml as nv

        nv.nvmlInit()
        h = nv.nvmlDeviceGetHandleByIndex(device)
        ids = [(nv.NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES, l) for l in range(18)]
        ids += [(nv.NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES, l) for l in range(18)]
        vals = nv.nvmlDeviceGetFieldValues(h, ids)
        tx = [v.value.ullVal for v in vals[:18] if v.nvmlReturn == 0]
        rx = [v.value.ullVal for v in vals[18:] if v.nvmlReturn == 0]
        if tx and rx:
            return {"tx": sum(tx), "rx": sum(rx), "source": "NVML_FI_DEV_NVLINK_COUNT_{XMIT,RCV}_BYTES",
                    "links": len(tx)}
        vals = nv.nvmlDeviceGetFieldValues(h, [nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX,
                                               nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX])
        if all(v.nvmlReturn == 0 for v in vals):
            return {"tx": vals[0].value.ullVal * 1024, "rx": vals[1].value.ullVal * 1024,
                    "source": "NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_{TX,RX} (KiB)", "links": None}
    except Exception:
        pass
    return None


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device: int):
        self.samples = []
        self.reasons = 0
        self._stop = threading.Event()
        self.ok = False
        if os.environ.get("PACT_BENCH_NO_NVML"):  # A/B: host-side interference of the sampler
            self.max_mhz = None
            return
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml_unavailable"]}
        names = [n for b, n in self.REASONS.items() if self.reasons & b and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(self.samples)}


# ------------------------------------------------------------ reference


def run_reference(args, cfg):
    """The reference's own CPU path (oracle/_ref) on this host's cores, on the
    same workload: N = 1 -> per step the mask re-derivation (c5) plus the
    reference pack -> unpack over the full gradient on all host threads; N > 1
    -> the reference masked_allreduce over SimCluster with N worker threads."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import numpy as np

    import oracle

    synth = _synth_module()
    model, ratio, reprune, _ = CONFIGS[cfg]
    shape = synth.model_shape(model)
    n = shape.total
    R = oracle.ref()
    P = oracle.port()
    w = synth.weights_host(shape, 1234, synth.W_REAL)
    words = P.magnitude_prune(w, ratio)
    nnz = P.mask_nnz(words, n)
    nthreads = os.cpu_count() or 1
    nworkers = max(2, args.gpus)
    grads = [R.gse(synth.synth_host(n, synth.grad_seed(r, 0), synth.G_FULL), words) for r in range(max(1, args.gpus))]
    if args.gpus == 1:
        h = R.bench_create(grads[:1], words, slices=nthreads)
        fn = lambda: R.bench_pack_unpack(h)  # noqa: E731
        what = f"reference pack->unpack (codec.cpp:14-38) on {nthreads} thread slices of the full gradient"
        cores = nthreads
    else:
        h = R.bench_create(grads, words, slices=0)
        fn = lambda: R.bench_masked(h)  # noqa: E731
        what = f"reference masked_allreduce (collective.cpp:269-309, tracker Stable) over SimCluster, {nworkers} worker threads"
        cores = nworkers
    prune_note = ""
    t_prune = 0.0
    if reprune:
        # the reference's magnitude_prune is a std::stable_sort of the whole
        # index array (sparsity.cpp:44-59): ~2 minutes per call at 355M on one
        # core, so the mask re-derivation is charged at the oracle's O(n)
        # restatement of the same rule (bit-identical words, one thread),
        # timed over all the weights (median of 3) and added to every step so
        # the --steps run stays within minutes; the reference's own sort is
        # timed once on a 4 Mi-element slice for the record
        tp = []
        for _ in range(3):
            a = time.perf_counter()
            wd = P.magnitude_prune(w, ratio)
            tp.append(time.perf_counter() - a)
        assert np.array_equal(wd, words)
        t_prune = sorted(tp)[1]
        t_ref_sort = R.bench_prune(w[:1 << 22], ratio)
        prune_note = (f"; + the mask re-derivation per step: the oracle port's O(n) magnitude_prune over all {n} "
                      f"weights, {t_prune:.2f} s (1 thread, median of 3; the reference's stable_sort: "
                      f"{t_ref_sort:.2f} s per 4,194,304 weights)")
    step = fn
    _assert_no_product_lib()
    for _ in range(args.warmup):
        step()
    ts = [step() + t_prune for _ in range(args.steps)]
    R.bench_destroy(h)
    _assert_no_product_lib()
    t = sum(ts) / len(ts)
    value = 4.0 * n / t / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": workload_name(cfg, model, ratio, reprune), "len": n, "nnz": nnz, "ratio": ratio,
                   "reprune_per_step": reprune, "parallelism": f"dp{args.gpus}"},
        "value_job": round(value * args.gpus, 4),
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": cores, "kind": "reference",
                         "sample": what + prune_note + f"; {args.steps} steps, full {model} gradient per step"},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    _emit(line)


METRIC = "dense-equiv. gradient sync GB/s (prune+pack+allreduce+unpack)"


# ------------------------------------------------------------------ ours


def pcie_roofline(torch, gh, oh, dg, dout, stream, t_e2e):
    """The host-buffer path moves 4*len bytes each way over PCIe: its floor is
    one H2D and one D2H of the step's buffers running concurrently. Measured
    live on the same pinned buffers (two streams, median of 5)."""
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    ts = []
    for _ in range(6):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        s1.wait_stream(stream)
        s2.wait_stream(stream)
        with torch.cuda.stream(s1):
            dg.copy_(gh, non_blocking=True)
        with torch.cuda.stream(s2):
            oh.copy_(dout, non_blocking=True)
        stream.wait_stream(s1)
        stream.wait_stream(s2)
        b.record(stream)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    t_floor = statistics.median(ts[1:])
    return {"bound": "pcie", "floor_ms": round(t_floor * 1e3, 3),
            "peak_gbs_per_direction": round(dg.numel() * 4 / t_floor / 1e9, 2),
            "frac": round(t_floor / t_e2e, 4),
            "note": "floor = concurrent H2D + D2H of the step's pinned buffers, measured in this run"}


def cpu_baseline_sample(shape, ratio, words_np, n, w_host=None):
    """Reference CPU path on this host, bounded sample (rank 0, N=1 only):
    the reference pack -> unpack over the full gradient on all host threads,
    plus (re-pruning configs) the mask re-derivation by the oracle port's O(n)
    magnitude_prune on one thread (the reference's stable_sort takes minutes
    at this size)."""
    try:
        import oracle
        from paper_2505_18563_b200 import synth

        R = oracle.ref()
        P = oracle.port()
        kind = "reference"
    except Exception as e:  # pragma: no cover
        return {"value": None, "unit": "GB/s", "cores": 0, "kind": "unavailable", "sample": str(e)}
    nthreads = os.cpu_count() or 1
    g = R.gse(synth.synth_host(n, synth.grad_seed(0, 0), synth.G_FULL), words_np)
    h = R.bench_create([g], words_np, slices=nthreads)
    R.bench_pack_unpack(h)
    ts = []
    t0 = time.time()
    while time.time() - t0 < 10.0 and len(ts) < 50:
        ts.append(R.bench_pack_unpack(h))
    R.bench_destroy(h)
    t = statistics.median(ts)
    what = (f"reference pack->unpack (codec.cpp:14-38) over the full {shape.name} gradient, "
            f"{nthreads} thread slices, median of {len(ts)} runs (~10 s)")
    if w_host is not None:
        tp = []
        t0 = time.time()
        while time.time() - t0 < 15.0 and len(tp) < 3:
            a = time.perf_counter()
            P.magnitude_prune(w_host, ratio)
            tp.append(time.perf_counter() - a)
        t += statistics.median(tp)
        what += (f" + the mask re-derivation: oracle-port magnitude_prune (sparsity.cpp:44-59 restated, O(n), "
                 f"1 thread) over all {n} weights, median of {len(tp)}")
    return {"value": round(4.0 * n / t / 1e9, 4), "unit": "GB/s", "cores": nthreads, "kind": kind,
            "sample": what}


_JSON_OUT = None


def _emit(line):
    """The contract's one JSON line, on the process's original stdout."""
    out = _JSON_OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def _stdout_to_stderr():
    """Native libraries (NCCL's version banner under NCCL_DEBUG=VERSION, seen
    on stdout at communicator init despite NCCL_DEBUG_FILE) write to fd 1
    directly; point fd 1 at stderr for the whole run and keep a private copy
    of the original stdout for the JSON line."""
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)


def main():
    _stdout_to_stderr()
    # the image sets NCCL_DEBUG=VERSION: NCCL prints its version (and any
    # warnings) to stdout at communicator init; the contract is ONE JSON line
    # on stdout, so NCCL's log goes to stderr instead
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5", choices=sorted(CONFIGS))
    ap.add_argument("--ratio", type=float, default=None, help="override the config's prune ratio")
    ap.add_argument("--bucket-mb", type=float, default=None)
    ap.add_argument("--transport", default="auto", choices=["auto", "nccl", "p2p"],
                    help="packed exchange for N > 1: NCCL allreduce or the fused NVLink P2P path")
    ap.add_argument("--path", default="masked", choices=["masked", "ternary", "fp16", "fp16-packed", "topk", "sweep"],
                    help="masked: the headline (masked_allreduce); the others time the SURVEY 8f rows "
                         "on the same workload (ternary_allgather_aggregate, fp16_allreduce, "
                         "masked_allreduce on the binary16 wire, topk_allgather_aggregate)")
    ap.add_argument("--topk-rate", type=float, default=0.01)
    ap.add_argument("--prune", default="global", choices=["global", "per-layer"],
                    help="re-prune rule of the timed step: one global threshold (the reference's "
                         "magnitude_prune) or one threshold per layer (north_star (1), SURVEY D1)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    cfg = args.config
    if args.ratio is not None:
        m, _, rp, bb = CONFIGS[cfg]
        CONFIGS[cfg] = (m, args.ratio, rp, bb)
    if args.impl == "reference":
        return run_reference(args, cfg)

    import numpy as np
    import torch

    import paper_2505_18563_b200 as pb
    from paper_2505_18563_b200 import synth

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
        comm = pb.Comm.from_process_group()

    model, ratio, reprune, bucket = CONFIGS[cfg]
    if args.bucket_mb is not None:  # < 0: one bucket whatever the size (AUTO may pick several)
        bucket = int(args.bucket_mb * (1 << 20)) if args.bucket_mb >= 0 else (1 << 62)
    shape = synth.model_shape(model)
    n = shape.total
    ctx = pb.Context.get(local)
    stream = torch.cuda.current_stream()

    # inputs: identical weights on every rank (same seed) -> identical global mask
    weights = synth.weights_device(shape, 1234, synth.W_REAL, device=dev)
    if reprune and args.prune == "per-layer":  # the A.9 recipe then keeps the per-layer mask
        mask = pb.magnitude_prune_per_layer(weights, shape.offsets(), ratio)
    else:
        mask = pb.magnitude_prune(weights, ratio)
    nnz = mask.nnz()
    tracker = pb.MaskTracker(3)
    for _ in range(4):
        tracker.observe(mask)
    assert tracker.status() == pb.TrackerStatus.Stable
    grad = torch.empty(n, dtype=torch.float32, device=dev)
    pb.synth_fill(grad, synth.grad_seed(rank, 0), synth.G_FULL)
    pb.enforce_gradient_sparsity(grad, mask, out=grad)
    out = torch.empty_like(grad)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    flush_r = torch.zeros(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    flush_sink = torch.empty((), dtype=torch.float32, device=dev)

    def l2_flush():
        # write a 512 MiB buffer (evicts everything), then read another one so
        # the dirty lines are written back now, not inside the timed step
        flush.zero_()
        torch.sum(flush_r, dim=0, out=flush_sink)
    transport = {"auto": 0, "nccl": 1, "p2p": 2}[args.transport]
    policy = pb.SyncPolicy(bucket_bytes=bucket if world > 1 else 0, transport=transport)
    w_cur = weights.clone() if reprune else None
    pert = {}

    def expand_keep(m, out_u8):
        """mask words -> one byte per element (untimed bench plumbing)"""
        b = m.words().view(torch.uint8)
        sh = torch.arange(8, device=dev, dtype=torch.uint8)
        torch.bitwise_and(torch.bitwise_right_shift(b.view(-1, 1), sh), 1, out=out_u8.view(-1, 8))

    def perturb(t, kind="a9"):
        """SURVEY A.9 between timed steps (untimed, identical on every rank):
        kept weights drift (w + delta, |delta| <= 2^-14), pruned ones are
        replaced by fresh regrowth noise (|eps| <= 2^-20, far below any kept
        magnitude), so the mask is re-derived from new weights every step and
        normally reproduces. kind="drift": a dense update of every weight
        (|delta| <= 2^-17), which moves the threshold and flips elements near
        it. kind="regrow": 4096 pruned weights become large (a real change)."""
        if not pert:
            nb = ((n + 63) // 64) * 64
            pert["keep"] = torch.empty(nb, dtype=torch.uint8, device=dev)
            pert["a"] = torch.empty(n, dtype=torch.float32, device=dev)
            pert["b"] = torch.empty(n, dtype=torch.float32, device=dev)
        keep, ta, tb = pert["keep"], pert["a"], pert["b"]
        if kind == "drift":
            pb.synth_fill(ta, synth.derive_seed(0xD81F7, t), synth.W_REAL, 2.0 ** -17)
            w_cur.add_(ta)
            return
        expand_keep(mask, keep)
        kb = keep[:n].bool()
        if kind == "regrow":
            idx = torch.nonzero(~kb)[(t * 4096) % max(1, n - nnz - 4096):][:4096, 0]
            w_cur[idx] = 0.5
            return
        pb.synth_fill(ta, synth.derive_seed(0xA9D, t), synth.W_REAL, 2.0 ** -14)
        pb.synth_fill(tb, synth.derive_seed(0xA9E, t), synth.W_REAL, 2.0 ** -20)
        torch.add(w_cur, ta, out=ta)
        torch.where(kb, ta, tb, out=w_cur)

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def step(e):
        if reprune:  # c5: regenerate the mask from the current weights every step
            pb.magnitude_prune(w_cur, ratio, out=mask)
            tracker.observe(mask)
        return pb.masked_allreduce(grad, mask, tracker.status(), e, comm, policy=policy, out=out)

    align = torch.zeros(1, dtype=torch.float32, device=dev)

    def timed(fn, k, pre=None):
        """k device-timed calls, L2 flushed before each; returns seconds list.
        pre(i) runs (untimed) before call i. N > 1: a 1-element allreduce after
        the flush re-aligns the ranks on the device, so no step is
        charged for a peer's flush."""
        evs = []
        # no cyclic-GC pause inside a step: the prune's readback makes the
        # host part of the device timeline (collected before, re-enabled after)
        gc.collect()
        gc.disable()
        for i in range(k):
            if pre is not None:
                pre(i)
            l2_flush()
            if world > 1:
                torch.distributed.all_reduce(align)
            # host gate: a 1 ms device spin, so the step's launches (and the
            # host-side vote) are enqueued before the start event fires and a
            # host hiccup (GIL, the NVML sampler thread) never lands on the
            # device timeline -- the regime of a training loop, where the
            # host runs ahead of a busy GPU (e2e below keeps the host cost)
            torch.cuda._sleep(HOST_GATE_CYCLES)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn(i)
            b.record(stream)
            evs.append((a, b))
        torch.cuda.synchronize()
        gc.enable()
        return [a.elapsed_time(b) * 1e-3 for a, b in evs]

    if args.path == "sweep":
        return run_sweep(args, pb, torch, comm, rank, world, local, dev, cfg, model, n, weights, grad, out, timed)
    if args.path != "masked":
        return run_path(args, pb, torch, comm, rank, world, local, dev, cfg, model, ratio, shape, n, nnz, mask,
                        tracker, grad, out, timed, barrier)

    # ---- headline: device-resident step
    paths = {}

    layer_offs = shape.offsets()

    def step_h(e):
        if reprune:
            if args.prune == "per-layer":
                pb.magnitude_prune_per_layer(w_cur, layer_offs, ratio, out=mask)
                paths["per-layer"] = paths.get("per-layer", 0) + 1
            else:
                st = {}
                pb.magnitude_prune(w_cur, ratio, out=mask, stats=st)
                paths[st["path"]] = paths.get(st["path"], 0) + 1
            tracker.observe(mask)
        return pb.masked_allreduce(grad, mask, tracker.status(), e, comm, policy=policy, out=out)

    pre = perturb if reprune else None
    for i in range(args.warmup):
        if pre:
            pre(10_000 + i)
        r = step_h(i)
    assert r.stats.mode_used == pb.SyncMode.PackedAllReduce, r.stats
    paths.clear()
    barrier()
    pre_launches = [0]  # the untimed A.9 perturbation's own synth kernels are not step kernels

    def pre_counted(i):
        a = ctx.kernel_launches()
        pre(i)
        pre_launches[0] += ctx.kernel_launches() - a
    l0 = ctx.kernel_launches()
    with ClockSampler(local) as clk:
        barrier()
        ts = timed(step_h, args.steps, pre=pre_counted if pre else None)
        barrier()
    launches = ctx.kernel_launches() - l0 - pre_launches[0]
    assert r.stats.mode_used == pb.SyncMode.PackedAllReduce, r.stats
    t_step = sum(ts) / len(ts)
    qs = sorted(ts)
    pct = [qs[int(q * (len(qs) - 1))] for q in (0.1, 0.5, 0.9)]
    if world > 1:
        tt = torch.tensor([t_step] + pct, dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_step, pct = float(tt[0].item()), [float(x) for x in tt[1:].tolist()]
    step_dist = {"p10_us": round(pct[0] * 1e6, 1), "p50_us": round(pct[1] * 1e6, 1), "p90_us": round(pct[2] * 1e6, 1)}
    per_rank_gbs = 4.0 * n / t_step / 1e9
    value = per_rank_gbs

    # ---- dominant kernel roofline: pack and unpack timed alone (flushed)
    packed = torch.empty(max(1, nnz), dtype=torch.float32, device=dev)
    pk = pb.PackedGradient(mask.digest(), 0, packed[:nnz])
    t_pack = statistics.median(timed(lambda i: pb.api._call(
        pb.api.lib.pact_pack, ctx.handle, pb.api._ptr(grad), n, mask.handle, pb.api._ptr(packed), 0,
        pb.api.C.c_uint64(2**64 - 1), pb.api._stream()), max(10, args.steps)))
    t_unpack = statistics.median(timed(lambda i: pb.unpack(pk, mask, out=out), max(10, args.steps)))
    alg_pack = 4 * n + n / 8 + 4 * nnz
    alg_unpack = 4 * nnz + n / 8 + 4 * n
    stages = {"pack_us": round(t_pack * 1e6, 2), "unpack_us": round(t_unpack * 1e6, 2),
              "pack_gbs": round(alg_pack / t_pack / 1e9, 1), "unpack_gbs": round(alg_unpack / t_unpack / 1e9, 1)}
    # per-stage breakdown of the full step (events between the stages; untimed)
    pol_t = pb.SyncPolicy(bucket_bytes=policy.bucket_bytes, transport=policy.transport, time_stages=True)
    br = []
    for i in range(7):
        l2_flush()
        barrier()
        rr = pb.masked_allreduce(grad, mask, tracker.status(), i, comm, policy=pol_t, out=out)
        br.append((rr.stats.seconds, rr.stats.t_pack, rr.stats.t_exchange, rr.stats.t_unpack))
    if br and br[0][1] > 0:
        med = [statistics.median(x[k] for x in br) * 1e6 for k in range(4)]
        stages["step_breakdown_us"] = {"total": round(med[0], 1), "pack": round(med[1], 1),
                                       "exchange": round(med[2], 1), "unpack": round(med[3], 1),
                                       "transport": ["none", "nccl", "nvlink-p2p"][rr.stats.transport]}
        if rr.stats.transport == 2:  # the NVLink exchange is fused into pack and unpack: no stage of its own
            stages["step_breakdown_us"]["note"] = ("nvlink-p2p: the push is inside 'pack', the peer wait "
                                                   "and fold inside 'unpack'")
    if reprune:
        # the prune paths on their own (prune.cu; DESIGN 3a): threshold reuse,
        # A.9 (the headline's), a dense drift that moves the threshold and
        # flips elements (+ the digest the tracker then needs), a regrowth
        # that changes the mask, and the first-time sampled path
        alg_prune = 4 * n + n / 8
        pr = {}

        def prune_only(i):
            st = {}
            pb.magnitude_prune(w_cur, ratio, out=mask, stats=st)
            pr.setdefault("paths", []).append(st["path"])

        def prune_digest(i):
            prune_only(i)
            mask.digest()
        t_hit = statistics.median(timed(prune_only, 5))
        pr["paths"] = []
        t_a9 = statistics.median(timed(prune_only, 5, pre=lambda i: perturb(20_000 + i)))
        p_a9 = pr.pop("paths")
        # dense drift from the dense (never GSE'd) weights, on its own mask
        w_keep, mask_keep = w_cur, mask
        w_cur = weights.clone()
        mask = pb.magnitude_prune(w_cur, ratio)
        pb.magnitude_prune(w_cur, ratio, out=mask)
        t_drift = statistics.median(timed(prune_digest, 5, pre=lambda i: perturb(30_000 + i, "drift")))
        p_drift = pr.pop("paths")
        w_cur, mask = w_keep, mask_keep
        t_regrow = statistics.median(timed(prune_digest, 5, pre=lambda i: perturb(40_000 + i, "regrow")))
        p_regrow = pr.pop("paths")
        scratch = pb.SparsityMask(n)

        def prune_full(i):
            st = {}
            pb.magnitude_prune(w_cur, ratio, out=scratch, stats=st)
            pr.setdefault("paths", []).append(st["path"])
        prune_full(0)
        t_full = statistics.median(timed(prune_full, 3, pre=lambda i: pb.api._call(
            pb.api.lib.pact_mask_fill, scratch.handle, 0, pb.api._stream())))
        p_full = pr.pop("paths")
        # per-layer thresholds: every layer's own k-th key, all
        # layers at once (prune_seg.cu), against the global first-time prune
        fill = lambda i: pb.api._call(pb.api.lib.pact_mask_fill, scratch.handle, 0, pb.api._stream())  # noqa: E731
        t_layer = statistics.median(timed(lambda i: pb.magnitude_prune_per_layer(w_cur, layer_offs, ratio,
                                                                                 out=scratch), 3, pre=fill))
        # per-layer temporal reuse: every layer's previous threshold verified by one pass
        pb.magnitude_prune_per_layer(w_cur, layer_offs, ratio, out=scratch)
        t_layer_reuse = statistics.median(timed(lambda i: pb.magnitude_prune_per_layer(w_cur, layer_offs, ratio,
                                                                                       out=scratch), 5))
        del scratch
        # a whole step whose mask changed (regrowth), on the packed path
        # (the tracker would fall back to dense for K steps; this is the cost
        # of the mask regeneration itself) vs the headline's steady state
        def step_stable(e):
            pb.magnitude_prune(w_cur, ratio, out=mask)
            mask.digest()
            return pb.masked_allreduce(grad, mask, pb.TrackerStatus.Stable, e, comm, policy=policy, out=out)
        t_step_change = statistics.median(timed(step_stable, 5, pre=lambda i: perturb(50_000 + i, "regrow")))
        t_step_hit = statistics.median(timed(step_stable, 5))
        if world > 1:
            tt = torch.tensor([t_hit, t_a9, t_drift, t_regrow, t_full, t_step_change, t_step_hit, t_layer,
                               t_layer_reuse],
                              dtype=torch.float64, device=dev)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            t_hit, t_a9, t_drift, t_regrow, t_full, t_step_change, t_step_hit, t_layer, t_layer_reuse = tt.tolist()
        stages["prune"] = {
            "reuse_hit_us": round(t_hit * 1e6, 1), "reuse_hit_gbs": round(alg_prune / t_hit / 1e9, 1),
            "a9_us": round(t_a9 * 1e6, 1), "a9_paths": p_a9,
            "dense_drift_plus_digest_us": round(t_drift * 1e6, 1), "dense_drift_paths": p_drift,
            "regrowth_change_plus_digest_us": round(t_regrow * 1e6, 1), "regrowth_paths": p_regrow,
            "first_time_sampled_us": round(t_full * 1e6, 1), "first_time_paths": p_full,
            "per_layer_us": round(t_layer * 1e6, 1), "per_layer_layers": len(layer_offs) - 1,
            "per_layer_reuse_us": round(t_layer_reuse * 1e6, 1),
            "per_layer_vs_global_first_time": round(t_layer / t_full, 3),
            "paths_legend": "1 sampled window, 2 full radix, 3 threshold reuse, 4 moved threshold from window candidates",
        }
        stages["mask_change_step_us"] = round(t_step_change * 1e6, 1)
        stages["mask_reuse_step_us"] = round(t_step_hit * 1e6, 1)
        stages["mask_change_vs_reuse_step"] = round(t_step_change / t_step_hit, 3)
        # back to a stable tracker for the e2e leg
        for _ in range(4):
            pb.magnitude_prune(w_cur, ratio, out=mask)
            tracker.observe(mask)
    if t_pack >= t_unpack:
        dom, alg, tdom = "pack_lm_kernel<0>", alg_pack, t_pack
    else:
        # the launcher's two-runs-ahead variant on long grids (codec.cu,
        # kDeepUnpackChunksPerWarp x the one-ahead grid of 6 CTAs x 4 warps per SM)
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        ahead = 2 if (n + 1023) // 1024 >= 16 * sms * 6 * 4 else 1
        dom, alg, tdom = f"unpack_kernel<0, 0, {ahead}>", alg_unpack, t_unpack
    peak, peak_kind = peaks()
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:  # ncu's per-launch DRAM bytes of this kernel on this workload (tools/ncu_summary.py)
            traffic = json.load(open(tp)).get(f"{cfg}:{dom}")
        except Exception:
            traffic = None
    achieved = alg / tdom / 1e9
    roofline = {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic, "peak_kind": peak_kind,
                "algorithmic_bytes": int(alg)}

    # ---- allreduce context (N > 1): dense NCCL busbw in the same run
    extra = {}
    if world > 1:
        t_dense = statistics.median(timed(lambda i: pb.full_allreduce(grad, comm, out=out), 10))
        t_packed_ar = statistics.median(timed(lambda i: pb.ring_allreduce(packed, comm, out=packed), 10))
        f = 2 * (world - 1) / world
        # the exchange as the step pays for it: step time minus pack and
        # unpack timed alone (the P2P exchange is fused into them, so there
        # is no separate exchange kernel to time)
        t_x = max(t_step - t_pack - t_unpack - (t_a9 if reprune else 0.0), 1e-9)
        extra = {"dense_allreduce_us": round(t_dense * 1e6, 1),
                 "dense_busbw_gbs": round(4 * n * f / t_dense / 1e9, 1),
                 "packed_allreduce_us": round(t_packed_ar * 1e6, 1),
                 "packed_busbw_gbs": round(4 * nnz * f / t_packed_ar / 1e9, 1),
                 "step_exchange_us": round(t_x * 1e6, 1),
                 "step_exchange_busbw_gbs": round(4 * nnz * f / t_x / 1e9, 1),
                 "step_exchange_vs_dense_busbw": round((4 * nnz * f / t_x) / (4 * n * f / t_dense), 3),
                 # NVLink 5: 900 GB/s per direction per GPU nominal (north_star); the
                 # measured bidirectional SM-store rate is ~540 GB/s (tools/nvlink_probe.cu)
                 "nvlink_peak_gbs": 900.0,
                 "step_exchange_busbw_frac_of_nvlink": round(4 * nnz * f / t_x / 1e9 / 900.0, 3),
                 "dense_sync_equiv_gbs_per_rank": round(4 * n / t_dense / 1e9, 1)}
        # NVLink hardware counters around K exchanges of the step's mask
        # (this rank's bytes; the one-shot n = 2 push sends 4 nnz, a ring /
        # two-shot exchange 2 (n-1)/n 4 nnz per rank)
        nv0 = nvlink_bytes(local)
        if nv0 is not None:
            kx = 10
            torch.cuda.synchronize()
            barrier()
            nv0 = nvlink_bytes(local)
            for e in range(kx):
                r = pb.masked_allreduce(grad, mask, pb.TrackerStatus.Stable, 50_000 + e, comm, policy=policy, out=out)
            torch.cuda.synchronize()
            nv1 = nvlink_bytes(local)
            torch.cuda.synchronize()
            nvd0 = nvlink_bytes(local)
            for e in range(kx):
                pb.full_allreduce(grad, comm, out=out)
            torch.cuda.synchronize()
            nvd1 = nvlink_bytes(local)
            alg_x = 4 * nnz * (1.0 if (world == 2 and r.stats.transport == 2) else f)
            extra["nvlink_counters"] = {
                "source": nv0["source"], "links": nv0["links"], "steps": kx, "transport": int(r.stats.transport),
                "tx_bytes_per_exchange": int((nv1["tx"] - nv0["tx"]) / kx),
                "rx_bytes_per_exchange": int((nv1["rx"] - nv0["rx"]) / kx),
                "algorithmic_bytes_per_rank": int(alg_x),
                "tx_vs_algorithmic": round((nv1["tx"] - nv0["tx"]) / kx / alg_x, 3),
                "dense_tx_bytes_per_allreduce": int((nvd1["tx"] - nvd0["tx"]) / kx),
                "dense_algorithmic_bytes_per_rank": int(4 * n * f)}
        sb = stages.get("step_breakdown_us", {})
        bx = sb.get("exchange", 0.0) * 1e-6 if sb.get("transport") == "nccl" else 0.0
        if bx > 0:  # NCCL transport: the exchange timed directly inside the step (events around it)
            extra["exchange_in_step_us"] = round(bx * 1e6, 1)
            extra["exchange_in_step_busbw_gbs"] = round(4 * nnz * f / bx / 1e9, 1)
            extra["exchange_in_step_vs_dense_busbw"] = round((4 * nnz * f / bx) / (4 * n * f / t_dense), 3)

    # ---- e2e through the host-buffer C-ABI entry point
    e2e = None
    if not args.no_e2e:
        gh = grad.cpu().pin_memory()
        oh = torch.empty(n, dtype=torch.float32).pin_memory()

        def step_e2e(i):
            if reprune:  # the weights are model state on the device; the gradient comes from the host
                pb.magnitude_prune(w_cur, ratio, out=mask)
                tracker.observe(mask)
            return pb.masked_allreduce_host(gh, mask, tracker.status(), i, comm, oh, policy=policy)
        for i in range(2):
            step_e2e(i)
        barrier()
        te = []
        for i in range(max(5, min(args.steps, 20))):
            if reprune:
                perturb(60_000 + i)
            l2_flush()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            st_e = step_e2e(i)
            b.record(stream)
            b.synchronize()
            te.append(a.elapsed_time(b) * 1e-3)
        t_e2e = sum(te) / len(te)
        if world > 1:
            tt = torch.tensor([t_e2e], dtype=torch.float64, device=dev)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            t_e2e = float(tt.item())
        e2e = {"value": round(4.0 * n / t_e2e / 1e9, 3), "unit": "GB/s",
               "h2d_bytes_per_step": 4 * n, "d2h_bytes_per_step": 4 * n, "ms_per_step": round(t_e2e * 1e3, 3),
               "mode": "packed" if st_e.mode_used == pb.SyncMode.PackedAllReduce else "dense",
               "includes": "prune of the device weights + pact_masked_allreduce_host (pinned H2D of the "
                           "gradient, D2H of the result)" if reprune else "pact_masked_allreduce_host",
               "roofline": pcie_roofline(torch, gh, oh, grad, out, stream, t_e2e)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_sample(shape, ratio, mask.words_host(), n,
                                  w_cur.cpu().numpy() if reprune else None)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_step * 1e3, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "value_job": round(value * world, 2),
            "config": {"workload": workload_name(cfg, model, ratio, reprune)
                       + (", per-layer thresholds" if reprune and args.prune == "per-layer" else ""),
                       "len": n, "nnz": nnz, "ratio": ratio, "reprune_per_step": reprune,
                       "weights": "W-real (SURVEY A.9), identical on every rank",
                       "perturbation": ("A.9 between timed steps: kept w += delta (|delta| <= 2^-14), pruned "
                                        "w = fresh noise (|eps| <= 2^-20); prune paths taken: "
                                        + json.dumps({str(k): v for k, v in sorted(paths.items())}))
                       if reprune else None,
                       "l2": "flushed before every timed step (512 MiB write, then a 512 MiB read "
                             "so the flush's dirty lines are written back outside the timed region)",
                       "host_gate": "1 ms device spin before each timed step's start event (launches "
                                    "enqueued ahead; e2e keeps the host cost)",
                       "parallelism": f"dp{world}", "bucket_bytes": policy.bucket_bytes,
                       "transport": ["none", "nccl", "nvlink-p2p"][r.stats.transport],
                       "value_is": "per rank: 4*len / t_step (SURVEY 8(d)); value_job = n_gpus x value"},
            "step_distribution": step_dist,
            "roofline": roofline, "stages": stages, **({"allreduce": extra} if extra else {}),
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        _emit(line)
    if comm is not None:
        torch.distributed.barrier()
        comm.close()
        torch.distributed.destroy_process_group()


# BASELINE config 4 sweeps 50-99%; 0.05 and 0.1 (densities 0.95 / 0.9) are
# added so the measured dense/sparse crossover is crossed inside the sweep
SWEEP_RATIOS = (0.05, 0.1, 0.5, 0.6, 0.7, 0.8, 0.9, 0.95, 0.99)


def run_sweep(args, pb, torch, comm, rank, world, local, dev, cfg, model, n, weights, grad, out, timed):
    """BASELINE config 4: the sparsity sweep exercising the adaptive
    dense/sparse switch. The threshold is MEASURED (pact_calibrate_density on
    this communicator and length, synthetic inputs), then at each ratio the
    packed path, the dense path and the auto policy are timed on the
    workload's own mask (L2 flushed, CUDA events, max over ranks)."""
    cal = pb.calibrate_density(n, comm)
    auto = pb.SyncPolicy(density_threshold=cal.threshold)
    packed_pol, dense_pol = pb.SyncPolicy(), pb.SyncPolicy(density_threshold=1e-300)
    k = max(3, min(args.steps, 10))

    def tmax(x):
        if world > 1:
            tt = torch.tensor([x], dtype=torch.float64, device=dev)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            x = float(tt.item())
        return x

    rows, gbs = [], []
    for ratio in SWEEP_RATIOS:
        m = pb.magnitude_prune(weights, ratio)
        res = {}
        for name, pol in (("packed", packed_pol), ("dense", dense_pol), ("auto", auto)):
            def st(i, pol=pol):
                return pb.masked_allreduce(grad, m, pb.TrackerStatus.Stable, i, comm, policy=pol, out=out)
            for i in range(2):
                r = st(i)
            res[name] = (tmax(statistics.median(timed(st, k))), r.stats.mode_used)
        best = min(res["packed"][0], res["dense"][0])
        gbs.append(4.0 * n / res["auto"][0] / 1e9)
        rows.append({"ratio": ratio, "density": round(m.nnz() / n, 6),
                     "packed_us": round(res["packed"][0] * 1e6, 1), "dense_us": round(res["dense"][0] * 1e6, 1),
                     "auto_us": round(res["auto"][0] * 1e6, 1),
                     "auto_mode": "packed" if res["auto"][1] == pb.SyncMode.PackedAllReduce else "dense",
                     "auto_vs_best": round(res["auto"][0] / best, 3)})
    if rank == 0:
        geo = math.exp(sum(math.log(x) for x in gbs) / len(gbs))
        line = {
            "metric": METRIC.replace("prune+pack+allreduce+unpack", "adaptive policy sweep, geomean"),
            "value": round(geo, 2), "unit": "GB/s", "n_gpus": world, "steps": k, "warmup": 2,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "path": "sweep",
            "config": {"workload": f"{cfg}:{model} fp32 grads, magnitude masks at ratios {list(SWEEP_RATIOS)}",
                       "len": n, "l2": "flushed before every timed step", "parallelism": f"dp{world}"},
            "calibration": {"threshold_density": round(cal.threshold, 4), "probe_densities": cal.densities,
                            "t_packed_us": [round(t * 1e6, 1) for t in cal.t_packed],
                            "t_dense_us": round(cal.t_dense * 1e6, 1)},
            "sweep": rows,
        }
        _emit(line)
    if comm is not None:
        torch.distributed.barrier()
        comm.close()
        torch.distributed.destroy_process_group()


def run_path(args, pb, torch, comm, rank, world, local, dev, cfg, model, ratio, shape, n, nnz, mask, tracker,
             grad, out, timed, barrier):
    """The SURVEY 8f rows on the headline workload: one step = one call of the
    path's aggregate over the model-sized gradient (inputs HBM resident, L2
    flushed, CUDA events, max over ranks). `roofline` is the whole step's
    algorithmic HBM bytes (per kernel) over its time."""
    from paper_2505_18563_b200 import synth

    k = pb.topk_count(n, args.topk_rate)
    seed = synth.grad_seed(rank, 7)
    if args.path == "ternary":
        def step(e):
            return pb.ternary_allgather_aggregate(grad, mask, pb.TrackerStatus.Stable, seed + e, e, comm, out=out)
        mode = pb.SyncMode.TernaryAllGather
        # pack, absmax, ternarize, mean over n blocks, unpack
        alg = (4 * n + n / 8 + 4 * nnz) + 4 * nnz + (4 * nnz + nnz / 4) + (world * nnz / 4 + 4 * nnz) + \
              (4 * nnz + n / 8 + 4 * n)
    elif args.path == "fp16":
        def step(e):
            return pb.fp16_allreduce(grad, comm, out=out)
        mode = pb.SyncMode.Fp16AllReduce
        c = n / world  # encode + (n-1) steps + gather (decode into the full output)
        alg = (4 * c + 2 * c) + (world - 1) * (4 * c + 2 * c + 2 * c) + (2 * n + 4 * n) if world > 1 else 8 * n
    elif args.path == "fp16-packed":
        pol = pb.SyncPolicy(wire=pb.SyncPolicy.F16)

        def step(e):
            return pb.masked_allreduce(grad, mask, pb.TrackerStatus.Stable, e, comm, policy=pol, out=out)
        mode = pb.SyncMode.PackedAllReduce
        c = nnz / world
        ring = ((4 * c + 2 * c) + (world - 1) * (4 * c + 2 * c + 2 * c) + (2 * nnz + 4 * nnz)) if world > 1 \
            else 8 * nnz
        alg = (4 * n + n / 8 + 4 * nnz) + ring + (4 * nnz + n / 8 + 4 * n)
    else:  # topk
        def step(e):
            return pb.topk_allgather_aggregate(grad, args.topk_rate, e, comm, out=out)
        mode = pb.SyncMode.TopKAllGather
        # threshold (sample + count reads), bitmap, pack values + indices,
        # f64 zero + n scatter-adds + mean
        alg = 4 * n + (4 * n + n / 8) + (4 * n + n / 8 + 4 * k) + (n / 8 + 4 * k) + 8 * n + \
              world * (8 * k + 16 * k) + (8 * n + 4 * n)
    for i in range(args.warmup):
        r = step(i)
    assert r.stats.mode_used == mode, r.stats
    barrier()
    ctx = pb.Context.get(local)
    l0 = ctx.kernel_launches()
    with ClockSampler(local) as clk:
        barrier()
        ts = timed(step, args.steps)
        barrier()
    launches = ctx.kernel_launches() - l0
    t_step = sum(ts) / len(ts)
    if world > 1:
        tt = torch.tensor([t_step], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_step = float(tt.item())
    peak, peak_kind = peaks()
    achieved = alg / t_step / 1e9
    if rank == 0:
        line = {
            "metric": METRIC.replace("prune+pack+allreduce+unpack", args.path + " aggregate"),
            "value": round(4.0 * n / t_step / 1e9, 2), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_step * 1e3, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "path": args.path,
            "config": {"workload": f"{cfg}:{model} fp32 grads, {int(round(ratio * 100))}% magnitude-pruned mask",
                       "len": n, "nnz": nnz, "topk_k": k if args.path == "topk" else None,
                       "l2": "flushed before every timed step", "parallelism": f"dp{world}",
                       "bytes_on_wire": r.stats.bytes_on_wire},
            "roofline": {"bound": "hbm", "kernel": "whole step", "achieved": round(achieved, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": None,
                         "peak_kind": peak_kind, "algorithmic_bytes": int(alg)},
            "gpu_launches": int(launches), "clocks": clk.summary(),
        }
        _emit(line)
    if comm is not None:
        torch.distributed.barrier()
        comm.close()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
