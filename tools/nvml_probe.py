"""Which NVML NVLink counters this driver exposes on this GPU (B200): field
values (per-link byte counters, aggregate throughput fields) and GPM
(NVLink TX/RX rates), read around 10 GPU0 -> GPU1 copies of 1 GiB."""
import time

import pynvml as nv
import torch

nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(0)
print("driver", nv.nvmlSystemGetDriverVersion(), "name", nv.nvmlDeviceGetName(h))


def fields():
    out = {}
    for name in ["NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX", "NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX",
                 "NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX", "NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_RX",
                 "NVML_FI_DEV_NVLINK_LINK_COUNT"]:
        fid = getattr(nv, name, None)
        if fid is None:
            continue
        for scope in (None, 0, 0xFFFFFFFF):
            try:
                v = nv.nvmlDeviceGetFieldValues(h, [fid if scope is None else (fid, scope)])[0]
                out[f"{name}[{scope}]"] = (v.nvmlReturn, v.value.ullVal)
            except Exception as e:
                out[f"{name}[{scope}]"] = ("exc", str(e))
    for name in ["NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES", "NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES"]:
        fid = getattr(nv, name)
        tot, rets = 0, set()
        for l in range(18):
            try:
                v = nv.nvmlDeviceGetFieldValues(h, [(fid, l)])[0]
                rets.add(v.nvmlReturn)
                if v.nvmlReturn == 0:
                    tot += v.value.ullVal
            except Exception as e:
                rets.add(str(e))
        out[name] = (sorted(map(str, rets)), tot)
    return out


def gpm_sample():
    try:
        s = nv.nvmlGpmSampleAlloc()
        nv.nvmlGpmSampleGet(h, s)
        return s
    except Exception as e:
        print("GPM sample failed:", e)
        return None


a = torch.empty(1 << 28, dtype=torch.float32, device="cuda:0")
b = torch.empty(1 << 28, dtype=torch.float32, device="cuda:1")
f0 = fields()
g0 = gpm_sample()
t0 = time.time()
for _ in range(10):
    b.copy_(a)
torch.cuda.synchronize(0)
torch.cuda.synchronize(1)
dt = time.time() - t0
g1 = gpm_sample()
f1 = fields()
print(f"10 x 1 GiB GPU0 -> GPU1 in {dt * 1e3:.1f} ms")
for k in f0:
    print(k, f0[k], f1[k])
if g0 is not None and g1 is not None:
    try:
        md = nv.c_nvmlGpmMetricsGet_t()
        md.version = nv.NVML_GPM_METRICS_GET_VERSION
        md.sample1 = g0
        md.sample2 = g1
        ids = [getattr(nv, n) for n in dir(nv) if n.startswith("NVML_GPM_METRIC_NVLINK_TOTAL")]
        md.numMetrics = len(ids)
        for i, m in enumerate(ids):
            md.metrics[i].metricId = m
        nv.nvmlGpmMetricsGet(md)
        for i in range(md.numMetrics):
            print("GPM", md.metrics[i].metricId, md.metrics[i].nvmlReturn, md.metrics[i].value)
    except Exception as e:
        print("GPM metrics failed:", e)
