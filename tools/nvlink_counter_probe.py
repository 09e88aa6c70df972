"""Which NVLink traffic counters can this box read? Runs a 1 GiB peer copy GPU0 -> GPU1 between two
readings of every candidate (NVML field values per link, GPM metrics, nvidia-smi nvlink -gt d)."""
import json
import subprocess
import time

import pynvml as nv
import torch

nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(0)
links = [l for l in range(nv.NVML_NVLINK_MAX_LINKS) if _ok] if False else []
for l in range(nv.NVML_NVLINK_MAX_LINKS):
    try:
        if nv.nvmlDeviceGetNvLinkState(h, l) == nv.NVML_FEATURE_ENABLED:
            links.append(l)
    except Exception:
        pass
out = {"links": links}


def fields(fid):
    res = {}
    for scope in ([0xFFFFFFFF] + links[:2]):
        try:
            v = nv.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
            res[str(scope)] = (v.nvmlReturn, int(v.value.ullVal))
        except Exception as e:
            res[str(scope)] = str(e)[:80]
    return res


def smi():
    try:
        return subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", "0"], capture_output=True, text=True,
                              timeout=20).stdout[-600:]
    except Exception as e:
        return str(e)


cands = {n: getattr(nv, n) for n in dir(nv) if n.startswith("NVML_FI_DEV_NVLINK") and
         any(k in n for k in ("BYTES", "THROUGHPUT", "COUNT_XMIT", "COUNT_RCV"))}
before = {n: fields(f) for n, f in cands.items()}
s0 = smi()
gpm = {}
try:
    samp0 = nv.nvmlGpmSampleAlloc()
    samp1 = nv.nvmlGpmSampleAlloc()
    nv.nvmlGpmSampleGet(h, samp0)
    gpm["alloc"] = "ok"
except Exception as e:
    gpm["alloc"] = str(e)[:120]
a = torch.empty(1 << 29, dtype=torch.int16, device="cuda:0")
b = torch.empty_like(a, device="cuda:1")
t0 = time.time()
for _ in range(4):
    b.copy_(a)
torch.cuda.synchronize(0)
torch.cuda.synchronize(1)
t1 = time.time()
after = {n: fields(f) for n, f in cands.items()}
s1 = smi()
try:
    nv.nvmlGpmSampleGet(h, samp1)
    mg = nv.c_nvmlGpmMetricsGet_t()
    mg.version = nv.NVML_GPM_METRICS_GET_VERSION
    mg.numMetrics = 2
    mg.sample1 = samp0
    mg.sample2 = samp1
    mg.metrics[0].metricId = nv.NVML_GPM_METRIC_NVLINK_TOTAL_TX_PER_SEC
    mg.metrics[1].metricId = nv.NVML_GPM_METRIC_NVLINK_TOTAL_RX_PER_SEC
    nv.nvmlGpmMetricsGet(mg)
    gpm["tx_per_sec"] = mg.metrics[0].value
    gpm["rx_per_sec"] = mg.metrics[1].value
except Exception as e:
    gpm["get"] = f"{type(e).__name__}: {e}"[:200]
out["copied_bytes"] = 4 * a.numel() * 2
out["seconds"] = t1 - t0
out["fields_before"] = before
out["fields_after"] = after
out["gpm"] = gpm
out["smi_before"] = s0
out["smi_after"] = s1
print(json.dumps(out, indent=1, default=str))
