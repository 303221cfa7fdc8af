"""GPM counters (NVML GPU Performance Monitoring) around a workload: SM
utilisation, DRAM bandwidth utilisation, NVLink TX/RX — the counters the
multi-GPU bench reports for each path (ncu cannot run under torchrun)."""
import os
import sys
import time

import pynvml
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_06605_b200 as cc  # noqa: E402

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
try:
    sup = pynvml.nvmlGpmQueryDeviceSupport(h)
    print("gpm supported:", sup.isSupportedDevice)
except Exception as e:  # noqa: BLE001
    print("gpm query failed:", e)
METRICS = {"sm_util_pct": pynvml.NVML_GPM_METRIC_SM_UTIL, "dram_bw_util_pct": pynvml.NVML_GPM_METRIC_DRAM_BW_UTIL,
           "nvlink_tx_MiBps": pynvml.NVML_GPM_METRIC_NVLINK_TOTAL_TX_PER_SEC,
           "nvlink_rx_MiBps": pynvml.NVML_GPM_METRIC_NVLINK_TOTAL_RX_PER_SEC}


def measure(fn, seconds=0.5):
    s1, s2 = pynvml.nvmlGpmSampleAlloc(), pynvml.nvmlGpmSampleAlloc()
    torch.cuda.synchronize()
    pynvml.nvmlGpmSampleGet(h, s1)
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        fn()
        torch.cuda.synchronize()
    pynvml.nvmlGpmSampleGet(h, s2)
    mg = pynvml.c_nvmlGpmMetricsGet_t()
    mg.version = pynvml.NVML_GPM_METRICS_GET_VERSION
    mg.numMetrics = len(METRICS)
    mg.sample1, mg.sample2 = s1, s2
    for i, m in enumerate(METRICS.values()):
        mg.metrics[i].metricId = m
    pynvml.nvmlGpmMetricsGet(mg)
    out = {k: (round(mg.metrics[i].value, 2) if mg.metrics[i].nvmlReturn == 0 else f"ret {mg.metrics[i].nvmlReturn}")
           for i, k in enumerate(METRICS)}
    pynvml.nvmlGpmSampleFree(s1)
    pynvml.nvmlGpmSampleFree(s2)
    return out


n, s = 8, 8 << 20
comms = cc.Comm.init_all([0] * n)
st = torch.cuda.Stream()
sends = [torch.empty(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)]
recvs = [torch.empty(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)]
for impl in ("sm", "b2b"):
    print(impl, measure(lambda: [cc.all_to_all(comms, sends, recvs, s, impl=impl, streams=st) for _ in range(20)]))
a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
print("gemm", measure(lambda: [torch.matmul(a, a) for _ in range(10)]))
print("idle", measure(lambda: time.sleep(0.05)))
cc.destroy_all(comms)
