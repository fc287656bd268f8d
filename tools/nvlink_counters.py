"""NVLink hardware traffic counters through NVML (not product code; bench.py uses it at P > 1).

ncu cannot profile a kernel that waits on another rank (its replays would deadlock the barrier), so the
bytes the fused F1/F2 kernels move over NVLink are read from the GPU's own counters around a run of steps:
  * GPM (GPU performance monitoring, Hopper and later): NVML_GPM_METRIC_NVLINK_TOTAL_{RX,TX}_PER_SEC between
    two GPM samples (MiB/s averaged over the interval) x the interval; or
  * the per-link field values NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_{TX,RX} (KiB) where supported.
On this pool's B200s the field values answer NVML_ERROR_NOT_SUPPORTED; GPM is tried first.
"""
from __future__ import annotations

import time

FI_DATA_TX, FI_DATA_RX = 138, 139   # NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_{TX,RX}: KiB
MAX_LINKS = 18


class NvlinkCounters:
    """start(); ...; stop() -> {"tx": bytes, "rx": bytes, "seconds": s} over the interval, or None."""

    def __init__(self, index: int):
        import pynvml as N

        self.N = N
        N.nvmlInit()
        self.h = N.nvmlDeviceGetHandleByIndex(index)
        self.mode = None
        try:
            sup = N.nvmlGpmQueryDeviceSupport(self.h)
            if getattr(sup, "isSupportedDevice", 0):
                self.s1, self.s2 = N.nvmlGpmSampleAlloc(), N.nvmlGpmSampleAlloc()
                N.nvmlGpmSampleGet(self.h, self.s1)  # answers NVML_ERROR_UNKNOWN on some pools: then no GPM
                self.mode = "gpm"
        except Exception:  # noqa: BLE001 - evidence only
            self.mode = None
        if self.mode is None:
            self.links = []
            for link in range(MAX_LINKS):
                try:
                    if N.nvmlDeviceGetNvLinkState(self.h, link) == N.NVML_FEATURE_ENABLED:
                        self.links.append(link)
                except N.NVMLError:
                    break
            if self._fields() is not None:
                self.mode = "fields"

    def _fields(self):
        N = self.N
        if not self.links:
            return None
        ids = [(FI_DATA_TX, ln) for ln in self.links] + [(FI_DATA_RX, ln) for ln in self.links]
        try:
            vals = N.nvmlDeviceGetFieldValues(self.h, ids)
        except N.NVMLError:
            return None
        tot = [0, 0]
        for k, v in enumerate(vals):
            if v.nvmlReturn != 0:
                return None
            tot[0 if k < len(self.links) else 1] += int(v.value.ullVal) * 1024
        return tot

    def available(self) -> bool:
        return self.mode is not None

    def describe(self) -> str:
        return {"gpm": "NVML GPM NVLINK_TOTAL_{RX,TX}_PER_SEC x interval",
                "fields": "NVML NVLINK_THROUGHPUT_DATA_{TX,RX} field values"}.get(self.mode, "unavailable")

    def start(self):
        self.t0 = time.perf_counter()
        if self.mode == "gpm":
            self.N.nvmlGpmSampleGet(self.h, self.s1)
        elif self.mode == "fields":
            self.f0 = self._fields()

    def stop(self):
        dt = time.perf_counter() - self.t0
        N = self.N
        if self.mode == "gpm":
            N.nvmlGpmSampleGet(self.h, self.s2)
            mg = N.c_nvmlGpmMetricsGet_t()
            mg.version = N.NVML_GPM_METRICS_GET_VERSION
            mg.numMetrics = 2
            mg.sample1, mg.sample2 = self.s1, self.s2
            mg.metrics[0].metricId = N.NVML_GPM_METRIC_NVLINK_TOTAL_RX_PER_SEC
            mg.metrics[1].metricId = N.NVML_GPM_METRIC_NVLINK_TOTAL_TX_PER_SEC
            N.nvmlGpmMetricsGet(mg)
            if mg.metrics[0].nvmlReturn != 0 or mg.metrics[1].nvmlReturn != 0:
                return None
            mib = 1024 * 1024
            return {"rx": mg.metrics[0].value * mib * dt, "tx": mg.metrics[1].value * mib * dt, "seconds": dt,
                    "rx_GBps": mg.metrics[0].value * mib / 1e9, "tx_GBps": mg.metrics[1].value * mib / 1e9}
        if self.mode == "fields":
            f1 = self._fields()
            return {"tx": f1[0] - self.f0[0], "rx": f1[1] - self.f0[1], "seconds": dt}
        return None
