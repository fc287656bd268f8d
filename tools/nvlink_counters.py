"""NVLink hardware byte counters through NVML (not product code; bench.py and tools use it at P > 1).

ncu cannot profile a kernel that waits on another rank (its replays would deadlock the barrier), so the
bytes the fused F1/F2 kernels move over NVLink are read from the GPU's own link counters around a run of
steps: NVML field values NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX / _RX (payload KiB, per link; scope = link
id) and, if those are unsupported, NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES / _RCV_BYTES.
"""
from __future__ import annotations

FI_DATA_TX, FI_DATA_RX = 138, 139   # NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_{TX,RX}: KiB
FI_XMIT_BYTES, FI_RCV_BYTES = 202, 204  # NVML_FI_DEV_NVLINK_COUNT_{XMIT,RCV}_BYTES: bytes
MAX_LINKS = 18


class NvlinkCounters:
    """read() -> {"tx": bytes, "rx": bytes, "source": field names} summed over the GPU's links."""

    def __init__(self, index: int):
        import pynvml as N

        self.N = N
        N.nvmlInit()
        self.h = N.nvmlDeviceGetHandleByIndex(index)
        self.links = []
        for link in range(MAX_LINKS):
            try:
                if N.nvmlDeviceGetNvLinkState(self.h, link) == N.NVML_FEATURE_ENABLED:
                    self.links.append(link)
            except N.NVMLError:
                break
        self.mode = None
        for mode, (ftx, frx, scale) in (("throughput_data_KiB", (FI_DATA_TX, FI_DATA_RX, 1024)),
                                        ("count_bytes", (FI_XMIT_BYTES, FI_RCV_BYTES, 1))):
            if self._query(ftx, frx, scale) is not None:
                self.mode, self.f = mode, (ftx, frx, scale)
                break

    def _query(self, ftx, frx, scale):
        if not self.links:
            return None
        N = self.N
        ids = [(ftx, ln) for ln in self.links] + [(frx, ln) for ln in self.links]
        try:
            vals = N.nvmlDeviceGetFieldValues(self.h, ids)
        except N.NVMLError:
            return None
        tot = [0, 0]
        for k, v in enumerate(vals):
            if v.nvmlReturn != 0:
                return None
            x = v.value.ullVal if v.valueType == N.NVML_VALUE_TYPE_UNSIGNED_LONG_LONG else v.value.uiVal
            tot[0 if k < len(self.links) else 1] += int(x) * scale
        return tot

    def read(self):
        if self.mode is None:
            return None
        tx, rx = self._query(*self.f)
        return {"tx": tx, "rx": rx}

    def available(self) -> bool:
        return self.mode is not None

    def describe(self) -> str:
        return f"NVML {self.mode} over {len(self.links)} active links" if self.mode else "unavailable"
