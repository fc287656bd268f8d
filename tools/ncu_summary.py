#!/usr/bin/env python
"""Summarise an ncu report (raw page) into the per-kernel numbers the bench/roofline uses."""
import csv
import io
import json
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct", "launch__grid_size",
        "launch__block_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__occupancy_limit_registers", "sm__maximum_warps_per_active_cycle_pct"]
SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "us": 1e-6, "ns": 1e-9, "ms": 1e-3}


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                u = units[i]
                if u in SCALE:
                    v *= SCALE[u]
                    w = w + ("[s]" if u in ("us", "ns", "ms") else "[B]")
                d[w] = v
        if "gpu__time_duration.sum[s]" in d and "dram__bytes_read.sum[B]" in d:
            d["dram_GBps"] = (d["dram__bytes_read.sum[B]"] + d["dram__bytes_write.sum[B]"]) / d["gpu__time_duration.sum[s]"] / 1e9
        res.append(d)
    return res


if __name__ == "__main__":
    print(json.dumps(summarise(sys.argv[1]), indent=1))
