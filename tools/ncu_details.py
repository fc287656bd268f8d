#!/usr/bin/env python
"""Print selected ncu 'details' sections for kernels matching a substring."""
import csv, io, subprocess, sys
rep, pat = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
secs = set(sys.argv[3].split(",")) if len(sys.argv) > 3 else {"GPU Speed Of Light Throughput", "Scheduler Statistics", "Warp State Statistics", "Occupancy", "Memory Workload Analysis"}
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
seen = set()
for r in rows[1:]:
    if pat in r[4] and r[h.index("Section Name")] in secs:
        key = (r[0], r[h.index("Metric Name")])
        if key in seen: continue
        seen.add(key)
        print(r[0], r[4][:28], "|", r[h.index("Section Name")][:18], "|", r[h.index("Metric Name")], "=", r[h.index("Metric Value")], r[h.index("Metric Unit")])
