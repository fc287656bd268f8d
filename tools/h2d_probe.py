#!/usr/bin/env python
"""Host->device copy bandwidth from pinned memory placed on each NUMA node (diagnostic for bench.py's e2e)."""
import glob
import os

import torch


def node_cpus(node):
    txt = open(f"/sys/devices/system/node/node{node}/cpulist").read().strip()
    cpus = set()
    for part in txt.split(","):
        a, _, b = part.partition("-")
        cpus.update(range(int(a), int(b or a) + 1))
    return cpus


def gpu_node(dev=0):
    pr = torch.cuda.get_device_properties(dev)
    bus = f"{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
    p = f"/sys/bus/pci/devices/{bus}/numa_node"
    return int(open(p).read()) if os.path.exists(p) else -1


def bw(nbytes=102_228_224, reps=10):
    x = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    x.fill_(1)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        d.copy_(x, non_blocking=True)
        e0.record(s)
        for _ in range(reps):
            d.copy_(x, non_blocking=True)
        e1.record(s)
    s.synchronize()
    return nbytes * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9


torch.cuda.init()
nodes = sorted(int(p.split("node")[-1]) for p in glob.glob("/sys/devices/system/node/node[0-9]*"))
print("numa nodes", nodes, "gpu0 node", gpu_node(0), "affinity", len(os.sched_getaffinity(0)), "cpus")
print("default placement: %.1f GB/s" % bw())
orig = os.sched_getaffinity(0)
for n in nodes:
    cpus = node_cpus(n) & orig
    if not cpus:
        continue
    os.sched_setaffinity(0, cpus)
    print("pinned memory first-touched on node %d: %.1f GB/s" % (n, bw()))
os.sched_setaffinity(0, orig)
