#!/usr/bin/env python
"""NCCL reduce-scatter / all-gather bus bandwidth on this box through torch.distributed (context for the
DP step's C1/C2; nccl-tests convention busBW = (P-1)/P * bytes / t). Run under torchrun."""
import os
import sys

import torch
import torch.distributed as dist


def main():
    rank, P = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
    sizes_mb = [float(x) for x in (sys.argv[1:] or ["8", "25.6", "51.2", "102.4", "256"])]
    for mb in sizes_mb:
        n = int(mb * 1e6) // 4 // P * P
        for name, dt in (("rs_f16", torch.float16), ("ag_f32", torch.float32)):
            elems = int(mb * 1e6) // (2 if dt == torch.float16 else 4) // P * P
            full = torch.ones(elems, dtype=dt, device="cuda")
            shard = torch.ones(elems // P, dtype=dt, device="cuda")
            op = (lambda: dist.reduce_scatter_tensor(shard, full)) if name.startswith("rs") else \
                (lambda: dist.all_gather_into_tensor(full, shard))
            for _ in range(5):
                op()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            it = 20
            for _ in range(it):
                op()
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / it * 1e-3
            bus = (P - 1) / P * full.numel() * full.element_size() / t / 1e9
            if rank == 0:
                print(f"P={P} {name} {full.numel() * full.element_size() / 1e6:8.1f} MB  {t * 1e6:8.1f} us  bus {bus:6.1f} GB/s",
                      flush=True)
        del n
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
