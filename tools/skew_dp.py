#!/usr/bin/env python
"""configs[4] at P > 1 (torchrun, one process per GPU): the 10^9-parameter, 1,000-tensor skewed layouts on the
data-parallel step with fp16 gradients — fused NVLink path (default contiguous shards: huge layers split
across ranks and finished through the share exchange) and the NCCL path — step time, bus GB/s per rank
((P-1)/P * (2 + 4) B per parameter) and its fraction of the 770 GB/s per-direction peer copy. CUDA events on
the launching stream, max over ranks; one JSON line per variant from rank 0."""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
NVLINK_PEER_GBS = 770.0


def main():
    import torch
    import torch.distributed as dist

    import paper_1903_12650_b200 as P
    from synth import gen_torch as GT
    from synth import layouts as LY

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    steps = int(os.environ.get("SKEW_STEPS", "10"))
    out = os.environ.get("SKEW_OUT")
    s = torch.cuda.current_stream()

    def timed(fn):
        for i in range(3):
            fn(700 + i)
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for i in range(steps):
            fn(703 + i)
        e1.record(s)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / steps], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for variant in ("uniform", "loguniform", "zipf", "giant"):
        lay = LY.skew1b(variant)
        N = sum(t.numel for t in lay)
        h = P.Lars([(t.numel, t.kind) for t in lay], device=local, nranks=world, base_lr=32.0, grad_dtype="f16",
                   grad_scale=1.0 / (1024 * world), flags=P.lars.FLAG_CARRY_WNORM)
        h.comm_init_torch()
        w, g = h.dp_buffers()
        m = torch.zeros(h.padded_numel, dtype=torch.float32, device=dev)
        GT.fill_weights(w, lay, h.offsets)
        GT.fill_grads(g, lay, h.offsets, rank, 0)
        GT.fill_momentum(m, lay, h.offsets)
        ms_fused = timed(lambda it: h.dp_allreduce_lars_step(w, g, m, it))
        assert h.last_step_status() == 0
        wn, gn = w.clone(), g.clone()  # ordinary buffers -> NCCL reduce-scatter / all-gather path
        ms_nccl = timed(lambda it: h.dp_allreduce_lars_step(wn, gn, m, it))
        bus = (world - 1) / world * 6 * h.padded_numel
        splits = sum(1 for l, t in enumerate(lay)
                     if h.offsets[l] // (h.padded_numel // world) != (h.offsets[l] + t.numel - 1) // (h.padded_numel // world))
        row = {"workload": f"skew1b:{variant}", "params": N, "P": world, "split_layers": splits,
               "fused_ms_per_step": round(ms_fused, 4), "nccl_ms_per_step": round(ms_nccl, 4),
               "fused_bus_GBps": round(bus / (ms_fused * 1e-3) / 1e9, 1),
               "fused_frac_of_770": round(bus / (ms_fused * 1e-3) / 1e9 / NVLINK_PEER_GBS, 4),
               "params_per_s": round(world * N / (ms_fused * 1e-3), 1)}
        if rank == 0:
            print(json.dumps(row), flush=True)
            if out:
                with open(out, "a") as f:
                    f.write(json.dumps(row) + "\n")
        del wn, gn, m, w, g
        h.close()
        torch.cuda.empty_cache()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
