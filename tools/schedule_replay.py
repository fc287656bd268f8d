#!/usr/bin/env python
"""BASELINE.json configs[3] measurement: the ResNet-152 layout (467 tensors, 60,192,808 params) over the whole
schedule at B = 81,920 — 16 updates/epoch x 90 epochs = 1,440 steps — replayed as CUDA
graphs of the device-iteration entry points (the iteration advances on the device; one graph per gradient
buffer of a ring of 4, so L2 never holds a step's inputs). Correctness of the same replay is in
tests/test_gpu_schedule.py; this tool only times it (CUDA events around all 1,440 replays).

P = 1: lars_step_dev_iter, fp32 gradients, carried weight norms.
P > 1 (torchrun): dp_allreduce_lars_step_dev_iter, fp16 gradients, on the fused NVLink path (the library's
symmetric gradient buffer, so the gradient is the same every step) or, with --nccl, the NCCL path with
the 4-buffer ring. Prints one JSON line (rank 0; max over ranks).
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_1903_12650_b200 as PK
    from synth import gen_torch as GT
    from synth import layouts as LY

    ap = argparse.ArgumentParser()
    ap.add_argument("--nccl", action="store_true")
    ap.add_argument("--no-carry", action="store_true")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    P = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if P > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    lay = LY.resnet152()
    flags = 0 if a.no_carry else 1
    dt = "f32" if P == 1 else "f16"
    h = PK.Lars([(t.numel, t.kind) for t in lay], device=local, nranks=P, base_lr=32.0, grad_dtype=dt,
                grad_scale=1.0 / (1024 * P), flags=flags)
    assert (h.ipe, h.total_iters, h.warmup_iters) == (16, 1440, 80)
    fused = False
    if P > 1:
        h.comm_init_torch()
        if not a.nccl:
            try:
                w, gsym = h.dp_buffers()
                fused = True
            except PK.LarsError:
                pass
    tdt = torch.float32 if dt == "f32" else torch.float16
    if not fused:
        w = torch.empty(h.padded_numel, dtype=torch.float32, device=dev)
    h.init_weights(w, 100000)
    m = torch.zeros(h.padded_numel, dtype=torch.float32, device=dev)
    if fused:
        ring = [gsym]
    else:
        ring = [torch.zeros(h.padded_numel, dtype=tdt, device=dev) for _ in range(4)]
    for k, g in enumerate(ring):
        GT.fill_grads(g, lay, h.offsets, rank, k)
    it = torch.zeros(1, dtype=torch.int64, device=dev)
    stream = torch.cuda.Stream(device=dev)
    step = h.lars_step_dev_iter if P == 1 else h.dp_allreduce_lars_step_dev_iter
    # warm-up outside the graphs (NCCL/PDL setup), then reset the device iteration
    for k in range(3):
        step(w, ring[k % len(ring)], m, it, stream=stream)
    stream.synchronize()
    graphs = []
    for g in ring:
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=stream):
            step(w, g, m, it, stream=stream)
        graphs.append(gr)
    it.zero_()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for t in range(1440):
            graphs[t % len(graphs)].replay()
        e1.record(stream)
    stream.synchronize()
    ms = e0.elapsed_time(e1)
    assert int(it.item()) == 1440 and h.last_step_status() == 0
    if dist:
        x = torch.tensor([ms], device=dev)
        dist.all_reduce(x, op=dist.ReduceOp.MAX)
        ms = float(x.item())
    N = sum(t.numel for t in lay)
    path = "1 GPU" if P == 1 else ("fused NVLink" if fused else "NCCL RS/AG")
    res = {"workload": "resnet152_full_schedule_replay", "params": N, "tensors": len(lay), "P": P,
           "grad_dtype": dt, "carry_wnorm": bool(flags), "path": path, "steps": 1440,
           "gradient_buffers": len(ring), "replay_s": round(ms / 1e3, 4), "ms_per_step": round(ms / 1440, 5),
           "params_per_s": round(N * P * 1440 / (ms / 1e3), 1)}
    if P == 1:  # K2 algorithmic bytes per step, as a whole-step fraction of the measured copy peak
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        hbm = float(peaks["hbm_gbs"])
        res["step_frac_of_hbm_copy_peak_20B"] = round(20 * N / (ms / 1440 * 1e-3) / 1e9 / hbm, 4)
    if rank == 0:
        print(json.dumps(res), flush=True)
        if a.out:
            with open(a.out, "a") as f:
                f.write(json.dumps(res) + "\n")
    for gr in graphs:  # release every graph (NCCL work captured in them) before the communicator goes
        gr.reset()
    torch.cuda.synchronize()
    del graphs, gr
    h.close()
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
