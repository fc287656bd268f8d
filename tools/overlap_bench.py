#!/usr/bin/env python
"""Overlap of the gradient combine with backward via static groups (§III-C-2; SURVEY
NEXT-f2), measured on B200 under torchrun (one process per GPU, NCCL).

A synthetic backward pass produces the ResNet-50 gradients in backward order (last tensor first): every
conv / fc weight gradient is a real bf16 tensor-core GEMM of the layer's backward shapes at the paper's
per-GPU batch (81,920 / 2,048 = 40 images, 224 px): wgrad dY^T [Cout x B*HW] . X [B*HW x Cin*k*k] written
(as fp16) into the layer's slot of g, plus the dgrad GEMM dY [B*HW x Cout] . W [Cout x Cin*k*k] whose output
is discarded. BN/bias gradients are copies.
Per configuration: (1) backward alone; (2) backward, then the whole dp step (no overlap): the NCCL path with
contiguous shards and the fused NVLink path; (3) static groups at several thresholds, each group reported with
dp_group_ready as soon as backward has written its last member. `exposed_ms` = iteration time - backward
time = the part of the combine + update that backward does not hide. One step per threshold is checked with
tools/overlap_trace.validate_trace. Device time by CUDA events on the compute stream, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def spatial(name: str) -> int:
    """Output H*W of a ResNet-50 (torchvision v1.5) tensor at 224 px input."""
    if name.startswith("conv1") or name.startswith("bn1"):
        return 112 * 112
    if name.startswith("fc"):
        return 1
    m = re.match(r"layer(\d)\.(\d+)\.(\w+)", name)
    stage, block, part = int(m.group(1)), int(m.group(2)), m.group(3)
    hw = {1: 56, 2: 28, 3: 14, 4: 7}[stage]
    if block == 0 and stage > 1 and part in ("conv1", "bn1"):  # stride sits on conv2 of block 0
        hw *= 2
    return hw * hw


def main():
    import torch
    import torch.distributed as dist

    import paper_1903_12650_b200 as PK
    from synth import layouts as LY
    from tools.overlap_trace import validate_trace

    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=40)
    ap.add_argument("--thresholds", default="262144,1048576,4194304,16777216,67108864")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--max-ctas", default="4", help="LARS_GROUP_MAX_CTAS values to sweep (0 = main comm)")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rank, P = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    lay = LY.resnet50()
    L = len(lay)
    gen = torch.Generator(device=dev)
    gen.manual_seed(100000 + rank)
    # backward work per tensor
    work = []
    maxa = maxy = maxw = 1
    for t in lay:
        if t.kind == "weight":
            M = a.batch * spatial(t.name)
            N, K = t.numel // t.fan_in, t.fan_in
            work.append((M, N, K))
            maxa, maxy, maxw = max(maxa, M * K), max(maxy, M * N), max(maxw, N * K)
        else:
            work.append(None)
    X = torch.randn(maxa, device=dev, dtype=torch.bfloat16, generator=gen) * 0.05
    DY = torch.randn(maxy, device=dev, dtype=torch.bfloat16, generator=gen) * 0.05
    W = torch.randn(maxw, device=dev, dtype=torch.bfloat16, generator=gen) * 0.05
    DX = torch.empty(maxa, device=dev, dtype=torch.bfloat16)
    flops = sum(2 * 2 * M * N * K for (M, N, K) in (w for w in work if w))
    s = torch.cuda.current_stream()

    def backward(h, g, gsrc, offsets, groups, report, done_ev=None):
        gi = 0
        for l in range(L - 1, -1, -1):
            o, n = offsets[l], lay[l].numel
            if work[l] is not None:
                M, N, K = work[l]
                dy, x = DY[:M * N].view(M, N), X[:M * K].view(M, K)
                torch.mm(dy, W[:N * K].view(N, K), out=DX[:M * K].view(M, K))  # dgrad (discarded)
                g[o:o + n].view(N, K).copy_(torch.mm(dy.t(), x))             # wgrad -> g (fp16)
            else:
                g[o:o + n].copy_(gsrc[o:o + n])
            if done_ev is not None:
                done_ev[l].record(s)
            if report and groups is not None and l == groups[gi]["first"]:
                h.dp_group_ready(g, gi)
                gi += 1

    def run(label, policy=None, thr=None, fused=False, step=True, overlap=False):
        kw = dict(base_lr=32.0, grad_dtype="f16", grad_scale=1.0 / (1024 * P), nranks=P, flags=1)
        if policy:
            kw["shard_policy"] = policy
        if thr:
            kw["group_bytes"] = thr
        h = PK.Lars([(t.numel, t.kind) for t in lay], device=local, **kw)
        h.comm_init_torch()
        if fused:
            w, g = h.dp_buffers()
        else:
            w = torch.empty(h.padded_numel, device=dev, dtype=torch.float32)
            g = torch.zeros(h.padded_numel, device=dev, dtype=torch.float16)
        h.init_weights(w, 100000)
        m = torch.zeros(h.padded_numel, device=dev, dtype=torch.float32)
        gsrc = (torch.randn(h.padded_numel, device=dev, generator=gen) * 1e-2).half()
        groups = h.groups() if overlap else None
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        times = []
        for i in range(a.warmup + a.steps):
            dist.barrier()
            torch.cuda.synchronize()
            e0.record(s)
            backward(h, g, gsrc, h.offsets, groups, overlap)
            if step:
                h.dp_allreduce_lars_step(w, g, m, 700 + i % 100)
            e1.record(s)
            torch.cuda.synchronize()
            if i >= a.warmup:
                times.append(e0.elapsed_time(e1))
        res = {"config": label, "ms": sorted(times)[len(times) // 2]}
        if overlap:  # one traced step through the schedule checker
            h.group_trace_enable(True)
            done = [torch.cuda.Event(enable_timing=True) for _ in range(L)]
            r0 = torch.cuda.Event(enable_timing=True)
            dist.barrier()
            r0.record(s)
            backward(h, g, gsrc, h.offsets, groups, True, done)
            h.dp_allreduce_lars_step(w, g, m, 700)
            torch.cuda.synchronize()
            tr = h.group_trace_read(r0)
            bwd = {l: r0.elapsed_time(done[l]) for l in range(L)}
            bad = validate_trace(groups, bwd, tr, L, h.padded_numel)
            res.update(groups=len(groups), trace_ok=not bad, violations=bad[:3],
                       last_group_rs_ms=round(tr["rs_end"][-1] - tr["rs_start"][-1], 4),
                       step_after_last_ready_ms=round(tr["applied"] - tr["ready"][-1], 4))
        h.close()
        t = torch.tensor([res["ms"]], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res["ms"] = round(float(t.item()), 4)
        return res

    out = []
    bwd = run("backward only", step=False)
    bwd_ms = bwd["ms"]
    out.append(dict(bwd, exposed_ms=0.0))
    for label, kw in [("no overlap: NCCL RS+K1+C3+K2+AG after backward", {}),
                      ("no overlap: fused NVLink path after backward", dict(fused=True))]:
        r = run(label, **kw)
        r["exposed_ms"] = round(r["ms"] - bwd_ms, 4)
        out.append(r)
    for mc in [int(x) for x in a.max_ctas.split(",")]:
        os.environ["LARS_GROUP_MAX_CTAS"] = str(mc)
        for thr in [int(x) for x in a.thresholds.split(",")]:
            r = run(f"static groups {thr / 2**20:g} MiB, max {mc} NCCL CTAs, dp_group_ready during backward",
                    policy="groups", thr=thr, overlap=True)
            r["exposed_ms"] = round(r["ms"] - bwd_ms, 4)
            r["group_bytes"], r["max_ctas"] = thr, mc
            out.append(r)
    if rank == 0:
        head = {"P": P, "backward": "bf16 GEMMs (dgrad + wgrad per conv/fc)", "batch_per_gpu": a.batch, "layout": "resnet50 (fp16 g)",
                "backward_gemm_tflop": round(flops / 1e12, 4), "steps": a.steps}
        print(json.dumps(head), flush=True)
        for r in out:
            print(json.dumps(r), flush=True)
        if a.out:
            with open(a.out, "w") as f:
                f.write(json.dumps(head) + "\n")
                for r in out:
                    f.write(json.dumps(r) + "\n")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
