#!/usr/bin/env python
"""Every kernel path of the library, briefly, for compute-sanitizer (memcheck / racecheck / synccheck) on ONE
GPU (not product code; tools/sanitize_round.sh runs it under one tool per gpurun call).

Cases: lars_step on tiny and ResNet-50 (fp32 / fp16 / bf16 gradients, with and without carried weight norms,
lr-at-apply), the device-iteration entry point, parallel initialization, and the data-parallel step through
a one-rank communicator on the fused NVLink kernels (F1/F2, also with half-precision compute weights and the
8-peer F1 instance) and on the NCCL path (reduce-scatter, K1, C3 allreduce + split finish, K2, all-gather).
A non-finite gradient case exercises the skip branches. Prints one line per case.
"""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_1903_12650_b200 as PK
    from synth import gen as G
    from synth import layouts as LY

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    big = "--small" not in sys.argv
    layouts = ["tiny"] + (["resnet50"] if big else [])
    for name in layouts:
        lay = LY.by_name(name)
        for dtype in ("f32", "f16", "bf16"):
            for flags in (0, PK.lars.FLAG_CARRY_WNORM, PK.lars.FLAG_CARRY_WNORM | PK.lars.FLAG_LR_AT_APPLY):
                h = PK.Lars([(t.numel, t.kind) for t in lay], device=0, grad_dtype=dtype, base_lr=32.0,
                            grad_scale=1.0 / G.GRAD_PRESCALE, flags=flags)
                pk = lambda a: torch.from_numpy(G.pack(a, h.offsets, h.padded_numel)).to(dev)
                w, g, m = pk(G.weights(lay)), pk(G.grads(lay, 0, 0, dtype)), pk(G.momentum(lay, 1e-3))
                for t in (79, 80, 81):
                    h.lars_step(w, g, m, t)
                it = torch.tensor([700], dtype=torch.int64, device=dev)
                h.lars_step_dev_iter(w, g, m, it)
                if dtype == "f32":  # non-finite gradient: the skip branches
                    g[h.offsets[-1]] = float("nan")
                    h.lars_step(w, g, m, 82)
                torch.cuda.synchronize()
                print("ok lars_step", name, dtype, "flags", flags, flush=True)
                h.close()
        h = PK.Lars([(t.numel, t.kind) for t in lay], device=0, grad_dtype="f32", base_lr=32.0)
        w = torch.empty(h.padded_numel, dtype=torch.float32, device=dev)
        h.init_weights(w, 100000)
        torch.cuda.synchronize()
        print("ok init_weights", name, flush=True)
        h.close()
        # data-parallel kernels through a one-rank communicator
        for fused in (True, False):
            for flags in (PK.lars.FLAG_CARRY_WNORM, PK.lars.FLAG_CARRY_WNORM | PK.lars.FLAG_HALF_WEIGHTS):
                for npt in ((None, "8") if fused else (None,)):
                    if npt:
                        os.environ["LARS_DP_NP"] = npt
                    h = PK.Lars([(t.numel, t.kind) for t in lay], device=0, grad_dtype="f16", base_lr=32.0,
                                nranks=1, grad_scale=1.0 / G.GRAD_PRESCALE, flags=flags)
                    h.comm_init(0, 1, PK.get_unique_id())
                    os.environ.pop("LARS_DP_NP", None)
                    pk = lambda a: torch.from_numpy(G.pack(a, h.offsets, h.padded_numel)).to(dev)
                    w, g, m = pk(G.weights(lay)), pk(G.grads(lay, 0, 0, "f16")), pk(G.momentum(lay, 1e-3))
                    if fused:
                        ws, gs = h.dp_buffers()
                        ws.copy_(w)
                        gs.copy_(g)
                        w, g = ws, gs
                    for t in (80, 81, 82):
                        h.dp_allreduce_lars_step(w, g, m, t)
                    g.view(torch.float16)[h.offsets[0]] = float("inf")
                    h.dp_allreduce_lars_step(w, g, m, 83)
                    torch.cuda.synchronize()
                    print("ok dp P=1", name, "fused" if fused else "nccl", "flags", flags, "np", npt, flush=True)
                    h.close()
    print("sanitize cases done", flush=True)


if __name__ == "__main__":
    main()
