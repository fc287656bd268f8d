#!/usr/bin/env python
"""Drives every kernel path of the library, for the device-checked build (compute-sanitizer is closed on the
GPU pool, so bounds and invariants are checked by the library itself):

    python -m paper_1903_12650_b200.build --checked
    LARS_LIB=build/checked/liblars_b200_checked.so python tools/checked_step.py --layout resnet50

Runs a few steps of every kernel path on one GPU and checks the last one against the oracle (a failed
LARS_DCHECK traps the kernel and the step raises; a silent run is also a correct run):
  single   K1 + K2 (lars_step), with and without carried weight norms, fp32 and fp16 gradients
  fused    F1 + F2 through a one-rank communicator (symmetric NCCL windows, LSA barrier, epoch flags)
  nccl     reduce-scatter + K1 + C3 + split finish + K2 + all-gather through a one-rank communicator
Under torchrun (WORLD_SIZE > 1) the dp modes run at that world size instead (one sanitizer per rank).
"""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layout", default="tiny")
    ap.add_argument("--modes", default="single,fused,nccl")
    ap.add_argument("--steps", type=int, default=2)
    args = ap.parse_args()
    import numpy as np
    import torch

    import paper_1903_12650_b200 as PK
    from oracle import oracle as O
    from synth import gen as G
    from synth import layouts as LY
    from tests._parity import TOL_F16_DP, TOL_F32, from_dev, gate, hp_kwargs, oracle_hp, to_dev

    rank, P = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if P > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lay = LY.by_name(args.layout)
    kinds, sizes = [t.kind for t in lay], [t.numel for t in lay]
    for mode in args.modes.split(","):
        cfgs = [("f32", 0), ("f32", 1), ("f16", 1)] if mode == "single" else [("f16", 1), ("bf16", 0)]
        for dtype, flags in cfgs:
            kw = hp_kwargs(grad_dtype=dtype, nranks=1 if mode == "single" else P, flags=flags,
                           grad_scale=1.0 / (G.GRAD_PRESCALE * (1 if mode == "single" else P)))
            h = PK.Lars([(t.numel, t.kind) for t in lay], device=local, **kw)
            if mode != "single":
                if P > 1:
                    h.comm_init_torch()
                else:
                    h.comm_init(0, 1, PK.get_unique_id())
            pack = lambda a: to_dev(G.pack(a, h.offsets, h.padded_numel), local)
            w, m = pack(G.weights(lay)), pack(G.momentum(lay, 1e-3))
            if mode == "fused":
                ws, gs = h.dp_buffers()
                ws.copy_(w)
                w = ws
            for k in range(args.steps):
                t = 79 + k
                g_all = [G.grads(lay, r, t, dtype) for r in range(P if mode != "single" else 1)]
                g = pack(g_all[rank if mode != "single" else 0])
                if mode == "fused":
                    gs.copy_(g)
                    g = gs
                pre_w = G.unpack(from_dev(w), h.offsets, sizes)
                pre_m = G.unpack(from_dev(m), h.offsets, sizes)
                (h.lars_step if mode == "single" else h.dp_allreduce_lars_step)(w, g, m, t)
                torch.cuda.synchronize()
            assert h.last_step_status() == 0
            r = O.dp_step(kinds, oracle_hp(kw), t, pre_w, g_all, pre_m)
            wg = G.unpack(from_dev(w), h.offsets, sizes)
            mine = range(len(lay))
            if mode != "single" and P > 1:  # this rank's shard only
                b, e = h.shard_range(rank)
                mine = [l for l in mine if b <= h.offsets[l] and h.offsets[l] + sizes[l] <= e]
            tol = TOL_F32 if (P == 1 or mode == "fused" or dtype == "f32") else TOL_F16_DP
            if mine:
                err = gate(f"{mode} {dtype} flags={flags}", np.concatenate([wg[l] for l in mine]),
                           np.concatenate([r.w[l] for l in mine]), np.concatenate([r.w_env[l] for l in mine]), tol)
                print(f"[rank {rank}] {args.layout} {mode} {dtype} flags={flags}: ok (w env err {err:.2e})", flush=True)
            h.close()
    if P > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
