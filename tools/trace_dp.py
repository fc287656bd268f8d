#!/usr/bin/env python
"""Per-CTA timeline of the fused data-parallel kernels (F1 reduce+norms, F2 update+gather) from the
diagnostics library (tools/trace_build.py). Run under torchrun, one process per GPU."""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist

    import paper_1903_12650_b200 as PK
    from synth import gen as G
    from synth import layouts as LY

    rank, P = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    lib = PK.load_library(os.path.join(ROOT, "build", f"liblars_trace{os.environ.get('TRACE_TAG', '')}.so"))
    lay = LY.resnet50()
    h = PK.Lars([(t.numel, t.kind) for t in lay], device=rank, grad_dtype="f16", nranks=P, base_lr=32.0,
                grad_scale=1 / (1024 * P), flags=1)
    h.comm_init_torch()
    w, g = h.dp_buffers()
    w.copy_(torch.from_numpy(G.pack(G.weights(lay), h.offsets, h.padded_numel)))
    g.copy_(torch.from_numpy(G.pack(G.grads(lay, rank, 0, "f16"), h.offsets, h.padded_numel)))
    m = torch.from_numpy(G.pack(G.momentum(lay, 1e-3), h.offsets, h.padded_numel)).to(dev)
    buf = torch.zeros(8 * 4096 * 4, dtype=torch.int64, device=dev)
    lib.lars_trace_arm.argtypes = [ctypes.c_void_p]
    for i in range(20):
        h.dp_allreduce_lars_step(w, g, m, 719 + i)
    torch.cuda.synchronize()
    assert lib.lars_trace_arm(buf.data_ptr()) == 0
    dist.barrier()
    spans = []
    for i in range(12):
        dist.barrier()
        h.dp_allreduce_lars_step(w, g, m, 740 + i)
        torch.cuda.synchronize()
        x = buf.view(8, 4096, 4).cpu().numpy()
        a, b = x[2], x[3]
        n1_, n2_ = int(a[0, 3]), int(b[0, 3])
        f0 = x[6]
        n0_ = int(f0[0, 3])
        s0 = min(a[:n1_, 0].min(), f0[:n0_, 0].min()) if n0_ else a[:n1_, 0].min()
        spans.append(((x[5][:n1_, 2].max() - s0) / 1e3, (a[:n1_, 1].max() - s0) / 1e3, (b[:n2_, 1].max() - s0) / 1e3))
    med = np.median(np.array(spans[2:]), axis=0)
    print(f"rank {rank} median of 10: barrier past {med[0]:.1f} us, F1 end {med[1]:.1f}, F2 end {med[2]:.1f}", flush=True)
    tr = buf.view(8, 4096, 4).cpu().numpy()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    np.save(os.path.join(ROOT, "gpurun_out", f"trace_dp_p{P}_r{rank}.npy"), tr)
    f1, f2, mk = tr[2], tr[3], tr[5]
    n1, n2 = int(f1[0, 3]), int(f2[0, 3])
    t0 = f1[:n1, 0].min()
    us = lambda x: (x - t0) / 1e3
    bar = us(mk[:n1, 2])
    f1s, f1e = us(f1[:n1, 0]), us(f1[:n1, 1])
    f2s, f2e = us(f2[:n2, 0]), us(f2[:n2, 1])
    q = lambda a: f"{np.min(a):.1f}/{np.median(a):.1f}/{np.max(a):.1f}"
    pre = us(tr[4][:n1, 2])
    coll = us(tr[4][:n2, 0])
    last = int(np.argmax(f1e))
    waited = us(tr[6][:n2, 0])
    polled = us(tr[6][:n2, 1])
    print(f"rank {rank}: F2 shares polled in {q(polled)}", flush=True)
    print(f"rank {rank}: final F1 CTA {last}: tile done {pre[last]:.1f} end {f1e[last]:.1f}; "
          f"F2 past griddepcontrol.wait {q(waited)}; F2 shares collected {q(coll)}", flush=True)
    print(f"rank {rank}: F1 ctas {n1}: start {q(f1s)}  past-barrier {q(bar)}  end {q(f1e)} | "
          f"F2 ctas {n2}: start {q(f2s)} end(before exit barrier) {q(f2e)}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
