#!/usr/bin/env python
"""Per-CTA timeline of K1/K2 from the diagnostics library (tools/trace_build.py)."""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_1903_12650_b200 as PK
    from synth import gen as G
    from synth import layouts as LY

    lib = PK.load_library(os.path.join(ROOT, "build", f"liblars_trace{os.environ.get('TRACE_TAG', '')}.so"))
    layout = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
    dtype = sys.argv[2] if len(sys.argv) > 2 else "f32"
    lay = LY.by_name(layout)
    h = PK.Lars([(t.numel, t.kind) for t in lay], device=0, grad_dtype=dtype, base_lr=32.0, grad_scale=1 / 1024,
                flags=int(os.environ.get("TRACE_FLAGS", "0")))
    dev = torch.device("cuda", 0)
    w = torch.from_numpy(G.pack(G.weights(lay), h.offsets, h.padded_numel)).to(dev)
    g = torch.from_numpy(G.pack(G.grads(lay, 0, 0, dtype), h.offsets, h.padded_numel)).to(dev)
    m = torch.from_numpy(G.pack(G.momentum(lay, 1e-3), h.offsets, h.padded_numel)).to(dev)
    buf = torch.zeros(6 * 4096 * 4, dtype=torch.int64, device=dev)
    lib.lars_trace_arm.argtypes = [ctypes.c_void_p]
    for i in range(30):
        h.lars_step(w, g, m, 719 + i)
    torch.cuda.synchronize()
    assert lib.lars_trace_arm(buf.data_ptr()) == 0
    spans = []
    for i in range(12):  # per step: K1 span, K1->K2 gap, K2 span, K1 start -> K2 end
        h.lars_step(w, g, m, 800 + i)
        torch.cuda.synchronize()
        x = buf.view(6, 4096, 4).cpu().numpy()
        n1, n2 = int(x[0, 0, 3]), int(x[1, 0, 3])
        a0, a1 = x[0, :n1, 0].min(), x[0, :n1, 1].max()
        b0, b1 = x[1, :n2, 0].min(), x[1, :n2, 1].max()
        spans.append(((a1 - a0) / 1e3, (b0 - a1) / 1e3, (b1 - b0) / 1e3, (b1 - a0) / 1e3))
    med = np.median(np.array(spans[2:]), axis=0)
    print(f"median over 10 steps: K1 {med[0]:.2f} us, gap {med[1]:.2f}, K2 {med[2]:.2f}, K1+K2 {med[3]:.2f}")
    tr = buf.view(6, 4096, 4).cpu().numpy()
    n1 = int(tr[0, 0, 3])
    t0k1 = tr[0, :n1, 0].min()
    pa = (tr[4, :n1, 0] - t0k1) / 1e3
    print(f"K1 phase A (chunk streaming) done: min/p50/max = {pa.min():.1f}/{np.median(pa):.1f}/{pa.max():.1f} us")
    n2 = int(tr[1, 0, 3])
    pro = (tr[5, :n2, 0] - tr[1, :n2, 0]) / 1e3
    if (tr[5, :n2, 0] > 0).all():
        print(f"K2 deferred-finish prologue: min/p50/max = {pro.min():.2f}/{np.median(pro):.2f}/{pro.max():.2f} us")
        for k, what in ((1, "segment records + flags in"), (2, "whole layers finished")):
            if not (tr[5, :n2, k] > 0).all():
                continue
            x = (tr[5, :n2, k] - tr[1, :n2, 0]) / 1e3
            print(f"  {what}: min/p50/max = {x.min():.2f}/{np.median(x):.2f}/{x.max():.2f} us")
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    np.save(os.path.join(ROOT, "gpurun_out", "trace_step.npy"), tr)
    for k, name in enumerate(["K1 norms", "K2 update"]):
        n = int(tr[k, 0, 3])
        t = tr[k, :n]
        t0 = t[:, 0].min()
        st, en = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3
        dur = en - st
        print(f"{name}: ctas={n} span={en.max():.1f}us start[min,max]=({st.min():.1f},{st.max():.1f}) "
              f"end[min,p50,max]=({en.min():.1f},{np.median(en):.1f},{en.max():.1f}) dur[min,p50,max]=("
              f"{dur.min():.1f},{np.median(dur):.1f},{dur.max():.1f})")
        slow = np.argsort(-en)[:8]
        print("  slowest CTAs (cta, sm, start, end):", [(int(c), int(t[c, 2]), round(st[c], 1), round(en[c], 1)) for c in slow])
        sms = t[:, 2]
        per_sm = {}
        for c in range(n):
            per_sm.setdefault(int(sms[c]), []).append(c)
        load = sorted(((len(v), s) for s, v in per_sm.items()), reverse=True)
        print("  CTAs per SM (max, min, #SMs):", load[0][0], load[-1][0], len(per_sm))


if __name__ == "__main__":
    main()
