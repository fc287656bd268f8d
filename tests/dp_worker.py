"""One rank of the multi-GPU parity test (launched by tests/test_gpu_dp.py through torchrun).

Checks, on every rank, for dp_allreduce_lars_step (BASELINE configs[2]):
  * the reduced gradient shard equals the brute-force rank sum: bitwise for integer-valued fp16
    gradients, within the (P-1)*2^-11*sum|g_r| fp16 reduction bound otherwise;
  * per-layer norms match the oracle on the exact buffer K1 read (1e-6);
  * the rank's w and m shard match the oracle's data-parallel step with the exact sum (envelope gate);
  * w is bitwise identical on all ranks after the all-gather;
  * a non-finite gradient on ONE rank makes EVERY rank skip (w, m untouched);
  * a layout that differs across ranks is rejected at lars_comm_init (LARS_ERR_LAYOUT).
"""
from __future__ import annotations

import json
import os
import re
import sys
import traceback
from datetime import timedelta

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist

    import paper_1903_12650_b200 as PK
    from oracle import oracle as O
    from synth import gen as G
    from synth import layouts as LY
    from tests._parity import TOL_BF16_DP, TOL_F16_DP, TOL_F32, from_dev, gate, gate_norms, hp_kwargs, oracle_hp

    rank, P = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev, timeout=timedelta(seconds=120))
    report = {"rank": rank, "P": P, "cases": [], "failures": []}

    def all_same(t):
        x = t.contiguous().view(torch.int32)
        lo, hi = x.clone(), x.clone()
        dist.all_reduce(lo, op=dist.ReduceOp.MIN)
        dist.all_reduce(hi, op=dist.ReduceOp.MAX)
        return bool(torch.equal(lo, hi))

    def owned_ranges(h, r):
        """Flat element ranges rank r reduces and updates (one shard, or slice r of every static group)."""
        if hpkw_policy(h) == "groups":
            return [(gk["begin"] + r * (gk["len"] // P), gk["begin"] + (r + 1) * (gk["len"] // P))
                    for gk in h.groups()]
        return [h.shard_range(r)]

    def hpkw_policy(h):
        return getattr(h, "_policy", "contiguous")

    def backward_then_ready(h, g_src, g, early):
        """Synthetic backward: tensors written into g in backward order (last tensor first), each after a
        short device spin; group k is reported (dp_group_ready) right after its last member is written.
        early = number of groups reported before the step (the step issues the rest)."""
        groups = h.groups()
        g.zero_()
        for k, gk in enumerate(groups):
            for l in range(gk["last"], gk["first"] - 1, -1):
                torch.cuda._sleep(2000)
                o, n = h.offsets[l], h.sizes[l]
                g[o:o + n].copy_(g_src[o:o + n])
            if k < early:
                h.dp_group_ready(g, k)

    def run_case(name, lay, dtype, t, kind="random", inject_nan=False, fused=False, overlap=None, graph=False,
                 **hpkw):
        kw = hp_kwargs(grad_dtype=dtype, grad_scale=1.0 / (G.GRAD_PRESCALE * P), **hpkw)
        h = PK.Lars([(x.numel, x.kind) for x in lay], device=local, nranks=P, **kw)
        h._policy = kw.get("shard_policy", "contiguous")
        h.sizes = [x.numel for x in lay]
        h.comm_init_torch()
        w_l, m_l = G.weights(lay), G.momentum(lay, 1e-3)
        if kind == "integer":
            g_all = [G.integer_grads(lay, r, t, dtype) for r in range(P)]
        else:
            g_all = [G.grads(lay, r, t, dtype) for r in range(P)]
        expect_skip = bool(inject_nan)
        if kind in ("overflow", "near-overflow"):  # reading #29: every rank's element is finite in fp16
            v = 40000.0 if kind == "overflow" else 65504.0 / (2 * P)
            for r in range(P):
                g_all[r][0] = g_all[r][0].copy()
                g_all[r][0][5] = np.float16(v)
            expect_skip = bool(np.isinf(O.combine([g_all[r][0][5:6] for r in range(P)], 1.0)).any())
            assert expect_skip == (kind == "overflow" and P > 1)
        if inject_nan:  # rank 1 poisons one element of ITS local gradient
            q, l0, i0 = 1 % P, 0, 3
            if inject_nan == "split":  # ... the last element of a layer that straddles a shard boundary
                rng0 = owned_ranges(h, 0) + owned_ranges(h, 1 % P)
                cuts = sorted({e for _, e in rng0} | {b for b, _ in rng0})
                # (P = 1: no layer straddles ranks; the last element of layer 0)
                l0 = next((l for l, x in enumerate(lay)
                           if any(h.offsets[l] < c < h.offsets[l] + x.numel for c in cuts)), 0)
                i0 = lay[l0].numel - 1
            g_all[q][l0] = g_all[q][l0].copy()
            g_all[q][l0][i0] = np.nan
        pack = lambda a: torch.from_numpy(G.pack(a, h.offsets, h.padded_numel).view(
            np.int16 if a[0].dtype == np.uint16 else a[0].dtype)).to(dev)
        w, g, m = pack(w_l), pack(g_all[rank]), pack(m_l)
        if fused:  # library-owned symmetric buffers: the fused NVLink path (F1, FX, F2)
            w_sym, g_sym = h.dp_buffers()
            w_sym.copy_(w)
            g_sym.copy_(g)
            w, g = w_sym, g_sym
            torch.cuda.synchronize()
        g_before = g.clone()
        if overlap:  # static groups reported while the synthetic backward still runs
            ng = len(h.groups())
            assert ng > 1, f"{name}: expected several groups"
            try:  # out-of-order report is rejected before anything is enqueued
                h.dp_group_ready(g, 1)
                raise AssertionError("out-of-order group accepted")
            except PK.LarsError as e:
                assert e.status == 1, e
            h.group_trace_enable(True)
            backward_then_ready(h, g_before, g, ng if overlap == "all" else ng // 2)
        if graph:  # the step captured once in a CUDA graph with a device-resident iteration, then replayed
            # one eager step first (NCCL sets up its connections lazily, outside any capture), then the
            # pre-step state is restored and the carried norms forgotten
            w_keep, m_keep = w.clone(), m.clone()
            h.dp_allreduce_lars_step(w, g, m, t)
            torch.cuda.synchronize()
            w.copy_(w_keep)
            m.copy_(m_keep)
            h.invalidate_carried_norms()
            torch.cuda.synchronize()
            it_dev = torch.tensor([t], dtype=torch.int64, device=dev)
            side = torch.cuda.Stream(device=dev)
            gr = torch.cuda.CUDAGraph()
            torch.cuda.synchronize()
            dbg = os.environ.get("DP_DEBUG")
            if dbg:
                print(f"[{rank}] {name}: capture", flush=True)
            with torch.cuda.graph(gr, stream=side, capture_error_mode="thread_local"):
                h.dp_allreduce_lars_step_dev_iter(w, g, m, it_dev, stream=side)
            if dbg:
                print(f"[{rank}] {name}: replay", flush=True)
            gr.replay()
            torch.cuda.synchronize()
            gr.reset()  # release the graph before the handle (and its NCCL communicator) can be destroyed
            torch.cuda.synchronize()
            if dbg:
                print(f"[{rank}] {name}: replayed it={int(it_dev.item())}", flush=True)
            assert int(it_dev.item()) == t + 1, "the device iteration did not advance"
        else:
            h.dp_allreduce_lars_step(w, g, m, t)
        torch.cuda.synchronize()
        res = {"name": name, "dtype": dtype, "t": t}
        half = bool(kw.get("flags", 0) & PK.lars.FLAG_HALF_WEIGHTS)
        if overlap:
            tr = h.group_trace_read()
            ng = len(tr["ready"])
            eps = 2e-3  # event timer resolution (ms)
            assert all(tr["rs_start"][k] + eps >= tr["ready"][k] for k in range(ng)), tr
            assert all(tr["rs_start"][k] + eps >= tr["rs_end"][k - 1] for k in range(1, ng)), tr
            assert tr["applied"] + eps >= max(tr["rs_end"]), tr
            res["groups"] = ng
            res["first_rs_before_backward_end_ms"] = round(tr["ready"][-1] - tr["rs_start"][0], 4)
        # collectives first: every rank calls them before any rank-local assertion. Half-precision compute
        # weights: the replicas are the compute-weight buffers (w outside the shard is stale by design).
        w16 = h.compute_weights() if half else None
        same = all_same(w16) if half else all_same(w)
        red_t, b, e = h.reduced_grad()
        red_dtype = {torch.float32: "f32", torch.float16: "f16", torch.int16: "bf16"}[red_t.dtype]
        if red_t.dtype == torch.int16:  # bf16 bit patterns travel as fp16 words (bit-preserving)
            red_t = red_t.view(torch.float16)
        parts = [torch.empty_like(red_t) for _ in range(P)]
        dist.all_gather(parts, red_t.clone())
        if hpkw_policy(h) == "groups":  # flat buffers: rank r's slices come from rank r
            full_red = np.zeros(h.padded_numel, dtype=from_dev(parts[0][:1]).dtype)
            for r in range(P):
                pr = from_dev(parts[r])
                for lo, hi in owned_ranges(h, r):
                    full_red[lo:hi] = pr[lo:hi]
            b, e = 0, h.padded_numel
        else:
            full_red = from_dev(torch.cat(parts))  # the exact buffer every K1 read, all shards
        if red_dtype == "bf16":
            full_red = full_red.view(np.uint16)
        res["reduced_dtype"] = red_dtype
        assert torch.equal(g.view(torch.int16) if g.element_size() == 2 else g.view(torch.int32),
                           g_before.view(torch.int16) if g.element_size() == 2 else g_before.view(torch.int32)), \
            "dp step modified the caller's gradient"
        assert same, f"{name}: w differs across ranks after the all-gather"
        status = h.last_step_status()
        sizes = [x.numel for x in lay]
        # this rank's piece of every layer (layers may straddle shard boundaries)
        pieces = {}
        for rb, re_ in owned_ranges(h, rank):
            for l in range(len(lay)):
                lo, hi = max(h.offsets[l], rb), min(h.offsets[l] + sizes[l], re_)
                if hi > lo:
                    assert l not in pieces, "a layer meets one rank in one piece"
                    pieces[l] = (lo - h.offsets[l], hi - h.offsets[l])
        mine = sorted(pieces)
        res["split_layers_here"] = sum(1 for l in mine if pieces[l] != (0, sizes[l]))
        wg = G.unpack(from_dev(w), h.offsets, sizes)
        mg = G.unpack(from_dev(m), h.offsets, sizes)
        if half:  # this rank's part of the compute weights is its new fp32 master rounded to nearest even
            w16_h = from_dev(w16)
            for l, (lo, hi) in pieces.items():
                mw = wg[l][lo:hi].astype(np.float32)
                if dtype == "f16":
                    want16 = mw.astype(np.float16).view(np.uint16)
                else:
                    u = mw.view(np.uint32).astype(np.uint64)
                    want16 = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
                got16 = w16_h[h.offsets[l] + lo: h.offsets[l] + hi].view(np.uint16)
                assert np.array_equal(got16, want16), f"{name}: compute weights != RNE(master) in tensor {l}"
            res["half_weights_checked"] = True
        if expect_skip:
            assert status == 1, f"{name}: rank {rank} did not skip (non-finite / overflowing gradient sum)"
            for l in mine:
                assert np.array_equal(wg[l], w_l[l]) and np.array_equal(mg[l], m_l[l])
            res["skipped_everywhere"] = True
            report["cases"].append(res)
            h.close()
            return
        assert status == 0
        kinds = [x.kind for x in lay]
        worst_sum = 0.0
        for l in mine:
            lo, hi = pieces[l]
            got = O.to_double(full_red[h.offsets[l] + lo: h.offsets[l] + hi])
            exact = O.combine([g_all[r][l][lo:hi] for r in range(P)], 1.0)
            if kind == "integer" and red_dtype != "bf16":
                assert np.array_equal(got, exact), f"{name}: integer sum not exact (tensor {l})"
            else:
                u = {"f16": 2.0 ** -11, "bf16": 2.0 ** -8, "f32": 2.0 ** -24}[red_dtype]
                bound = (P - 1) * u \
                    * sum(np.abs(O.to_double(g_all[r][l][lo:hi])) for r in range(P))
                err = np.abs(got - exact)
                assert (err <= bound).all(), f"{name}: reduction error above the (P-1)u sum|g| bound at tensor {l}"
                worst_sum = max(worst_sum, float(np.max(np.where(bound > 0, err / np.maximum(bound, 1e-300), 0))))
        res["sum_err_over_bound"] = worst_sum
        # norms (split layers included) on the exact reduced buffer
        hp = oracle_hp(kw)
        wn, gn, lam, coef = h.last_norms()
        s = kw["grad_scale"]
        for l in mine:
            red_l = full_red[h.offsets[l]: h.offsets[l] + sizes[l]]
            gate_norms(f"{name} ||w|| t{l}", [wn[l]], [O.l2norm(w_l[l])])
            gate_norms(f"{name} ||g|| t{l}", [gn[l]], [abs(s) * O.l2norm(O.to_double(red_l))])
        # this rank's pieces of w and m vs the oracle DP step (exact sum) of the layers it touches
        r_or = O.dp_step([kinds[l] for l in mine], hp, t, [w_l[l] for l in mine],
                         [[g_all[r][l] for l in mine] for r in range(P)], [m_l[l] for l in mine])
        # fp32 sums (the fused path, fp32 wire) or P = 1 (nothing summed): the fp32 gate; fp16 / bf16 sums on
        # the NCCL wire at P > 1: readings #17 / #18
        if red_dtype == "f32" or P == 1:
            tol = TOL_F32
        else:
            tol = TOL_F16_DP if red_dtype == "f16" else TOL_BF16_DP
        res["tol"] = tol
        if mine:
            sl = lambda arrs: np.concatenate([a[pieces[l][0]:pieces[l][1]] for a, l in zip(arrs, mine)])
            res["m_err"] = gate(f"{name} m", sl([mg[l] for l in mine]), sl(r_or.m), sl(r_or.m_env), tol)
            res["w_err"] = gate(f"{name} w", sl([wg[l] for l in mine]), sl(r_or.w), sl(r_or.w_env), tol)
        report["cases"].append(res)
        h.close()

    lay_r50 = LY.resnet50()
    cases = [("tiny-int", LY.tiny(), "f16", 80, dict(kind="integer")),
             ("random-f16", LY.random_layout(np.random.default_rng(7), 37), "f16", 81, {}),
             ("random-bf16", LY.random_layout(np.random.default_rng(8), 29), "bf16", 700, {}),
             ("random-f32", LY.random_layout(np.random.default_rng(9), 23), "f32", 3, {}),
             ("r50-f16", lay_r50, "f16", 719, {}),
             ("r50-int", lay_r50, "f16", 1439, dict(kind="integer")),
             ("r50-lpt-f16", lay_r50, "f16", 80, dict(shard_policy="lpt")),
             # 3 layers, whole-layer shards: at P >= 4 a rank owns no layer (it still takes part in every
             # collective and advances its iteration)
             ("tiny-lpt-f16", LY.tiny(), "f16", 80, dict(shard_policy="lpt")),
             ("fused-tiny-lpt-f16", LY.tiny(), "f16", 81, dict(shard_policy="lpt", fused=True)),
             ("r50-f16-buckets4", lay_r50, "f16", 81, dict(buckets=4)),
             ("random-bf16-buckets3", LY.random_layout(np.random.default_rng(18), 40), "bf16", 82, dict(buckets=3)),
             ("r50-int-buckets8-carry", lay_r50, "f16", 83, dict(kind="integer", buckets=8, flags=1)),
             ("zipf-f16", LY.skew1b("zipf", n_tensors=200, total=4_000_000), "f16", 500, {}),
             ("nan-on-rank1", LY.tiny(), "f16", 100, dict(inject_nan=True)),
             # reading #29: per-rank finite fp16 gradients whose sum overflows fp16 -> skipped on every path
             ("overflow-sum-f16", LY.tiny(), "f16", 100, dict(kind="overflow")),
             ("fused-overflow-sum-f16", LY.tiny(), "f16", 100, dict(kind="overflow", fused=True)),
             ("near-overflow-sum-f16", LY.tiny(), "f16", 100, dict(kind="near-overflow")),
             ("fused-near-overflow-sum-f16", LY.tiny(), "f16", 100, dict(kind="near-overflow", fused=True)),
             # a skipped FIRST step still leaves the compute weights = RNE(master) on every rank
             ("halfw-nan-first-step", LY.tiny(), "f16", 100, dict(inject_nan=True, flags=4)),
             ("fused-halfw-nan-first-step", LY.tiny(), "f16", 100, dict(inject_nan=True, flags=4, fused=True)),
             ("fused-tiny-int", LY.tiny(), "f16", 80, dict(kind="integer", fused=True)),
             ("fused-r50-f16", lay_r50, "f16", 719, dict(fused=True)),
             ("fused-r50-f16-carry", lay_r50, "f16", 720, dict(fused=True, flags=1)),
             ("fused-r50-f16-apply-step", lay_r50, "f16", 481, dict(fused=True, flags=1, momentum_form="apply",
                                                                   decay="step", milestones=(30, 60))),
             ("fused-random-bf16", LY.random_layout(np.random.default_rng(8), 29), "bf16", 700, dict(fused=True)),
             ("fused-zipf-f32", LY.skew1b("zipf", n_tensors=200, total=4_000_000), "f32", 500, dict(fused=True)),
             ("fused-nan-in-split-layer", LY.skew1b("zipf", n_tensors=50, total=1_000_000), "f16", 100,
              dict(inject_nan="split", fused=True)),
             ("nan-in-split-layer", LY.skew1b("zipf", n_tensors=50, total=1_000_000), "f16", 100,
              dict(inject_nan="split")),
             # one step captured in a CUDA graph (device iteration), NCCL and fused paths
             ("r50-f16-graph", lay_r50, "f16", 719, dict(graph=True)),
             ("fused-r50-f16-carry-graph", lay_r50, "f16", 1439, dict(fused=True, flags=1, graph=True)),
             # half-precision compute weights (NEXT-f3, ZeRO-1 style all-gather in the wire dtype)
             ("r50-f16-halfw", lay_r50, "f16", 719, dict(flags=4)),
             ("fused-r50-f16-halfw-carry", lay_r50, "f16", 720, dict(fused=True, flags=5)),
             ("fused-random-bf16-halfw", LY.random_layout(np.random.default_rng(8), 29), "bf16", 700,
              dict(fused=True, flags=4)),
             ("lpt-zipf-bf16-halfw", LY.skew1b("zipf", n_tensors=200, total=4_000_000), "bf16", 500,
              dict(flags=4, shard_policy="lpt")),
             # static backward-order groups (NEXT-f2)
             ("groups-r50-f16", lay_r50, "f16", 719, dict(shard_policy="groups", group_bytes=4 << 20)),
             ("groups-r50-int-overlap", lay_r50, "f16", 80, dict(kind="integer", shard_policy="groups",
                                                                 group_bytes=4 << 20, overlap="all")),
             ("groups-random-bf16-overlap-half", LY.random_layout(np.random.default_rng(8), 29), "bf16", 700,
              dict(shard_policy="groups", group_bytes=64 << 10, overlap="half")),
             ("groups-zipf-f32-carry-overlap", LY.skew1b("zipf", n_tensors=200, total=4_000_000), "f32", 500,
              dict(shard_policy="groups", group_bytes=1 << 20, flags=1, overlap="all")),
             ("groups-nan-in-split-layer", LY.skew1b("zipf", n_tensors=50, total=1_000_000), "f16", 100,
              dict(inject_nan="split", shard_policy="groups", group_bytes=256 << 10, overlap="all"))]
    sel = os.environ.get("DP_CASES")  # optional regex over case names
    if sel:
        cases = [c for c in cases if re.search(sel, c[0])]
    for name, lay, dtype, t, kw in cases:
        ok = 1
        try:
            run_case(name, lay, dtype, t, **kw)
        except Exception:  # keep every rank in lock-step: report, then stop together
            ok = 0
            report["failures"].append(f"{name}: {traceback.format_exc()[-1500:]}")
        flag = torch.tensor([ok], device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) == 0:
            print(json.dumps(report), flush=True)
            dist.destroy_process_group()
            sys.exit(1)
    # host-gradient entry point (dp_allreduce_lars_step_host_grad): five consecutive steps issued without
    # synchronizing — the fused path alternates its two symmetric gradient buffers, the copy of step k+1
    # overlapping step k — must equal, bit for bit, the same steps on device gradients; one step's gradient
    # has a NaN on one rank and is skipped everywhere
    for fused_h in (True, False):
        if sel and not re.search(sel, "host-grad-fused" if fused_h else "host-grad-nccl"):
            continue
        lay_h = LY.resnet50()[:40]
        kw_h = hp_kwargs(grad_dtype="f16", grad_scale=1.0 / (G.GRAD_PRESCALE * P), flags=1)
        hs = [PK.Lars([(x.numel, x.kind) for x in lay_h], device=local, nranks=P, **kw_h) for _ in range(2)]
        for hh in hs:
            hh.comm_init_torch()
        pk = lambda hh, a: torch.from_numpy(G.pack(a, hh.offsets, hh.padded_numel).view(a[0].dtype)).to(dev)
        grads = [G.grads(lay_h, rank, 30 + k, "f16") for k in range(5)]
        if rank == (1 % P):
            grads[2][3] = grads[2][3].copy()
            grads[2][3][0] = np.nan
        ws, ms = [], []
        for hh in hs:
            w0, m0 = pk(hh, G.weights(lay_h)), pk(hh, G.momentum(lay_h, 1e-3))
            if fused_h:
                wsym, _ = hh.dp_buffers()
                wsym.copy_(w0)
                w0 = wsym
            ws.append(w0)
            ms.append(m0)
        hosts = [torch.from_numpy(G.pack(gk, hs[0].offsets, hs[0].padded_numel)).pin_memory() for gk in grads]
        for k in range(5):
            hs[0].dp_allreduce_lars_step_host_grad(ws[0], hosts[k], ms[0], 700 + k)
        torch.cuda.synchronize()
        g_dev = hs[1].dp_buffers()[1] if fused_h else torch.empty_like(hosts[0], device=dev)
        for k in range(5):
            g_dev.copy_(hosts[k])
            hs[1].dp_allreduce_lars_step(ws[1], g_dev, ms[1], 700 + k)
            torch.cuda.synchronize()
            assert (hs[1].last_step_status() == 1) == (k == 2), (k, hs[1].last_step_status())
        same_h = torch.equal(ws[0], ws[1]) and torch.equal(ms[0], ms[1])
        report["cases"].append({"name": "host-grad-fused" if fused_h else "host-grad-nccl", "bitwise": same_h})
        if not same_h:
            report["failures"].append(f"host-grad ({'fused' if fused_h else 'nccl'}) differs from device path")
        for hh in hs:
            hh.close()
    # fused-path handshake stress: a tiny layout (3 tiles, far fewer than F1's grid, so most CTAs leave
    # without a tile) captured once in a CUDA graph with a device iteration and replayed DP_REPLAYS times
    # back to back with no host synchronization (the epoch / go / exit-barrier exchange runs every replay);
    # the result must equal, bit for bit, the same steps issued eagerly with host iterations, on every rank
    if not sel or re.search(sel, "fused-tiny-graph-replay"):
        n_rep = int(os.environ.get("DP_REPLAYS", "1000"))
        lay_s = LY.tiny()
        kw_s = hp_kwargs(grad_dtype="f16", grad_scale=1.0 / (G.GRAD_PRESCALE * P), flags=1)
        hs = [PK.Lars([(x.numel, x.kind) for x in lay_s], device=local, nranks=P, **kw_s) for _ in range(2)]
        pk = lambda hh, a: torch.from_numpy(G.pack(a, hh.offsets, hh.padded_numel).view(a[0].dtype)).to(dev)
        ws, ms = [], []
        for hh in hs:
            hh.comm_init_torch()
            wsym, gsym = hh.dp_buffers()
            wsym.copy_(pk(hh, G.weights(lay_s)))
            gsym.copy_(pk(hh, G.grads(lay_s, rank, 5, "f16")))
            ws.append(wsym)
            ms.append(pk(hh, G.momentum(lay_s, 1e-3)))
            hh.dp_allreduce_lars_step(wsym, gsym, ms[-1], 100)  # eager first step: connections, carried norms
        torch.cuda.synchronize()
        it_dev = torch.tensor([101], dtype=torch.int64, device=dev)
        side = torch.cuda.Stream(device=dev)
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=side, capture_error_mode="thread_local"):
            hs[0].dp_allreduce_lars_step_dev_iter(ws[0], hs[0].dp_buffers()[1], ms[0], it_dev, stream=side)
        for _ in range(n_rep):
            gr.replay()
        torch.cuda.synchronize()
        gr.reset()
        for k in range(n_rep):
            hs[1].dp_allreduce_lars_step(ws[1], hs[1].dp_buffers()[1], ms[1], 101 + k)
        torch.cuda.synchronize()
        same_s = all_same(ws[0])
        ok_s = (int(it_dev.item()) == 101 + n_rep and torch.equal(ws[0], ws[1]) and torch.equal(ms[0], ms[1])
                and bool(torch.isfinite(ws[0]).all()) and hs[0].last_step_status() == 0 and same_s)
        report["cases"].append({"name": "fused-tiny-graph-replay", "replays": n_rep, "bitwise": ok_s})
        if not ok_s:
            report["failures"].append("fused graph replays differ from the eager steps (or across ranks)")
        for hh in hs:
            hh.close()
    # parallel deterministic initialization: every rank initializes its own replica from
    # the same seed; the replicas are bitwise identical with zero bytes broadcast
    lay_i = LY.resnet50()
    hi = PK.Lars([(x.numel, x.kind, x.fan_in) for x in lay_i], device=local, nranks=P, **hp_kwargs())
    w_i = torch.zeros(hi.padded_numel, dtype=torch.float32, device=dev)  # padding is not written
    hi.init_weights(w_i, 100000)
    torch.cuda.synchronize()
    report["parallel_init_identical"] = all_same(w_i)
    assert report["parallel_init_identical"]
    hi.close()
    # layout disagreement across ranks -> LARS_ERR_LAYOUT on every rank (needs two ranks)
    report["layout_mismatch_rejected"] = None if P == 1 else False
    bad = LY.tiny() if rank == 0 else LY.tiny()[:2]
    if P > 1:
        h = PK.Lars([(x.numel, x.kind) for x in bad], device=local, nranks=P, **hp_kwargs())
        try:
            h.comm_init_torch()
            raise AssertionError("layout mismatch accepted")
        except PK.LarsError as e:
            assert e.status == 2, e
        report["layout_mismatch_rejected"] = True
    dist.barrier()
    out = os.environ.get("DP_REPORT_DIR")
    if out:
        with open(os.path.join(out, f"rank{rank}.json"), "w") as f:
            json.dump(report, f)
    print(json.dumps(report))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
