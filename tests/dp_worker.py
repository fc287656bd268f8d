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

    def run_case(name, lay, dtype, t, kind="random", inject_nan=False, **hpkw):
        kw = hp_kwargs(grad_dtype=dtype, grad_scale=1.0 / (G.GRAD_PRESCALE * P), **hpkw)
        h = PK.Lars([(x.numel, x.kind) for x in lay], device=local, nranks=P, **kw)
        h.comm_init_torch()
        w_l, m_l = G.weights(lay), G.momentum(lay, 1e-3)
        if kind == "integer":
            g_all = [G.integer_grads(lay, r, t, dtype) for r in range(P)]
        else:
            g_all = [G.grads(lay, r, t, dtype) for r in range(P)]
        if inject_nan and rank == 1 % P:
            g_all[rank][0] = g_all[rank][0].copy()
            g_all[rank][0][3] = np.nan
        pack = lambda a: torch.from_numpy(G.pack(a, h.offsets, h.padded_numel).view(
            np.int16 if a[0].dtype == np.uint16 else a[0].dtype)).to(dev)
        w, g, m = pack(w_l), pack(g_all[rank]), pack(m_l)
        g_before = g.clone()
        h.dp_allreduce_lars_step(w, g, m, t)
        torch.cuda.synchronize()
        res = {"name": name, "dtype": dtype, "t": t}
        same = all_same(w)  # collective: every rank calls it before any rank-local assertion
        assert torch.equal(g.view(torch.int16) if g.element_size() == 2 else g.view(torch.int32),
                           g_before.view(torch.int16) if g.element_size() == 2 else g_before.view(torch.int32)), \
            "dp step modified the caller's gradient"
        assert same, f"{name}: w differs across ranks after the all-gather"
        skipped = h.last_step_skipped()
        owner = h.tensor_owner()
        mine = [l for l in range(len(lay)) if owner[l] == rank]
        sizes = [x.numel for x in lay]
        wg = G.unpack(from_dev(w), h.offsets, sizes)
        mg = G.unpack(from_dev(m), h.offsets, sizes)
        if inject_nan:
            assert skipped, f"{name}: rank {rank} did not skip although rank 1 had a NaN"
            for l in mine:
                assert np.array_equal(wg[l], w_l[l]) and np.array_equal(mg[l], m_l[l])
            res["skipped_everywhere"] = True
            report["cases"].append(res)
            h.close()
            return
        assert not skipped
        # reduced shard vs brute-force sum over ranks
        red, b, e = h.reduced_grad()
        red = from_dev(red)
        kinds = [x.kind for x in lay]
        exact = {l: O.combine([g_all[r][l] for r in range(P)], 1.0) for l in mine}
        worst_sum = 0.0
        for l in mine:
            got = O.to_double(red[h.offsets[l] - b: h.offsets[l] - b + sizes[l]])
            if kind == "integer" and dtype != "bf16":
                assert np.array_equal(got, exact[l]), f"{name}: integer sum not exact (tensor {l})"
            else:
                bound = (P - 1) * (2.0 ** -11 if dtype == "f16" else 2.0 ** -8 if dtype == "bf16" else 2.0 ** -24) \
                    * sum(np.abs(O.to_double(g_all[r][l])) for r in range(P))
                err = np.abs(got - exact[l])
                ok = err <= bound + 0.0
                assert ok.all(), f"{name}: reduction error above the (P-1)u sum|g| bound at tensor {l}"
                worst_sum = max(worst_sum, float(np.max(np.where(bound > 0, err / np.maximum(bound, 1e-300), 0))))
        res["sum_err_over_bound"] = worst_sum
        # norms on the exact buffer K1 read (the reduced shard)
        hp = oracle_hp(kw)
        wn, gn, lam, coef = h.last_norms()
        s = kw["grad_scale"]
        for l in mine:
            got_red = red[h.offsets[l] - b: h.offsets[l] - b + sizes[l]]
            gate_norms(f"{name} ||w|| t{l}", [wn[l]], [O.l2norm(w_l[l])])
            gate_norms(f"{name} ||g|| t{l}", [gn[l]], [abs(s) * O.l2norm(O.to_double(got_red))])
        # the rank's w/m shard vs the oracle DP step with the exact sum
        r_or = O.dp_step([kinds[l] for l in mine], hp, t, [w_l[l] for l in mine],
                         [[g_all[r][l] for l in mine] for r in range(P)], [m_l[l] for l in mine])
        tol = TOL_F32 if dtype == "f32" else TOL_F16_DP if dtype == "f16" else TOL_BF16_DP
        if mine:
            res["m_err"] = gate(f"{name} m", np.concatenate([mg[l] for l in mine]), np.concatenate(r_or.m),
                                np.concatenate(r_or.m_env), tol)
            res["w_err"] = gate(f"{name} w", np.concatenate([wg[l] for l in mine]), np.concatenate(r_or.w),
                                np.concatenate(r_or.w_env), tol)
        report["cases"].append(res)
        h.close()

    lay_r50 = LY.resnet50()
    cases = [("tiny-int", LY.tiny(), "f16", 80, dict(kind="integer")),
             ("random-f16", LY.random_layout(np.random.default_rng(7), 37), "f16", 81, {}),
             ("random-bf16", LY.random_layout(np.random.default_rng(8), 29), "bf16", 700, {}),
             ("random-f32", LY.random_layout(np.random.default_rng(9), 23), "f32", 3, {}),
             ("r50-f16", lay_r50, "f16", 719, {}),
             ("r50-int", lay_r50, "f16", 1439, dict(kind="integer")),
             ("nan-on-rank1", LY.tiny(), "f16", 100, dict(inject_nan=True))]
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
    # layout disagreement across ranks -> LARS_ERR_LAYOUT on every rank
    bad = LY.tiny() if rank == 0 else LY.tiny()[:2]
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
