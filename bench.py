#!/usr/bin/env python
"""bench.py — ResNet-50 allreduce+LARS step: ms/step and params/s at N B200s, HBM / NVLink roofline.

Workloads (BASELINE.json):
  N = 1  configs[1]  "resnet50_f32_lars_step_1gpu": 161 tensors, 25,557,032 params, fp32 gradients,
                     lars_step (K1 norms + K2 fused update) on one B200.
  N > 1  configs[2]  "resnet50_f16_rs_lars_ag_dp{N}": fp16 gradients, NCCL reduce-scatter + sharded
                     LARS update + fp32 weight all-gather (dp_allreduce_lars_step), one process per GPU.

value = gradient elements combined and applied per second over the whole job: every rank contributes a
full local gradient of 25,557,032 params per step (data parallelism), so a step processes
N x 25,557,032 params; per-GPU work is fixed as N grows ("weak"). ms_per_step is the max over ranks.
Inputs stay resident in HBM for `value`; `e2e` copies each step's gradient from pinned host memory
(H2D) and reads the step status + per-layer norms back (D2H) inside the timed region.

`--impl reference` times the float64 CPU oracle (oracle/oracle.py) on the host cores — the only other
place bench.py executes oracle code besides the `cpu_baseline` leg.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ResNet-50 allreduce+LARS step ms & params/s at 1/2/4/8 B200; HBM/NVLink GB/s"
NVLINK_PEER_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md); 900 nominal
NVLINK_NOMINAL_GBS = 900.0
HBM_NOMINAL_GBS = 8000.0  # north_star "~8 TB/s"; the roofline uses MEASURED_PEAKS.json's copy rate
HP = dict(base_lr=32.0, eta=1e-3, momentum=0.9, weight_decay=5e-5, eps=0.0, warmup_epochs=5.0, poly_power=2.0,
          global_batch=81920)
T0 = 719  # mid-schedule start iteration (t cycles through the 1,440-step schedule)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--soak-s", type=float, default=1.5, help="untimed steps while clocks settle/sampling")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--layout", default="resnet50")
    ap.add_argument("--no-fused", action="store_true",
                    help="P > 1: use the NCCL collective path instead of the fused NVLink kernels")
    ap.add_argument("--buckets", type=int, default=0, help="NCCL path: K tile-aligned buckets (0/1 = single shot)")
    ap.add_argument("--no-carry", action="store_true",
                    help="disable LARS_FLAG_CARRY_WNORM (K2 carries sum(w^2) so K1 reads only g)")
    return ap.parse_args()


def workload_name(P: int, layout: str) -> str:
    return f"{layout}_f32_lars_step_1gpu" if P == 1 else f"{layout}_f16_rs_lars_ag_dp{P}"


def workload_config(P: int, layout: str, lay) -> dict:
    """The workload both arms report (identical dict for `--impl ours` and `--impl reference`)."""
    E = sum(t.numel for t in lay)
    gbytes = 4 if P == 1 else 2
    return {"workload": workload_name(P, layout), "layout": layout, "tensors": len(lay), "params": E,
            "grad_dtype": "f32" if P == 1 else "f16", "global_batch": HP["global_batch"],
            "iters": f"t=({T0}+k) mod 1440", "parallelism": f"dp{P}",
            "units": f"{P} x {E} gradient params combined+applied per step",
            "l2": f"inputs larger than L2: w+g+m = {(8 + gbytes) * E / 1e6:.0f} MB > 126 MB, no flush"}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class OneCore:
    """Runs the oracle on exactly one host core: the calling thread pinned to one CPU of its affinity set
    and BLAS/OpenMP pools limited to one thread (the oracle's NumPy ufuncs and math.fsum are single-threaded
    anyway); the previous affinity is restored on exit."""

    def __enter__(self):
        self.prev = os.sched_getaffinity(0)
        self.core = max(self.prev)  # away from core 0 (interrupts, the GPU driver's threads)
        os.sched_setaffinity(0, {self.core})
        self.pool = None
        try:
            from threadpoolctl import threadpool_limits

            self.pool = threadpool_limits(1)
        except ImportError:
            pass
        return self

    def __exit__(self, *exc):
        if self.pool is not None:
            self.pool.restore_original_limits()
        os.sched_setaffinity(0, self.prev)
        return False

    def describe(self) -> str:
        return f"pinned to CPU {self.core} of {len(self.prev)} ({cpu_model()})"


def measured_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the measured region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.lines, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------------------------- ours
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1903_12650_b200 as PK
    from synth import gen as G
    from synth import layouts as LY

    rank, P = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", args.gpus))
    local = int(os.environ.get("LOCAL_RANK", 0))
    assert P == args.gpus, f"WORLD_SIZE={P} but --gpus {args.gpus}"
    t_start = time.time()

    def phase(name):  # progress on stderr (locates a stall in a log)
        print(f"[bench] rank {rank} +{time.time() - t_start:.1f}s {name}", file=sys.stderr, flush=True)

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if P > 1:
        dist.init_process_group("nccl", device_id=dev)
    dtype = "f32" if P == 1 else "f16"
    lay = LY.by_name(args.layout)
    E = sum(t.numel for t in lay)
    carry = not args.no_carry
    mk = lambda flags: PK.Lars([(t.numel, t.kind) for t in lay], device=local, grad_dtype=dtype, nranks=P,
                               grad_scale=1.0 / (G.GRAD_PRESCALE * P), flags=flags, buckets=args.buckets, **HP)
    h = mk(PK.lars.FLAG_CARRY_WNORM if carry else 0)
    if P > 1:
        try:
            h.comm_init_torch()
        except PK.LarsError as e:  # fused-path setup failed (every rank alike): rerun on the NCCL path
            print(f"[bench] lars_comm_init failed ({e}); retrying with LARS_DP_FUSED=0", file=sys.stderr)
            h.close()
            os.environ["LARS_DP_FUSED"] = "0"
            h = mk(PK.lars.FLAG_CARRY_WNORM if carry else 0)
            h.comm_init_torch()
    phase("handle ready")
    gbytes = 4 if dtype == "f32" else 2

    def dev_flat(arrs):
        flat = G.pack(arrs, h.offsets, h.padded_numel)
        return torch.from_numpy(flat).to(dev)

    w_host, g_host, m_host = G.weights(lay), G.grads(lay, rank, 0, dtype), G.momentum(lay, 1e-3)
    w, g, m = dev_flat(w_host), dev_flat(g_host), dev_flat(m_host)
    w_n, g_n, fused = w, g, False
    if P > 1 and not args.no_fused:  # library-owned symmetric buffers -> fused NVLink path
        try:
            w_s, g_s = h.dp_buffers()
            w_s.copy_(w)
            g_s.copy_(g)
            w, g, fused = w_s, g_s, True
        except PK.LarsError:
            pass
    T = h.total_iters
    step = h.lars_step if P == 1 else h.dp_allreduce_lars_step
    stream = torch.cuda.current_stream()
    k = 0

    def run(n):
        nonlocal k
        for _ in range(n):
            step(w, g, m, (T0 + k) % T, stream)
            k += 1

    def barrier():
        if P > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if P == 1:
            return x
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    phase("warm-up")
    run(args.warmup)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    t_end = time.time() + args.soak_s
    while time.time() < t_end:
        run(20)
        torch.cuda.synchronize()
    nvl = None
    if P > 1:  # NVLink hardware byte counters around the timed steps (ncu cannot replay cross-rank kernels)
        try:
            from tools.nvlink_counters import NvlinkCounters

            nvl = NvlinkCounters(local)
            nvl = nvl if nvl.available() else None
        except Exception:  # noqa: BLE001 - counters are evidence, not part of the step
            nvl = None
    barrier()
    torch.cuda.synchronize()
    phase("timed steps")
    if nvl:
        try:
            nvl.start()
        except Exception:  # noqa: BLE001 - counters are evidence, not part of the step
            nvl = None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    run(args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    try:
        nvl1 = nvl.stop() if nvl else None
    except Exception:  # noqa: BLE001 - counters are evidence, not part of the step
        nvl1 = None
    barrier()
    clk = clocks.stop()
    ms_total = max_over_ranks(e0.elapsed_time(e1))
    assert not h.last_step_skipped(), "a timed step was skipped (non-finite) — invalid timing"
    ms_step = ms_total / args.steps

    # per-phase device times (library CUDA events on the same stream; separate pass)
    nprof = min(args.steps, 200)
    phase("phase timing")
    h.profile_enable(True)
    barrier()
    run(nprof)
    phases, nsteps = h.profile_read()
    h.profile_enable(False)
    ph = {kk: max_over_ranks(v / max(1, nsteps)) for kk, v in phases.items()}

    # comparison loops: P = 1 without carried weight norms (K1 re-reads w every step); P > 1 the NCCL
    # collective path (reduce-scatter + K1 + allreduce + K2 + all-gather) on ordinary buffers
    alt = {}

    def time_loop(fn, ww, gg):
        for i in range(args.warmup):
            fn(ww, gg, m, (T0 + i) % T, stream)
        barrier()
        torch.cuda.synchronize()
        e4, e5 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e4.record(stream)
        for i in range(args.steps):
            fn(ww, gg, m, (T0 + i) % T, stream)
        e5.record(stream)
        torch.cuda.synchronize()
        return round(max_over_ranks(e4.elapsed_time(e5)) / args.steps, 5)

    phase("alternatives")
    if P == 1 and carry:
        h0 = mk(0)
        alt["no_carry_ms_per_step"] = time_loop(h0.lars_step, w, g)
        h0.close()
        # the paper's wire format at N = 1: fp16 gradients (18 B/param update), carried norms
        hf = PK.Lars([(t.numel, t.kind) for t in lay], device=local, grad_dtype="f16", nranks=1,
                     grad_scale=1.0 / G.GRAD_PRESCALE, flags=PK.lars.FLAG_CARRY_WNORM, **HP)
        g16 = dev_flat(G.grads(lay, rank, 0, "f16"))
        alt["f16_grad_ms_per_step"] = time_loop(hf.lars_step, w, g16)
        hf.close()
        del g16
        h.invalidate_carried_norms()  # w was advanced by other handles
    if P > 1 and fused:
        alt["nccl_path_ms_per_step"] = time_loop(h.dp_allreduce_lars_step, w_n, g_n)
        # the NCCL path's phases, with reduce-scatter / all-gather bus bandwidth (nccl-tests convention:
        # busBW = (P-1)/P * bytes / t, bytes = the full buffer)
        h.profile_enable(True)
        barrier()
        for i in range(nprof):
            h.dp_allreduce_lars_step(w_n, g_n, m, (T0 + i) % T, stream)
        nph, nn = h.profile_read()
        h.profile_enable(False)
        nph = {kk: max_over_ranks(v / max(1, nn)) for kk, v in nph.items()}
        gb = h.padded_numel * (2 if dtype != "f32" else 4)
        alt["nccl_path_phases_ms"] = {kk: round(v, 5) for kk, v in nph.items()}
        alt["nccl_rs_busbw_GBps"] = round((P - 1) / P * gb / (nph["reduce_scatter"] * 1e-3) / 1e9, 1)
        alt["nccl_ag_busbw_GBps"] = round((P - 1) / P * h.padded_numel * 4 / (nph["all_gather"] * 1e-3) / 1e9, 1)
        alt["nccl_nvls_enable"] = os.environ.get("NCCL_NVLS_ENABLE", "default")
    if P > 1 and not args.buckets:
        # LARS_FLAG_HALF_WEIGHTS (NEXT-f3): fp32 masters stay on their shard, the all-gather moves the new
        # weights in the wire dtype into the compute-weight buffer (half the all-gather bytes)
        hh = mk((PK.lars.FLAG_CARRY_WNORM if carry else 0) | PK.lars.FLAG_HALF_WEIGHTS)
        hh.comm_init_torch()
        wh, gh = w_n.clone(), g_n
        if fused:
            wh, gh = hh.dp_buffers()
            wh.copy_(w_n)
            gh.copy_(g_n)
        mh = m.clone()
        for i in range(args.warmup):
            hh.dp_allreduce_lars_step(wh, gh, mh, (T0 + i) % T, stream)
        barrier()
        torch.cuda.synchronize()
        e6, e7 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e6.record(stream)
        for i in range(args.steps):
            hh.dp_allreduce_lars_step(wh, gh, mh, (T0 + i) % T, stream)
        e7.record(stream)
        torch.cuda.synchronize()
        alt["half_weights_ms_per_step"] = round(max_over_ranks(e6.elapsed_time(e7)) / args.steps, 5)
        alt["half_weights_path"] = "fused-nvlink" if fused else "nccl"
        hh.close()

    phase("e2e")
    # end to end through the public API with host gradients
    g_pin = torch.from_numpy(G.pack(g_host, h.offsets, h.padded_numel)).pin_memory()  # lands in g's buffer
    step_h = h.lars_step_host_grad if P == 1 else h.dp_allreduce_lars_step_host_grad
    ne = max(1, args.e2e_steps)
    step_h(w, g_pin, m, T0 % T, stream)
    torch.cuda.synchronize()
    barrier()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    for i in range(ne):
        step_h(w, g_pin, m, (T0 + i) % T, stream)
    e3.record(stream)
    torch.cuda.synchronize()
    skipped = h.last_step_skipped()
    assert not skipped
    ms_e2e = max_over_ranks(e2.elapsed_time(e3)) / ne
    h2d = h.padded_numel * gbytes
    # the same bytes as a bare pinned host -> device copy on this box: what the e2e step can at best reach
    g_dst = torch.empty(g_pin.shape, dtype=g_pin.dtype, device=dev)
    g_dst.copy_(g_pin, non_blocking=True)
    torch.cuda.synchronize()
    e8, e9 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e8.record()
    for i in range(ne):
        g_dst.copy_(g_pin, non_blocking=True)
    e9.record()
    torch.cuda.synchronize()
    ms_h2d = max_over_ranks(e8.elapsed_time(e9)) / ne
    del g_dst
    d2h = 4 + 2 * 8 * (len(lay) if P == 1 else sum(1 for o in h.tensor_owner() if o == rank))

    units = P * E
    value = units / (ms_step * 1e-3)
    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs")
    peak_note = "measured (MEASURED_PEAKS.json hbm_gbs)" if hbm else "fallback (B200_PROFILING.md 6.65 TB/s)"
    hbm = hbm or 6650.0
    shard_elems = sum(t.numel for t, o in zip(lay, h.tensor_owner()) if o == rank)
    upd_bytes = (4 + gbytes + 4 + 4 + 4) * shard_elems          # read w, g, m; write w, m
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            ns = json.load(f).get(workload_name(P, args.layout), {})
        traffic = ns.get("update_dram_bytes")
    except (OSError, ValueError):
        pass
    if P == 1:
        ach = upd_bytes / (ph["update"] * 1e-3) / 1e9
        roof = {"bound": "hbm", "kernel": "lars_update_kernel (K2)", "achieved": round(ach, 1), "peak": hbm,
                "unit": "GB/s", "frac": round(ach / hbm, 4), "traffic": traffic,
                "algorithmic_bytes_per_launch": upd_bytes, "launch_ms": round(ph["update"], 5),
                "peak_source": peak_note,
                # north_star framing: the nominal ~8 TB/s HBM3e peak beside the measured copy peak
                "frac_of_nominal": round(ach / HBM_NOMINAL_GBS, 4), "nominal_peak": HBM_NOMINAL_GBS}
    else:
        bus = (P - 1) / P * (gbytes + 4) * h.padded_numel
        if fused:  # F1 (reduce+norms) + F2 (update+gather): the transfers ARE these kernels
            coll_ms = ph["norms"] + ph["skip_allreduce"] + ph["update"]
            kname = "fused NVLink path: F1 reduce+norms, F2 update+gather"
        else:
            coll_ms = ph["reduce_scatter"] + ph["all_gather"]
            kname = "NCCL reduce-scatter + all-gather (C1+C2)"
        ach = bus / (coll_ms * 1e-3) / 1e9
        roof = {"bound": "nvlink", "kernel": kname, "achieved": round(ach, 1),
                "peak": NVLINK_PEER_GBS, "unit": "GB/s", "frac": round(ach / NVLINK_PEER_GBS, 4), "traffic": None,
                "bus_bytes_per_step": int(bus), "peak_source": "measured peer copy per direction, B200_PROFILING.md",
                "step_frac_of_bus_roofline": round(bus / NVLINK_PEER_GBS / 1e9 / (ms_step * 1e-3), 4),
                # north_star framing: 900 GB/s per direction nominal NVLink 5 beside the measured peer copy
                "frac_of_nominal": round(ach / NVLINK_NOMINAL_GBS, 4), "nominal_peak": NVLINK_NOMINAL_GBS}
    if nvl1:  # this rank's link traffic per step (hardware counters) vs the algorithmic bus bytes
        roof["nvlink_counters"] = {
            "tx_bytes_per_step": int(nvl1["tx"] / args.steps),
            "rx_bytes_per_step": int(nvl1["rx"] / args.steps),
            "interval_s": round(nvl1["seconds"], 6), "timed_region_s": round(ms_total * 1e-3, 6),
            # each direction of a GPU's links carries (P-1)/P * (gbytes + 4) * N per step: the shard pulls
            # (RS) and the weight stores (AG) leave on one direction and arrive on the other
            "algorithmic_bytes_per_direction": int(bus),
            "source": nvl.describe()}
    step_alg = (upd_bytes) / (ms_step * 1e-3) / 1e9
    two_pass = upd_bytes + (gbytes if carry else 4 + gbytes) * shard_elems
    out = {
        "metric": METRIC, "value": round(value, 1), "unit": "params/s", "n_gpus": P, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 5), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "grad_dtype": dtype, "data": "synthetic",
        "carry_wnorm": carry, **alt,
        "config": workload_config(P, args.layout, lay),
        "dp_path": None if P == 1 else ("fused-nvlink" if fused else "nccl"),
        "nccl_buckets": args.buckets if P > 1 else None,
        "phases_ms": {kk: round(v, 5) for kk, v in ph.items() if v > 0},
        "roofline": roof,
        "roofline_step": ({"bound": "hbm", "achieved": round(step_alg, 1), "peak": hbm, "unit": "GB/s",
                           "frac": round(step_alg / hbm, 4),
                           "note": "algorithmic update bytes (w,g,m read; w,m write) / whole step time",
                           # the whole-step skip on a non-finite norm (reading #13) needs every norm before any
                           # update, so g is streamed twice (norm pass, update pass; w too without carry)
                           "two_pass_bytes": int(two_pass),
                           "two_pass_frac": round(two_pass / (ms_step * 1e-3) / 1e9 / hbm, 4)} if P == 1 else
                          {"bound": "nvlink", "achieved": round(roof["bus_bytes_per_step"] / (ms_step * 1e-3) / 1e9, 1),
                           "peak": NVLINK_PEER_GBS, "unit": "GB/s",
                           "frac": roof["step_frac_of_bus_roofline"],
                           "note": "reduce-scatter + all-gather bus bytes per rank / whole step time"}),
        "e2e": {"value": round(units / (ms_e2e * 1e-3), 1), "unit": "params/s", "ms_per_step": round(ms_e2e, 4),
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "h2d_copy_ms": round(ms_h2d, 4), "frac_of_h2d_copy": round(ms_h2d / ms_e2e, 4)},
        "clocks": clk,
        "gpu_launches": (2 if fused else 2 if P == 1 else 3) * args.steps,
        "nccl_launches": (3 * args.steps) if (P > 1 and not fused) else 0,
    }
    if P == 1 and rank == 0 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(lay, w_host, [g_host], m_host, dtype, P)
    phase("done")
    if rank == 0:
        emit(out)
    if P > 1:
        # every rank releases its communicator and symmetric windows at the same point (not in garbage-
        # collection order at interpreter exit)
        torch.cuda.synchronize()
        dist.barrier()
        h.close()
        dist.destroy_process_group()
    del np


def cpu_baseline(lay, w, g_ranks, m, dtype, P):
    """The oracle, as it stands, on the host: one full ResNet-50 step (bounded ~10-30 s), 1 core."""
    from oracle import oracle as O
    from synth import gen as G

    hp = O.HParams(grad_scale=1.0 / (G.GRAD_PRESCALE * P), **HP)
    kinds = [t.kind for t in lay]
    with OneCore() as oc:
        t0 = time.perf_counter()
        O.step(kinds, hp, T0, w, g_ranks, m)
        dt = time.perf_counter() - t0
    E = sum(t.numel for t in lay)
    return {"value": round(P * E / dt, 1), "unit": "params/s", "cores": 1, "kind": "oracle",
            "cpu": cpu_model(),
            "sample": f"1 full {len(lay)}-tensor step ({E} params, {dtype} grads) in {dt:.2f} s, "
                      f"NumPy float64 + math.fsum, {oc.describe()}"}


# ----------------------------------------------------------------------------------------- reference
def run_reference(args):
    rank, P = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", args.gpus))
    if rank != 0:
        return
    from oracle import oracle as O
    from synth import gen as G
    from synth import layouts as LY

    dtype = "f32" if P == 1 else "f16"
    lay = LY.by_name(args.layout)
    E = sum(t.numel for t in lay)
    hp = O.HParams(grad_scale=1.0 / (G.GRAD_PRESCALE * P), **HP)
    oc = OneCore().__enter__()  # the whole reference arm runs on one host core
    # calibrate on the first few tensors, then size a contiguous tensor prefix so the whole run is bounded
    cal = lay[:40]
    wc, gc, mc = G.weights(cal), [G.grads(cal, r, 0, dtype) for r in range(P)], G.momentum(cal, 1e-3)
    t0 = time.perf_counter()
    O.step([t.kind for t in cal], hp, T0, wc, gc, mc)
    rate = sum(t.numel for t in cal) / (time.perf_counter() - t0)
    budget_s = 120.0
    want = max(200_000, min(E, int(rate * budget_s / max(1, args.steps + args.warmup))))
    n, acc = 0, 0
    while n < len(lay) and acc < want:
        acc += lay[n].numel
        n += 1
    sub = lay[:n]
    w, m = G.weights(sub), G.momentum(sub, 1e-3)
    g = [G.grads(sub, r, 0, dtype) for r in range(P)]
    kinds = [t.kind for t in sub]
    for i in range(args.warmup):
        O.step(kinds, hp, (T0 + i) % 1440, w, g, m)
    t0 = time.perf_counter()
    for i in range(args.steps):
        O.step(kinds, hp, (T0 + i) % 1440, w, g, m)
    dt = time.perf_counter() - t0
    value = P * acc * args.steps / dt
    sample = (f"first {n} of {len(lay)} tensors ({acc} of {E} params), {P} rank gradient(s) of {dtype}, "
              f"per step; NumPy float64 + math.fsum, {oc.describe()}")
    out = {"impl": "reference", "metric": METRIC, "value": round(value, 1), "unit": "params/s", "n_gpus": P,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 3),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "grad_dtype": dtype,
           "data": "synthetic",
           "config": workload_config(P, args.layout, lay),
           "cpu_baseline": {"value": round(value, 1), "unit": "params/s", "cores": 1, "kind": "oracle",
                            "cpu": cpu_model(), "sample": sample},
           "e2e": {"value": round(value, 1), "unit": "params/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(out)


_JSON_OUT = None


def emit(out: dict) -> None:
    """The one JSON line, on the process's real stdout (everything else written to fd 1 goes to stderr)."""
    f = _JSON_OUT or sys.stdout
    f.write(json.dumps(out) + "\n")
    f.flush()


def main():
    global _JSON_OUT
    # stdout carries exactly one JSON line: fd 1 is pointed at stderr for the whole run, so banners printed by
    # native libraries (NCCL's "NCCL version ...") cannot land on it; the JSON goes to a duplicate of the
    # original stdout
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
