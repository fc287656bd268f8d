"""Thin ctypes binding over ``liblars_b200.so`` (include/lars.h) — argument marshalling only.

Every step of the hot path runs inside the library's CUDA kernels / NCCL calls. torch is used for
plumbing only (device pointers, the current CUDA stream, process-group broadcast of the NCCL id).
There is no CPU fallback: if the shared library is missing this module raises on import of the
handle (``LarsLibraryMissing``).

Names follow the C ABI: ``lars_init`` -> :class:`Lars`, ``lars_step`` -> :meth:`Lars.lars_step`,
``dp_allreduce_lars_step`` -> :meth:`Lars.dp_allreduce_lars_step`.
"""
from __future__ import annotations

import ctypes
import os
import re
from ctypes import POINTER, byref, c_double, c_int32, c_int64, c_uint64, c_void_p

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "liblars_b200.so")
HEADER = os.path.join(os.path.dirname(PKG), "include", "lars.h")

KIND = {"weight": 0, "bias": 1, "bn_gamma": 2, "bn_beta": 3}
DTYPE = {"f32": 0, "f16": 1, "bf16": 2}
DTYPE_BYTES = {"f32": 4, "f16": 2, "bf16": 2}
SHARD_POLICY = {"contiguous": 0, "lpt": 1, "groups": 2}
DECAY = {"poly": 0, "step": 1}
FLAG_CARRY_WNORM = 1
FLAG_LR_AT_APPLY = 2
FLAG_HALF_WEIGHTS = 4  # LARS_FLAG_HALF_WEIGHTS


class LarsLibraryMissing(RuntimeError):
    pass


class LarsError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"{what}: {_strerror(status)} (status {status})")


class TensorDesc(ctypes.Structure):
    _fields_ = [("numel", c_int64), ("kind", c_int32), ("fan_in", c_int32)]


class HParams(ctypes.Structure):
    _fields_ = [("base_lr", c_double), ("eta", c_double), ("momentum", c_double), ("weight_decay", c_double),
                ("eps", c_double), ("warmup_epochs", c_double), ("poly_power", c_double),
                ("grad_scale", c_double), ("global_batch", c_int64), ("dataset_size", c_int64),
                ("total_epochs", c_int32), ("grad_dtype", c_int32), ("nranks", c_int32),
                ("tile_elems", c_int32), ("shard_policy", c_int32), ("flags", ctypes.c_uint32),
                ("buckets", c_int32), ("decay", c_int32), ("n_milestones", c_int32), ("reserved", c_int32),
                ("step_gamma", c_double), ("milestones", c_double * 8), ("group_bytes", c_int64)]


_lib = None


def load_library(path: str | None = None) -> ctypes.CDLL:
    """Loads the in-tree library (built by ``__graft_entry__.build()``). Fails loudly if absent.
    LARS_LIB=<path> selects another build of the same library (the device-checked diagnostics variant,
    ``python -m paper_1903_12650_b200.build --checked``)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("LARS_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise LarsLibraryMissing(f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    h = c_void_p
    sig = {
        "lars_hparams_default": (None, [POINTER(HParams)]),
        "lars_init": (c_int32, [POINTER(TensorDesc), c_int32, POINTER(HParams), c_int32, POINTER(h)]),
        "lars_layout": (c_int32, [h, POINTER(c_int64), POINTER(c_int64)]),
        "lars_schedule": (c_int32, [h, POINTER(c_int64), POINTER(c_int64), POINTER(c_int64)]),
        "lars_lr_at": (c_int32, [h, c_int64, POINTER(c_double)]),
        "lars_shard_range": (c_int32, [h, c_int32, POINTER(c_int64), POINTER(c_int64)]),
        "lars_tensor_owner": (c_int32, [h, POINTER(c_int32)]),
        "lars_layout_hash": (c_int32, [h, POINTER(c_uint64)]),
        "lars_check_work": (c_int32, [h, c_int32, POINTER(ctypes.c_char_p)]),
        "lars_init_weights": (c_int32, [h, c_void_p, ctypes.c_uint64, c_void_p]),
        "lars_work_info": (c_int32, [h, c_int32, POINTER(c_int32), POINTER(c_int32), POINTER(c_int32)]),
        "lars_step": (c_int32, [h, c_void_p, c_void_p, c_void_p, c_int64, c_void_p]),
        "lars_step_host_grad": (c_int32, [h, c_void_p, c_void_p, c_void_p, c_int64, c_void_p]),
        "lars_step_dev_iter": (c_int32, [h, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
        "dp_allreduce_lars_step_dev_iter": (c_int32, [h, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
        "lars_get_unique_id": (c_int32, [c_void_p]),
        "lars_comm_init": (c_int32, [h, c_int32, c_int32, c_void_p]),
        "dp_allreduce_lars_step": (c_int32, [h, c_void_p, c_void_p, c_void_p, c_int64, c_void_p]),
        "dp_allreduce_lars_step_host_grad": (c_int32, [h, c_void_p, c_void_p, c_void_p, c_int64, c_void_p]),
        "lars_profile_enable": (c_int32, [h, c_int32]),
        "lars_profile_read": (c_int32, [h, POINTER(c_double), POINTER(c_int64)]),
        "lars_reduced_grad": (c_int32, [h, POINTER(c_void_p), POINTER(c_int32), POINTER(c_int64), POINTER(c_int64)]),
        "lars_dp_buffers": (c_int32, [h, POINTER(c_void_p), POINTER(c_void_p)]),
        "lars_compute_weights": (c_int32, [h, POINTER(c_void_p)]),
        "lars_publish_compute_weights": (c_int32, [h, c_void_p, c_void_p]),
        "lars_groups": (c_int32, [h, POINTER(c_int32), POINTER(c_int64), POINTER(c_int64), POINTER(c_int32),
                                  POINTER(c_int32)]),
        "dp_group_ready": (c_int32, [h, c_void_p, c_int32, c_void_p]),
        "lars_group_trace_enable": (c_int32, [h, c_int32]),
        "lars_group_trace_read": (c_int32, [h, c_void_p, POINTER(c_double), POINTER(c_double), POINTER(c_double),
                                            POINTER(c_double)]),
        "lars_last_norms": (c_int32, [h, POINTER(c_double), POINTER(c_double), POINTER(c_double),
                                      POINTER(c_double)]),
        "lars_last_step_skipped": (c_int32, [h, POINTER(c_int32)]),
        "lars_invalidate_carried_norms": (c_int32, [h]),
        "lars_destroy": (c_int32, [h]),
        "lars_strerror": (ctypes.c_char_p, [c_int32]),
        "lars_version": (ctypes.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def declared_functions(header: str = HEADER) -> list[str]:
    """Names of every function the public header declares."""
    txt = open(header).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:lars_status_t|void|const char\*)\s+(\w+)\s*\(", txt, flags=re.M)))


def _strerror(status: int) -> str:
    try:
        return load_library().lars_strerror(status).decode()
    except Exception:  # pragma: no cover
        return "?"


def _check(status: int, what: str) -> None:
    if status != 0:
        raise LarsError(status, what)


def _ptr(x) -> int:
    """Device/host address of a torch tensor (or a raw int address)."""
    if x is None:
        return 0
    if isinstance(x, int):
        return x
    return x.data_ptr()


def _stream(stream) -> int:
    if stream is None:
        import torch

        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def default_hparams(**kw) -> HParams:
    hp = HParams()
    load_library().lars_hparams_default(byref(hp))
    for k, v in kw.items():
        if k == "grad_dtype" and isinstance(v, str):
            v = DTYPE[v]
        if k == "shard_policy" and isinstance(v, str):
            v = SHARD_POLICY[v]
        if k == "decay" and isinstance(v, str):
            v = DECAY[v]
        if k == "milestones":
            hp.n_milestones = len(v)
            for i, x in enumerate(v):
                hp.milestones[i] = float(x)
            continue
        if k == "momentum_form":
            continue
        setattr(hp, k, v)
    if "momentum_form" in kw:  # oracle-style spelling of LARS_FLAG_LR_AT_APPLY
        hp.flags = (hp.flags & ~FLAG_LR_AT_APPLY) | (FLAG_LR_AT_APPLY if kw["momentum_form"] == "apply" else 0)
    return hp


def get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load_library().lars_get_unique_id(buf), "lars_get_unique_id")
    return buf.raw


class _DevView:
    """__cuda_array_interface__ wrapper so torch can view library-owned device memory."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3}


class Lars:
    """A planned LARS step: ``lars_init`` on construction, ``lars_destroy`` on close()."""

    def __init__(self, tensors, device: int = 0, **hparams):
        """tensors: iterable of (numel, kind[, fan_in]) with kind a name in KIND or its code.
        hparams: fields of lars_hparams_t (base_lr is required)."""
        lib = load_library()
        descs = [(int(t[0]), KIND[t[1]] if isinstance(t[1], str) else int(t[1]), int(t[2]) if len(t) > 2 else 0)
                 for t in tensors]
        arr = (TensorDesc * max(1, len(descs)))(*[TensorDesc(n, k, f) for n, k, f in descs])
        self.hp = default_hparams(**hparams)
        self.n = len(descs)
        self.device = device
        self.grad_dtype = [k for k, v in DTYPE.items() if v == self.hp.grad_dtype][0]
        h = c_void_p()
        _check(lib.lars_init(arr, len(descs), byref(self.hp), device, byref(h)), "lars_init")
        self._h = h
        self._lib = lib
        offs = (c_int64 * self.n)()
        pad = c_int64()
        _check(lib.lars_layout(h, offs, byref(pad)), "lars_layout")
        self.offsets = [int(x) for x in offs]
        self.padded_numel = int(pad.value)
        ipe, T, W = c_int64(), c_int64(), c_int64()
        _check(lib.lars_schedule(h, byref(ipe), byref(T), byref(W)), "lars_schedule")
        self.ipe, self.total_iters, self.warmup_iters = int(ipe.value), int(T.value), int(W.value)
        self.rank = 0

    # ---- plan queries (no GPU needed) ----
    def lr_at(self, it: int) -> float:
        x = c_double()
        _check(self._lib.lars_lr_at(self._h, it, byref(x)), "lars_lr_at")
        return x.value

    def shard_range(self, rank: int) -> tuple[int, int]:
        b, e = c_int64(), c_int64()
        _check(self._lib.lars_shard_range(self._h, rank, byref(b), byref(e)), "lars_shard_range")
        return int(b.value), int(e.value)

    def groups(self) -> list[dict]:
        """Static backward-order groups: k = 0 is the group backward completes first (LARS_SHARD_GROUPS;
        any other policy: one group covering the whole flat buffer)."""
        n = c_int32()
        _check(self._lib.lars_groups(self._h, byref(n), None, None, None, None), "lars_groups")
        G = int(n.value)
        b, ln, f, l = (c_int64 * G)(), (c_int64 * G)(), (c_int32 * G)(), (c_int32 * G)()
        _check(self._lib.lars_groups(self._h, byref(n), b, ln, f, l), "lars_groups")
        return [{"begin": int(b[k]), "len": int(ln[k]), "first": int(f[k]), "last": int(l[k])} for k in range(G)]

    def tensor_owner(self) -> list[int]:
        o = (c_int32 * self.n)()
        _check(self._lib.lars_tensor_owner(self._h, o), "lars_tensor_owner")
        return list(o)

    def init_weights(self, w, seed: int, stream=None) -> None:
        """Parallel deterministic initialization: same seed -> same weights everywhere."""
        _check(self._lib.lars_init_weights(self._h, _ptr(w), seed, _stream(stream)), "lars_init_weights")

    def work_info(self, rank: int = -1) -> dict:
        t, sg, c = c_int32(), c_int32(), c_int32()
        _check(self._lib.lars_work_info(self._h, rank, byref(t), byref(sg), byref(c)), "lars_work_info")
        return {"tiles": t.value, "segments": sg.value, "chunks": c.value}

    def check_work(self, rank: int = -1) -> str:
        """Structural invariants of a work list (lars_check_work): 'ok', or raises LarsError with the reason."""
        why = ctypes.c_char_p()
        st = self._lib.lars_check_work(self._h, rank, byref(why))
        if st != 0:
            raise LarsError(st, f"lars_check_work: {why.value.decode() if why.value else '?'}")
        return why.value.decode()

    def layout_hash(self) -> int:
        x = c_uint64()
        _check(self._lib.lars_layout_hash(self._h, byref(x)), "lars_layout_hash")
        return int(x.value)

    # ---- steps ----
    def lars_step(self, w, g, m, it: int, stream=None) -> None:
        _check(self._lib.lars_step(self._h, _ptr(w), _ptr(g), _ptr(m), it, _stream(stream)), "lars_step")

    step = lars_step

    def lars_step_dev_iter(self, w, g, m, iter_dev, stream=None) -> None:
        """iter_dev: an int64 device tensor (or address); advanced by one by the step itself."""
        _check(self._lib.lars_step_dev_iter(self._h, _ptr(w), _ptr(g), _ptr(m), _ptr(iter_dev), _stream(stream)),
               "lars_step_dev_iter")

    def dp_allreduce_lars_step_dev_iter(self, w, g, m, iter_dev, stream=None) -> None:
        _check(self._lib.dp_allreduce_lars_step_dev_iter(self._h, _ptr(w), _ptr(g), _ptr(m), _ptr(iter_dev),
                                                         _stream(stream)), "dp_allreduce_lars_step_dev_iter")

    def lars_step_host_grad(self, w, g_host, m, it: int, stream=None) -> None:
        _check(self._lib.lars_step_host_grad(self._h, _ptr(w), _ptr(g_host), _ptr(m), it, _stream(stream)),
               "lars_step_host_grad")

    def comm_init(self, rank: int, nranks: int, uid: bytes) -> None:
        buf = ctypes.create_string_buffer(uid, 128)
        _check(self._lib.lars_comm_init(self._h, nranks, rank, buf), "lars_comm_init")
        self.rank = rank

    def comm_init_torch(self, group=None) -> None:
        """Creates the communicator, broadcasting the NCCL id over a torch.distributed group."""
        import torch
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        uid = get_unique_id() if rank == 0 else bytes(128)
        obj = [uid]
        dist.broadcast_object_list(obj, src=0, group=group)
        self.comm_init(rank, world, obj[0])
        del torch

    def dp_allreduce_lars_step(self, w, g, m, it: int, stream=None) -> None:
        _check(self._lib.dp_allreduce_lars_step(self._h, _ptr(w), _ptr(g), _ptr(m), it, _stream(stream)),
               "dp_allreduce_lars_step")

    dp_step = dp_allreduce_lars_step

    def dp_group_ready(self, g, group: int, stream=None) -> None:
        """Backward has written every tensor of `group` into g (ordered on `stream`): start its reduction."""
        _check(self._lib.dp_group_ready(self._h, _ptr(g), group, _stream(stream)), "dp_group_ready")

    def group_trace_enable(self, on: bool = True) -> None:
        _check(self._lib.lars_group_trace_enable(self._h, 1 if on else 0), "lars_group_trace_enable")

    def group_trace_read(self, ref_event=None) -> dict:
        """Last step, ms relative to ref_event (a recorded torch.cuda.Event with timing; None = group 0's
        ready event): ready/rs_start/rs_end per group, applied."""
        G = len(self.groups())
        r, a, b, ap = (c_double * G)(), (c_double * G)(), (c_double * G)(), c_double()
        ev = ref_event.cuda_event if ref_event is not None else None
        _check(self._lib.lars_group_trace_read(self._h, ev, r, a, b, byref(ap)), "lars_group_trace_read")
        return {"ready": list(r), "rs_start": list(a), "rs_end": list(b), "applied": ap.value}

    def dp_allreduce_lars_step_host_grad(self, w, g_host, m, it: int, stream=None) -> None:
        _check(self._lib.dp_allreduce_lars_step_host_grad(self._h, _ptr(w), _ptr(g_host), _ptr(m), it,
                                                          _stream(stream)), "dp_allreduce_lars_step_host_grad")

    # ---- per-phase device timing ----
    PHASES = ("reduce_scatter", "norms", "skip_allreduce", "update", "all_gather")

    def profile_enable(self, on: bool = True) -> None:
        _check(self._lib.lars_profile_enable(self._h, 1 if on else 0), "lars_profile_enable")

    def profile_read(self) -> tuple[dict, int]:
        ms = (c_double * 5)()
        n = c_int64()
        _check(self._lib.lars_profile_read(self._h, ms, byref(n)), "lars_profile_read")
        return dict(zip(self.PHASES, list(ms))), int(n.value)

    def reduced_grad(self):
        """torch view of the library's reduced-gradient shard (last dp step) and its [begin, end)."""
        import torch

        p, dt, b, e = c_void_p(), c_int32(), c_int64(), c_int64()
        _check(self._lib.lars_reduced_grad(self._h, byref(p), byref(dt), byref(b), byref(e)), "lars_reduced_grad")
        typestr = {0: "<f4", 1: "<f2", 2: "<i2"}[int(dt.value)]
        t = torch.as_tensor(_DevView(p.value, int(e.value - b.value), typestr), device=f"cuda:{self.device}")
        return t, int(b.value), int(e.value)

    def dp_buffers(self):
        """torch views of the library-owned symmetric weight and gradient buffers (fused NVLink path);
        raises LarsError(LARS_ERR_NO_COMM) when the fused path is unavailable."""
        import torch

        wp, gp = c_void_p(), c_void_p()
        _check(self._lib.lars_dp_buffers(self._h, byref(wp), byref(gp)), "lars_dp_buffers")
        dev = f"cuda:{self.device}"
        w = torch.as_tensor(_DevView(wp.value, self.padded_numel, "<f4"), device=dev)
        g = torch.as_tensor(_DevView(gp.value, self.padded_numel, {"f32": "<f4", "f16": "<f2", "bf16": "<i2"}[
            self.grad_dtype]), device=dev)
        return w, g

    def compute_weights(self):
        """LARS_FLAG_HALF_WEIGHTS: torch view of the library-owned compute weights (full layout, grad dtype;
        bf16 viewed as int16 bit patterns)."""
        import torch

        p = c_void_p()
        _check(self._lib.lars_compute_weights(self._h, byref(p)), "lars_compute_weights")
        typestr = {"f16": "<f2", "bf16": "<i2"}[self.grad_dtype]
        return torch.as_tensor(_DevView(p.value, self.padded_numel, typestr), device=f"cuda:{self.device}")

    def publish_compute_weights(self, w, stream=None) -> None:
        """LARS_FLAG_HALF_WEIGHTS: compute weights = RNE(w) for the whole layout (w: a full fp32 replica)."""
        _check(self._lib.lars_publish_compute_weights(self._h, _ptr(w), _stream(stream)),
               "lars_publish_compute_weights")

    # ---- readbacks (synchronize) ----
    def last_norms(self):
        a, b, c, d = [(c_double * self.n)(*([float("nan")] * self.n)) for _ in range(4)]
        _check(self._lib.lars_last_norms(self._h, a, b, c, d), "lars_last_norms")
        return list(a), list(b), list(c), list(d)

    def invalidate_carried_norms(self) -> None:
        _check(self._lib.lars_invalidate_carried_norms(self._h), "lars_invalidate_carried_norms")

    def last_step_status(self) -> int:
        """0 applied, 1 skipped (non-finite norm), 2 skipped (device iteration out of range)."""
        x = c_int32()
        _check(self._lib.lars_last_step_skipped(self._h, byref(x)), "lars_last_step_skipped")
        return int(x.value)

    def last_step_skipped(self) -> bool:
        return self.last_step_status() != 0

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.lars_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def lars_init(tensors, device: int = 0, **hparams) -> Lars:
    return Lars(tensors, device=device, **hparams)
