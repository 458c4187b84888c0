"""Thin Python binding of libspark (include/spark.h): argument marshalling only.

Every step of the hot path runs in the CUDA kernels of ``libspark.so``; this
module allocates the caller-owned device arena with torch, passes raw pointers
and the torch stream through ctypes, and turns status codes into exceptions.
It never falls back to a CPU path: if the library is missing it raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPARK_LIB") or os.path.join(_PKG, "lib", "libspark.so")  # SPARK_LIB: design-experiment builds

SPARK_OK, SPARK_ERR_ARG, SPARK_ERR_CUDA, SPARK_ERR_NCCL, SPARK_ERR_OOM, SPARK_ERR_NONPHYSICAL, SPARK_ERR_STATE = range(7)

# Every entry point declared in include/spark.h (checked by tests/test_abi.py).
EXPORTS = [
    "spark_abi_version", "spark_status_string", "spark_check_config", "spark_rank_grid", "spark_rank_box",
    "spark_halo_plan", "spark_required_bytes", "spark_nccl_unique_id", "spark_init", "spark_init_local_group",
    "spark_finalize", "spark_last_error", "spark_set_state", "spark_set_primitive", "spark_get_state",
    "spark_get_time", "spark_get_cfl_min", "spark_fill_guardcells", "spark_step", "spark_advance",
    "spark_step_group", "spark_stage_apply", "spark_profile_enable", "spark_profile_read",
    "spark_selftest_riemann", "spark_axpy", "spark_step_telescoping", "spark_run", "spark_set_time",
    "spark_step_host", "spark_telescoping_scratch_bytes", "spark_set_scratch", "spark_step_group_telescoping",
    "spark_telescoping_plan",
    "spark_amr_leaves", "spark_amr_required_bytes", "spark_amr_init", "spark_amr_finalize", "spark_amr_last_error",
    "spark_amr_set_state", "spark_amr_get_state", "spark_amr_fill_guardcells", "spark_amr_step", "spark_amr_get_time",
    "spark_amr_rank_leaves", "spark_amr_group_required_bytes", "spark_amr_init_local_group", "spark_amr_step_group",
]


class SparkError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{msg} (status {status})")
        self.status = status


class NonPhysicalError(SparkError):
    pass


class CConfig(ctypes.Structure):
    _fields_ = [
        ("ndim", ctypes.c_int32),
        ("nb", ctypes.c_int32 * 3),
        ("nblk", ctypes.c_int32 * 3),
        ("ng", ctypes.c_int32),
        ("lo", ctypes.c_double * 3),
        ("hi", ctypes.c_double * 3),
        ("bc", (ctypes.c_int32 * 2) * 3),
        ("recon", ctypes.c_int32),
        ("riemann", ctypes.c_int32),
        ("rk_stages", ctypes.c_int32),
        ("gamma", ctypes.c_double),
        ("cfl", ctypes.c_double),
        ("grav", ctypes.c_double * 3),
        ("shock_thresh", ctypes.c_double),
    ]


class CRefine(ctypes.Structure):
    _fields_ = [("rlo", ctypes.c_int32 * 3), ("rhi", ctypes.c_int32 * 3)]


class CFacePlan(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("side", ctypes.c_int32), ("peer", ctypes.c_int32),
                ("pad", ctypes.c_int32), ("cells", ctypes.c_int64)]


def to_cconfig(cfg: dict) -> CConfig:
    c = CConfig()
    c.ndim = int(cfg["ndim"])
    for d in range(3):
        c.nb[d] = int(cfg["nb"][d])
        c.nblk[d] = int(cfg["nblk"][d])
        c.lo[d] = float(cfg.get("lo", (0.0,) * 3)[d])
        c.hi[d] = float(cfg.get("hi", (1.0,) * 3)[d])
        bc = cfg.get("bc", ((1, 1),) * 3)[d]
        c.bc[d][0] = int(bc[0])
        c.bc[d][1] = int(bc[1])
    c.ng = int(cfg["ng"])
    c.recon = int(cfg.get("recon", 1))
    c.riemann = int(cfg.get("riemann", 1))
    c.rk_stages = int(cfg.get("rk_stages", 2))
    c.gamma = float(cfg.get("gamma", 1.4))
    c.cfl = float(cfg.get("cfl", 0.8))
    for d in range(3):
        c.grav[d] = float(cfg.get("grav", (0.0,) * 3)[d])
    c.shock_thresh = float(cfg.get("shock_thresh", 0.0))
    return c


_lib = None


def lib() -> ctypes.CDLL:
    """Load libspark.so (built by ``python -m paper_2401_03378_b200.build``); raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libspark.so not built ({LIB_PATH}); run `python -m paper_2401_03378_b200.build`")
    L = ctypes.CDLL(LIB_PATH)
    P, vp, i32, i64, d = ctypes.POINTER, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    cp = P(CConfig)
    sig = {
        "spark_abi_version": (i32, []),
        "spark_status_string": (ctypes.c_char_p, [i32]),
        "spark_check_config": (i32, [cp, i32]),
        "spark_rank_grid": (i32, [cp, i32, P(i32)]),
        "spark_rank_box": (i32, [cp, i32, i32, P(i32), P(i32)]),
        "spark_halo_plan": (i32, [cp, i32, i32, P(CFacePlan), P(i32)]),
        "spark_required_bytes": (i32, [cp, i32, i32, P(ctypes.c_size_t)]),
        "spark_nccl_unique_id": (i32, [P(ctypes.c_uint8)]),
        "spark_init": (i32, [cp, i32, i32, P(ctypes.c_uint8), i32, vp, vp, ctypes.c_size_t, P(vp)]),
        "spark_init_local_group": (i32, [cp, i32, i32, vp, P(vp), ctypes.c_size_t, P(vp)]),
        "spark_finalize": (i32, [vp]),
        "spark_last_error": (ctypes.c_char_p, [vp]),
        "spark_set_state": (i32, [vp, vp, i32]),
        "spark_set_primitive": (i32, [vp, vp, i32]),
        "spark_get_state": (i32, [vp, vp, i32]),
        "spark_get_time": (i32, [vp, P(d), P(i64), P(d)]),
        "spark_get_cfl_min": (i32, [vp, P(d)]),
        "spark_set_time": (i32, [vp, d, i64]),
        "spark_step_host": (i32, [vp, vp, vp, d, d, i32]),
        "spark_telescoping_scratch_bytes": (i32, [cp, i32, i32, P(ctypes.c_size_t)]),
        "spark_set_scratch": (i32, [vp, vp, ctypes.c_size_t]),
        "spark_telescoping_plan": (i32, [cp, i32, i32, P(i32), P(i64), P(i32), P(i32)]),
        "spark_step_group_telescoping": (i32, [P(vp), i32, d, d, P(d)]),
        "spark_amr_leaves": (i32, [cp, P(CRefine), P(i64), P(i64)]),
        "spark_amr_required_bytes": (i32, [cp, P(CRefine), P(ctypes.c_size_t)]),
        "spark_amr_init": (i32, [cp, P(CRefine), i32, vp, vp, ctypes.c_size_t, P(vp)]),
        "spark_amr_finalize": (i32, [vp]),
        "spark_amr_last_error": (ctypes.c_char_p, [vp]),
        "spark_amr_set_state": (i32, [vp, vp, i32]),
        "spark_amr_get_state": (i32, [vp, vp, i32]),
        "spark_amr_fill_guardcells": (i32, [vp, vp]),
        "spark_amr_step": (i32, [vp, d, d, P(d)]),
        "spark_amr_get_time": (i32, [vp, P(d), P(i64), P(d)]),
        "spark_amr_rank_leaves": (i32, [cp, P(CRefine), i32, i32, P(i64), P(i64)]),
        "spark_amr_group_required_bytes": (i32, [cp, P(CRefine), i32, P(ctypes.c_size_t)]),
        "spark_amr_init_local_group": (i32, [cp, P(CRefine), i32, i32, vp, P(vp), ctypes.c_size_t, P(vp)]),
        "spark_amr_step_group": (i32, [P(vp), i32, d, d, P(d)]),
        "spark_fill_guardcells": (i32, [vp, vp]),
        "spark_step": (i32, [vp, d, d, P(d)]),
        "spark_advance": (i32, [vp, i64, d, i32, P(i64)]),
        "spark_step_group": (i32, [P(vp), i32, d, d, P(d)]),
        "spark_stage_apply": (i32, [vp, vp, vp, d, d, d, vp]),
        "spark_profile_enable": (i32, [vp, i32]),
        "spark_profile_read": (i32, [vp, P(d), P(i64), P(i64)]),
        "spark_selftest_riemann": (i32, [i32, i32, i32, i32, d, i64, P(d), P(d), P(d)]),
        "spark_axpy": (i32, [i32, i32, i64, d, vp, vp, vp]),
        "spark_step_telescoping": (i32, [vp, d, d, P(d)]),
        "spark_run": (i32, [vp, i64, d, d]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def _check(st: int, ctx=None, what: str = ""):
    if st == SPARK_OK:
        return
    msg = lib().spark_last_error(ctx).decode() if ctx else ""
    text = f"{what}: {lib().spark_status_string(st).decode()}" + (f" — {msg}" if msg else "")
    if st == SPARK_ERR_NONPHYSICAL:
        raise NonPhysicalError(st, text)
    raise SparkError(st, text)


# ------------------------------------------------------------ host-only queries
def telescoping_plan(cfg: dict, rank: int, nranks: int):
    """(peer[27], cells[27], ops) of the telescoping shell exchange (host only);
    ops: ("recv" | "send", direction) in posting order."""
    c = to_cconfig(cfg)
    peer = (ctypes.c_int32 * 27)()
    cells = (ctypes.c_int64 * 27)()
    ops = (ctypes.c_int32 * 54)()
    n = ctypes.c_int32()
    _check(lib().spark_telescoping_plan(ctypes.byref(c), rank, nranks, peer, cells, ops, ctypes.byref(n)),
           what="telescoping_plan")
    return list(peer), list(cells), [("recv", o - 1) if o > 0 else ("send", -o - 1) for o in ops[:n.value]]


def check_config(cfg: dict, nranks: int = 1) -> bool:
    c = to_cconfig(cfg)
    return lib().spark_check_config(ctypes.byref(c), nranks) == SPARK_OK


def rank_grid(cfg: dict, nranks: int):
    c = to_cconfig(cfg)
    out = (ctypes.c_int32 * 3)()
    _check(lib().spark_rank_grid(ctypes.byref(c), nranks, out), what="rank_grid")
    return tuple(out)


def rank_box(cfg: dict, rank: int, nranks: int):
    c = to_cconfig(cfg)
    lo, n = (ctypes.c_int32 * 3)(), (ctypes.c_int32 * 3)()
    _check(lib().spark_rank_box(ctypes.byref(c), rank, nranks, lo, n), what="rank_box")
    return tuple(lo), tuple(n)


def halo_plan(cfg: dict, rank: int, nranks: int):
    c = to_cconfig(cfg)
    faces = (CFacePlan * 6)()
    n = ctypes.c_int32()
    _check(lib().spark_halo_plan(ctypes.byref(c), rank, nranks, faces, ctypes.byref(n)), what="halo_plan")
    return [dict(dim=f.dim, side=f.side, peer=f.peer, cells=f.cells) for f in faces[: n.value]]


def required_bytes(cfg: dict, rank: int = 0, nranks: int = 1) -> int:
    c = to_cconfig(cfg)
    b = ctypes.c_size_t()
    _check(lib().spark_required_bytes(ctypes.byref(c), rank, nranks, ctypes.byref(b)), what="required_bytes")
    return b.value


def nccl_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(lib().spark_nccl_unique_id(buf), what="nccl_unique_id")
    return bytes(buf)


def selftest_riemann(kind: int, ndim: int, direction: int, gamma: float, wl: np.ndarray, wr: np.ndarray,
                     device: int = 0) -> np.ndarray:
    """Device Riemann fluxes for face states wl, wr ([n][ndim+2], unrotated primitive)."""
    wl = np.ascontiguousarray(wl, dtype=np.float64)
    wr = np.ascontiguousarray(wr, dtype=np.float64)
    f = np.empty_like(wl)
    dp = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    _check(lib().spark_selftest_riemann(device, kind, ndim, direction, gamma, wl.shape[0], dp(wl), dp(wr), dp(f)),
           what="selftest_riemann")
    return f


AXPY_VARIANTS = {0: "axpy_increment_1", 1: "axpy_increment_threads", 2: "axpy_single_iter", 3: "axpy_vec2"}


def axpy(variant: int, a: float, x, y, stream=None):
    """y <- a x + y on the device (torch float64 CUDA tensors), paper AXPY mapping `variant`."""
    import torch

    assert x.dtype == torch.float64 and y.dtype == torch.float64 and x.is_cuda and y.is_cuda
    assert x.numel() == y.numel() and x.is_contiguous() and y.is_contiguous()
    st = stream if stream is not None else torch.cuda.current_stream(y.device)
    _check(lib().spark_axpy(y.device.index, variant, y.numel(), a, ctypes.c_void_p(x.data_ptr()),
                            ctypes.c_void_p(y.data_ptr()), ctypes.c_void_p(st.cuda_stream)), what="axpy")
    return y


def local_shape(cfg: dict, rank: int = 0, nranks: int = 1):
    """Canonical shape (nvar, nblocks_local, nb_z, nb_y, nb_x) of one rank's state."""
    _, n = rank_box(cfg, rank, nranks)
    nb = cfg["nb"]
    return (int(cfg["ndim"]) + 2, n[0] * n[1] * n[2], nb[2], nb[1], nb[0])


# ------------------------------------------------------------------ the context
class Spark:
    """One libspark context (one rank on one GPU).  State lives in a torch-owned arena."""

    def __init__(self, cfg: dict, rank: int = 0, nranks: int = 1, nccl_id: Optional[bytes] = None,
                 device: Optional[int] = None, stream=None, _handle=None, _arena=None):
        import torch

        self.torch = torch
        self.cfg = dict(cfg)
        self.rank, self.nranks = rank, nranks
        self.device = torch.cuda.current_device() if device is None else device
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.shape = local_shape(cfg, rank, nranks)
        self.nccl = False
        self.scratch = None
        if _handle is not None:
            self.ctx, self.arena = _handle, _arena
            return
        nbytes = required_bytes(cfg, rank, nranks)
        self.arena = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{self.device}")
        c = to_cconfig(cfg)
        h = ctypes.c_void_p()
        idp = None
        self.nccl = nccl_id is not None
        if nccl_id is not None:
            idp = (ctypes.c_uint8 * 128).from_buffer_copy(nccl_id)
        _check(lib().spark_init(ctypes.byref(c), rank, nranks, idp, self.device,
                                ctypes.c_void_p(self.stream.cuda_stream), ctypes.c_void_p(self.arena.data_ptr()),
                                nbytes, ctypes.byref(h)), what="spark_init")
        self.ctx = h

    # ---- state I/O
    def _ptr(self, x, writable=False):
        torch = self.torch
        if isinstance(x, torch.Tensor):
            assert x.dtype == torch.float64 and x.is_contiguous()
            assert x.numel() == int(np.prod(self.shape)), (x.shape, self.shape)
            return ctypes.c_void_p(x.data_ptr()), int(x.is_cuda)
        assert isinstance(x, np.ndarray) and x.dtype == np.float64 and x.flags["C_CONTIGUOUS"]
        assert x.size == int(np.prod(self.shape))
        return ctypes.c_void_p(x.ctypes.data), 0

    def set_state(self, U):
        p, dev = self._ptr(U)
        _check(lib().spark_set_state(self.ctx, p, dev), self.ctx, "set_state")
        if not dev:
            self.sync()

    def set_primitive(self, W):
        p, dev = self._ptr(W)
        _check(lib().spark_set_primitive(self.ctx, p, dev), self.ctx, "set_primitive")
        if not dev:
            self.sync()

    def get_state(self, out=None):
        """Current U^n; returns a new CUDA tensor unless `out` (tensor or ndarray) is given."""
        torch = self.torch
        if out is None:
            out = torch.empty(self.shape, dtype=torch.float64, device=f"cuda:{self.device}")
        p, dev = self._ptr(out, True)
        _check(lib().spark_get_state(self.ctx, p, dev), self.ctx, "get_state")
        return out

    def sync(self):
        self.stream.synchronize()

    # ---- hot path
    def step(self, dt: float = 0.0, t_end: float = 0.0, sync: bool = False):
        if sync:
            d = ctypes.c_double()
            _check(lib().spark_step(self.ctx, dt, t_end, ctypes.byref(d)), self.ctx, "step")
            return d.value
        _check(lib().spark_step(self.ctx, dt, t_end, None), self.ctx, "step")
        return None

    def enable_tiles(self):
        """Allocate the HBM-tile scratch (torch-owned) and select the tile
        telescoping path (3-D / multi-rank; spark_set_scratch)."""
        c = to_cconfig(self.cfg)
        n = ctypes.c_size_t()
        _check(lib().spark_telescoping_scratch_bytes(ctypes.byref(c), self.rank, self.nranks, ctypes.byref(n)),
               what="telescoping_scratch_bytes")
        self.scratch = self.torch.empty(max(n.value, 256), dtype=self.torch.uint8, device=f"cuda:{self.device}")
        _check(lib().spark_set_scratch(self.ctx, ctypes.c_void_p(self.scratch.data_ptr()), n.value), self.ctx,
               "set_scratch")

    def step_host(self, U_in, U_out, dt: float = 0.0, t_end: float = 0.0, nchunks: int = 8):
        """One step from host memory to host memory (spark_step_host), with the
        copies pipelined; asynchronous: both arrays must stay alive (and pinned
        for overlap) until sync()."""
        for x in (U_in, U_out):
            if not (isinstance(x, np.ndarray) and x.dtype == np.float64 and x.flags["C_CONTIGUOUS"]
                    and x.size == int(np.prod(self.shape))):
                raise ValueError("host state must be a C-contiguous float64 array of the local shape")
        _check(lib().spark_step_host(self.ctx, ctypes.c_void_p(U_in.ctypes.data), ctypes.c_void_p(U_out.ctypes.data),
                                     dt, t_end, nchunks), self.ctx, "step_host")

    def run(self, nsteps: int, dt: float = 0.0, t_end: float = 0.0):
        """nsteps steps, asynchronous; CUDA-graph replay on a non-default stream."""
        _check(lib().spark_run(self.ctx, nsteps, dt, t_end), self.ctx, "run")

    def step_telescoping(self, dt: float = 0.0, t_end: float = 0.0, sync: bool = False):
        """One telescoping SSP-RK step: on chip for 1-D/2-D single-rank contexts,
        through HBM tiles (scratch allocated on first use) for 3-D, NCCL
        contexts, or after enable_tiles()."""
        if getattr(self, "scratch", None) is None and (self.cfg["ndim"] == 3 or self.nranks > 1 or self.nccl):
            self.enable_tiles()
        if sync:
            d = ctypes.c_double()
            _check(lib().spark_step_telescoping(self.ctx, dt, t_end, ctypes.byref(d)), self.ctx, "step_telescoping")
            return d.value
        _check(lib().spark_step_telescoping(self.ctx, dt, t_end, None), self.ctx, "step_telescoping")
        return None

    def advance(self, max_steps: int, t_end: float = 0.0, check_every: int = 16) -> int:
        n = ctypes.c_int64()
        _check(lib().spark_advance(self.ctx, max_steps, t_end, check_every, ctypes.byref(n)), self.ctx, "advance")
        return n.value

    def fill_guardcells(self, padded: bool = True):
        torch = self.torch
        out = None
        if padded:
            g = [self.cfg["ng"] if d < self.cfg["ndim"] else 0 for d in range(3)]
            nb = self.cfg["nb"]
            out = torch.empty((self.shape[0], self.shape[1], nb[2] + 2 * g[2], nb[1] + 2 * g[1], nb[0] + 2 * g[0]),
                              dtype=torch.float64, device=f"cuda:{self.device}")
        _check(lib().spark_fill_guardcells(self.ctx, ctypes.c_void_p(out.data_ptr()) if padded else None),
               self.ctx, "fill_guardcells")
        return out

    def stage_apply(self, U_prev, U_n, a: float, b: float, dt: float, out=None):
        """One fused stage on device tensors (canonical layout); synchronises
        the library stream before returning, so `out` is ready to read."""
        torch = self.torch
        if out is None:
            out = torch.empty_like(U_prev)
        for name, x in (("U_prev", U_prev), ("U_n", U_n), ("out", out)):
            if x is None and name == "U_n":
                if a != 0.0:
                    raise ValueError("U_n is required when a != 0")
                continue
            if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.float64 and x.is_contiguous()
                    and x.numel() == int(np.prod(self.shape))):
                raise ValueError(f"{name} must be a contiguous float64 CUDA tensor of {int(np.prod(self.shape))} "
                                 "elements")
        _check(lib().spark_stage_apply(self.ctx, ctypes.c_void_p(U_prev.data_ptr()),
                                       ctypes.c_void_p(U_n.data_ptr()) if U_n is not None else None,
                                       a, b, dt, ctypes.c_void_p(out.data_ptr())), self.ctx, "stage_apply")
        self.sync()
        return out

    def time(self):
        t, dt = ctypes.c_double(), ctypes.c_double()
        n = ctypes.c_int64()
        _check(lib().spark_get_time(self.ctx, ctypes.byref(t), ctypes.byref(n), ctypes.byref(dt)), self.ctx, "time")
        return t.value, n.value, dt.value

    def set_time(self, t: float, steps: int):
        """Restore t and the step count after set_state (checkpoint/resume)."""
        _check(lib().spark_set_time(self.ctx, float(t), int(steps)), self.ctx, "set_time")

    def cfl_min(self) -> float:
        v = ctypes.c_double()
        _check(lib().spark_get_cfl_min(self.ctx, ctypes.byref(v)), self.ctx, "cfl_min")
        return v.value

    def profile(self, on: bool = True):
        _check(lib().spark_profile_enable(self.ctx, int(on)), self.ctx, "profile_enable")

    def profile_read(self):
        ms = ctypes.c_double()
        n, tot = ctypes.c_int64(), ctypes.c_int64()
        _check(lib().spark_profile_read(self.ctx, ctypes.byref(ms), ctypes.byref(n), ctypes.byref(tot)),
               self.ctx, "profile_read")
        return ms.value, n.value, tot.value

    def close(self):
        if getattr(self, "ctx", None):
            _check(lib().spark_finalize(self.ctx), None, "finalize")
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LocalGroup:
    """nranks virtual ranks on one GPU (spark_init_local_group / spark_step_group)."""

    def __init__(self, cfg: dict, nranks: int, device: Optional[int] = None, stream=None):
        import torch

        self.torch = torch
        device = torch.cuda.current_device() if device is None else device
        stream = stream if stream is not None else torch.cuda.current_stream(device)
        nbytes = max(required_bytes(cfg, r, nranks) for r in range(nranks))
        self.arenas = [torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{device}") for _ in range(nranks)]
        ptrs = (ctypes.c_void_p * nranks)(*[a.data_ptr() for a in self.arenas])
        outs = (ctypes.c_void_p * nranks)()
        c = to_cconfig(cfg)
        _check(lib().spark_init_local_group(ctypes.byref(c), nranks, device, ctypes.c_void_p(stream.cuda_stream),
                                            ptrs, nbytes, outs), what="init_local_group")
        self.ranks = [Spark(cfg, r, nranks, device=device, stream=stream, _handle=ctypes.c_void_p(outs[r]),
                            _arena=self.arenas[r]) for r in range(nranks)]
        self._handles = (ctypes.c_void_p * nranks)(*[outs[r] for r in range(nranks)])

    def step(self, dt: float = 0.0, t_end: float = 0.0, sync: bool = False):
        d = ctypes.c_double()
        _check(lib().spark_step_group(self._handles, len(self.ranks), dt, t_end, ctypes.byref(d) if sync else None),
               self.ranks[0].ctx, "step_group")
        return d.value if sync else None

    def step_telescoping(self, dt: float = 0.0, t_end: float = 0.0, sync: bool = False):
        """Telescoping step of the group (one shell exchange per step); the
        members' tile scratch is allocated on first use."""
        for r in self.ranks:
            if getattr(r, "scratch", None) is None:
                r.enable_tiles()
        d = ctypes.c_double()
        _check(lib().spark_step_group_telescoping(self._handles, len(self.ranks), dt, t_end,
                                                  ctypes.byref(d) if sync else None),
               self.ranks[0].ctx, "step_group_telescoping")
        return d.value if sync else None

    def close(self):
        for r in self.ranks:
            r.close()


# ------------------------------------------------ NEXT N3: static two-level AMR
def _refine(rlo, rhi) -> CRefine:
    r = CRefine()
    for d in range(3):
        r.rlo[d] = int(rlo[d])
        r.rhi[d] = int(rhi[d])
    return r


def amr_leaves(cfg: dict, rlo, rhi):
    c, r = to_cconfig(cfg), _refine(rlo, rhi)
    nc, nf = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().spark_amr_leaves(ctypes.byref(c), ctypes.byref(r), ctypes.byref(nc), ctypes.byref(nf)),
           what="amr_leaves")
    return nc.value, nf.value


def amr_rank_leaves(cfg: dict, rlo, rhi, rank: int, nranks: int):
    """(first leaf, leaf count) of `rank` in a group of nranks."""
    c, r = to_cconfig(cfg), _refine(rlo, rhi)
    a, n = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().spark_amr_rank_leaves(ctypes.byref(c), ctypes.byref(r), rank, nranks, ctypes.byref(a),
                                       ctypes.byref(n)), what="amr_rank_leaves")
    return a.value, n.value


class Amr:
    """A static two-level refinement (spark_amr_*): coarse blocks [rlo, rhi)
    refined by 2; state U[v][leaf][k][j][i] (coarse leaves, then fine)."""

    def __init__(self, cfg: dict, rlo, rhi, device: Optional[int] = None, stream=None, _handle=None, _arena=None,
                 _nleaf=None):
        import torch

        self.torch = torch
        self.cfg = dict(cfg)
        self.device = torch.cuda.current_device() if device is None else device
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        if _handle is not None:  # a member of an AmrGroup
            self.ctx, self.arena, self.nleaf = _handle, _arena, _nleaf
            self.shape = (cfg["ndim"] + 2, self.nleaf) + tuple(reversed(cfg["nb"]))
            return
        nc, nf = amr_leaves(cfg, rlo, rhi)
        self.nleaf = nc + nf
        self.shape = (cfg["ndim"] + 2, self.nleaf) + tuple(reversed(cfg["nb"]))
        c, r = to_cconfig(cfg), _refine(rlo, rhi)
        nbytes = ctypes.c_size_t()
        _check(lib().spark_amr_required_bytes(ctypes.byref(c), ctypes.byref(r), ctypes.byref(nbytes)),
               what="amr_required_bytes")
        self.arena = torch.empty(nbytes.value, dtype=torch.uint8, device=f"cuda:{self.device}")
        h = ctypes.c_void_p()
        st = lib().spark_amr_init(ctypes.byref(c), ctypes.byref(r), self.device,
                                  ctypes.c_void_p(self.stream.cuda_stream), ctypes.c_void_p(self.arena.data_ptr()),
                                  nbytes.value, ctypes.byref(h))
        _check(st, what="amr_init")
        self.ctx = h

    def _chk(self, st, what):
        if st != SPARK_OK:
            msg = lib().spark_amr_last_error(self.ctx).decode()
            text = f"{what}: {lib().spark_status_string(st).decode()} — {msg}"
            raise (NonPhysicalError if st == SPARK_ERR_NONPHYSICAL else SparkError)(st, text)

    def set_state(self, U):
        torch = self.torch
        if isinstance(U, torch.Tensor):
            if not (U.is_cuda and U.dtype == torch.float64 and U.is_contiguous() and tuple(U.shape) == self.shape):
                raise ValueError("U must be a contiguous float64 CUDA tensor of the leaf shape")
            self._chk(lib().spark_amr_set_state(self.ctx, ctypes.c_void_p(U.data_ptr()), 1), "amr_set_state")
        else:
            U = np.ascontiguousarray(U, dtype=np.float64)
            if U.shape != self.shape:
                raise ValueError(f"U has shape {U.shape}, expected {self.shape}")
            self._chk(lib().spark_amr_set_state(self.ctx, ctypes.c_void_p(U.ctypes.data), 0), "amr_set_state")
            self.stream.synchronize()

    def get_state(self):
        out = np.empty(self.shape, dtype=np.float64)
        self._chk(lib().spark_amr_get_state(self.ctx, ctypes.c_void_p(out.ctypes.data), 0), "amr_get_state")
        return out

    def fill_guardcells(self):
        ng = self.cfg["ng"]
        nd = self.cfg["ndim"]
        pn = [self.cfg["nb"][d] + (2 * ng if d < nd else 0) for d in range(3)]
        out = self.torch.empty((nd + 2, self.nleaf, pn[2], pn[1], pn[0]), dtype=self.torch.float64,
                               device=f"cuda:{self.device}")
        self._chk(lib().spark_amr_fill_guardcells(self.ctx, ctypes.c_void_p(out.data_ptr())), "amr_fill")
        self.stream.synchronize()
        return out

    def step(self, dt: float = 0.0, t_end: float = 0.0, sync: bool = False):
        d = ctypes.c_double()
        self._chk(lib().spark_amr_step(self.ctx, dt, t_end, ctypes.byref(d) if sync else None), "amr_step")
        return d.value if sync else None

    def time(self):
        t, dt = ctypes.c_double(), ctypes.c_double()
        n = ctypes.c_int64()
        self._chk(lib().spark_amr_get_time(self.ctx, ctypes.byref(t), ctypes.byref(n), ctypes.byref(dt)), "amr_time")
        return t.value, n.value, dt.value

    def close(self):
        if getattr(self, "ctx", None):
            lib().spark_amr_finalize(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class AmrGroup:
    """nranks virtual ranks of a static two-level refinement on one GPU
    (spark_amr_init_local_group / spark_amr_step_group); member r owns the
    leaves amr_rank_leaves(cfg, rlo, rhi, r, nranks)."""

    def __init__(self, cfg: dict, rlo, rhi, nranks: int, device: Optional[int] = None, stream=None):
        import torch

        device = torch.cuda.current_device() if device is None else device
        stream = stream if stream is not None else torch.cuda.current_stream(device)
        c, r = to_cconfig(cfg), _refine(rlo, rhi)
        nbytes = ctypes.c_size_t()
        _check(lib().spark_amr_group_required_bytes(ctypes.byref(c), ctypes.byref(r), nranks, ctypes.byref(nbytes)),
               what="amr_group_required_bytes")
        self.arenas = [torch.empty(nbytes.value, dtype=torch.uint8, device=f"cuda:{device}") for _ in range(nranks)]
        ptrs = (ctypes.c_void_p * nranks)(*[a.data_ptr() for a in self.arenas])
        outs = (ctypes.c_void_p * nranks)()
        _check(lib().spark_amr_init_local_group(ctypes.byref(c), ctypes.byref(r), nranks, device,
                                                ctypes.c_void_p(stream.cuda_stream), ptrs, nbytes.value, outs),
               what="amr_init_local_group")
        self.leaves = [amr_rank_leaves(cfg, rlo, rhi, q, nranks) for q in range(nranks)]
        self.ranks = [Amr(cfg, rlo, rhi, device=device, stream=stream, _handle=ctypes.c_void_p(outs[q]),
                          _arena=self.arenas[q], _nleaf=self.leaves[q][1]) for q in range(nranks)]
        self._handles = (ctypes.c_void_p * nranks)(*[outs[q] for q in range(nranks)])

    def step(self, dt: float = 0.0, t_end: float = 0.0, sync: bool = False):
        d = ctypes.c_double()
        self.ranks[0]._chk(lib().spark_amr_step_group(self._handles, len(self.ranks), dt, t_end,
                                                      ctypes.byref(d) if sync else None), "amr_step_group")
        return d.value if sync else None

    def close(self):
        for a in self.ranks:
            a.close()
