"""CPU oracle for the Spark block-update hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product path
(``paper_2401_03378_b200``) never imports it and shares no code with it.

The arithmetic lives in ``spark_oracle.c`` (plain FP64 C, ``-ffp-contract=off``),
which cites the PAPER.md passages it follows.  This module only compiles it
with gcc and marshals numpy arrays through ctypes.

Parity status per function (DESIGN.md §3 lists the pins):
  fill_guardcells  pinned: brute-force per-dimension map, index-encoded state
  prim/cons EOS    pinned: closed-form round trip, hand-computed values
  plm_face         pinned: linear exactness, extrema -> zero slope
  weno5_edge       pinned: quadratic exactness, observed order on smooth data,
                   the Jiang-Shu beta_k / omega_k written out from their
                   definition on fixed and random stencils, ENO at a jump
                   (JS and Z); MC: closed forms, linear exactness, order
  riemann          pinned: consistency F(W,W) = physical flux, supersonic
                   upwinding, stationary contact, mirror antisymmetry; HLLC
                   star flux = physical flux of the star state (Toro 10.39)
  shock_face       pinned: sensor cases (compression / expansion / dead band),
                   Sod flags only the shock, HLLC bitwise where nothing is flagged
  stage/step/run   pinned: exact Sod (Toro 2009, Table 4.3 Test 1),
                   conservation, uniform state, x<->y symmetry, 2-D row == 1-D,
                   advected density wave convergence order
  step_telescoping pinned: periodic = non-telescoping bitwise, differences
                   confined to (S-1)*NGK boundary cells, exact Sod
  amr_*            pinned: brute-force composite guard fill, uniform state,
                   conservation to round-off (and the correction matters),
                   empty / full refined box = the uniform scheme, transposition
                   symmetry, Sod through a refined half
  tools/oracle_mutations.py: every listed mutation of this C file fails a pin
  (profiles/r02_oracle_mutations.txt).
  Faithfulness to Flash-X Spark's own constants (limiter, eps, wave speeds):
  parity unpinned — PAPER.md prints none.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "spark_oracle.c")
_LIB = os.path.join(_HERE, "libspark_oracle.so")
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-std=c11", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no-op when the .so is newer than the source)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Cfg(ctypes.Structure):
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


class _Amr(ctypes.Structure):
    _fields_ = [("c", _Cfg), ("rlo", ctypes.c_int32 * 3), ("rhi", ctypes.c_int32 * 3)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        # SPARK_ORACLE_LIB: a mutated copy of the oracle (tools/oracle_mutations.py)
        _lib = ctypes.CDLL(os.environ.get("SPARK_ORACLE_LIB") or build())
        P = ctypes.POINTER
        d, i32, i64 = ctypes.c_double, ctypes.c_int, ctypes.c_long
        dp = P(ctypes.c_double)
        sig = {
            "oracle_check_config": (i32, [P(_Cfg)]),
            "oracle_fill_guardcells": (i32, [P(_Cfg), dp, dp]),
            "oracle_prim_to_cons": (None, [i32, d, i64, dp, dp]),
            "oracle_cons_to_prim": (None, [i32, d, i64, dp, dp]),
            "oracle_plm_face": (None, [d, d, d, d, dp, dp]),
            "oracle_weno5_edge": (d, [d, d, d, d, d]),
            "oracle_weno5_face": (None, [dp, dp, dp]),
            "oracle_mc_face": (None, [d, d, d, d, dp, dp]),
            "oracle_weno5z_edge": (d, [d, d, d, d, d]),
            "oracle_weno5z_face": (None, [dp, dp, dp]),
            "oracle_riemann": (None, [i32, i32, d, dp, dp, dp]),
            "oracle_shock_face": (i32, [dp, dp, dp, d, d]),
            "oracle_dt_raw": (d, [P(_Cfg), dp]),
            "oracle_dt": (d, [P(_Cfg), dp, d, d]),
            "oracle_stage_padded": (i32, [P(_Cfg), dp, dp, d, d, d, dp]),
            "oracle_stage": (i32, [P(_Cfg), dp, dp, d, d, d, dp]),
            "oracle_rk_coeffs": (None, [i32, i32, dp, dp]),
            "oracle_step": (i32, [P(_Cfg), dp, d, d, d, dp]),
            "oracle_step_telescoping": (i32, [P(_Cfg), dp, d, d, d, dp]),
            "oracle_run": (i32, [P(_Cfg), dp, d, i64, dp, P(ctypes.c_long)]),
            "oracle_num_threads": (i32, []),
            "oracle_set_threads": (None, [i32]),
            "oracle_amr_check": (i32, [P(_Amr)]),
            "oracle_amr_leaves": (i32, [P(_Amr), P(ctypes.c_long), P(ctypes.c_long)]),
            "oracle_amr_fill": (i32, [P(_Amr), dp, dp]),
            "oracle_amr_dt": (d, [P(_Amr), dp, d, d]),
            "oracle_amr_step": (i32, [P(_Amr), dp, d, d, d, i32, dp]),
            "oracle_amr_run": (i32, [P(_Amr), dp, d, i64, dp, P(ctypes.c_long)]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(_lib, name)
            fn.restype = res
            fn.argtypes = args
    return _lib


@dataclass
class Config:
    """Problem description (same fields as spark_config in include/spark.h)."""

    ndim: int
    nb: tuple
    nblk: tuple
    ng: int
    lo: tuple = (0.0, 0.0, 0.0)
    hi: tuple = (1.0, 1.0, 1.0)
    bc: tuple = ((1, 1), (1, 1), (1, 1))
    recon: int = 1
    riemann: int = 1
    rk_stages: int = 2
    gamma: float = 1.4
    cfl: float = 0.8
    grav: tuple = (0.0, 0.0, 0.0)
    shock_thresh: float = 0.0
    extra: dict = field(default_factory=dict)

    def c(self) -> _Cfg:
        s = _Cfg()
        s.ndim = self.ndim
        for d in range(3):
            s.nb[d] = self.nb[d]
            s.nblk[d] = self.nblk[d]
            s.lo[d] = self.lo[d]
            s.hi[d] = self.hi[d]
            s.bc[d][0] = self.bc[d][0]
            s.bc[d][1] = self.bc[d][1]
        s.ng = self.ng
        s.recon, s.riemann, s.rk_stages = self.recon, self.riemann, self.rk_stages
        s.gamma, s.cfl = self.gamma, self.cfl
        for d in range(3):
            s.grav[d] = self.grav[d]
        s.shock_thresh = self.shock_thresh
        return s

    @property
    def nvar(self) -> int:
        return self.ndim + 2

    @property
    def nblocks(self) -> int:
        return self.nblk[0] * self.nblk[1] * self.nblk[2]

    @property
    def cells_per_block(self) -> int:
        return self.nb[0] * self.nb[1] * self.nb[2]

    @property
    def ncells(self) -> int:
        return self.nblocks * self.cells_per_block

    def padded_shape(self):
        g = [self.ng if d < self.ndim else 0 for d in range(3)]
        return (self.nvar, self.nblocks, self.nb[2] + 2 * g[2], self.nb[1] + 2 * g[1], self.nb[0] + 2 * g[0])


def _as_cfg(cfg):
    if isinstance(cfg, Config):
        return cfg
    return Config(**cfg)


def _dp(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


class OracleError(RuntimeError):
    pass


def _chk(st: int, what: str):
    if st != 0:
        raise OracleError(f"{what}: oracle status {st}")


def check_config(cfg) -> int:
    c = _as_cfg(cfg).c()
    return lib().oracle_check_config(ctypes.byref(c))


def fill_guardcells(cfg, U: np.ndarray) -> np.ndarray:
    cfg = _as_cfg(cfg)
    U = np.ascontiguousarray(U, dtype=np.float64)
    P = np.empty(cfg.padded_shape(), dtype=np.float64)
    c = cfg.c()
    _chk(lib().oracle_fill_guardcells(ctypes.byref(c), _dp(U), _dp(P)), "fill_guardcells")
    return P


def prim_to_cons(ndim: int, gamma: float, W: np.ndarray) -> np.ndarray:
    W = np.ascontiguousarray(W, dtype=np.float64)
    U = np.empty_like(W)
    n = W.size // (ndim + 2)
    lib().oracle_prim_to_cons(ndim, gamma, n, _dp(W), _dp(U))
    return U


def cons_to_prim(ndim: int, gamma: float, U: np.ndarray) -> np.ndarray:
    U = np.ascontiguousarray(U, dtype=np.float64)
    W = np.empty_like(U)
    n = U.size // (ndim + 2)
    lib().oracle_cons_to_prim(ndim, gamma, n, _dp(U), _dp(W))
    return W


def plm_face(wm1, w0, w1, w2):
    l, r = ctypes.c_double(), ctypes.c_double()
    lib().oracle_plm_face(wm1, w0, w1, w2, ctypes.byref(l), ctypes.byref(r))
    return l.value, r.value


def weno5_edge(a, b, c, d, e) -> float:
    return lib().oracle_weno5_edge(a, b, c, d, e)


def mc_face(wm1, w0, w1, w2):
    l, r = ctypes.c_double(), ctypes.c_double()
    lib().oracle_mc_face(wm1, w0, w1, w2, ctypes.byref(l), ctypes.byref(r))
    return l.value, r.value


def weno5z_edge(a, b, c, d, e) -> float:
    return lib().oracle_weno5z_edge(a, b, c, d, e)


def weno5z_face(s):
    s = np.ascontiguousarray(s, dtype=np.float64)
    l, r = ctypes.c_double(), ctypes.c_double()
    lib().oracle_weno5z_face(_dp(s), ctypes.byref(l), ctypes.byref(r))
    return l.value, r.value


def weno5_face(s):
    s = np.ascontiguousarray(s, dtype=np.float64)
    l, r = ctypes.c_double(), ctypes.c_double()
    lib().oracle_weno5_face(_dp(s), ctypes.byref(l), ctypes.byref(r))
    return l.value, r.value


def shock_face(un, p, thresh: float, rho=(1.0, 1.0, 1.0, 1.0), gamma: float = 1.4) -> bool:
    """shockDet face flag from the normal velocity, pressure and density of the
    cells i-1, i, i+1, i+2 of the face between cells i and i+1."""
    un = np.ascontiguousarray(un, dtype=np.float64)
    p = np.ascontiguousarray(p, dtype=np.float64)
    rho = np.ascontiguousarray(rho, dtype=np.float64)
    return bool(lib().oracle_shock_face(_dp(un), _dp(p), _dp(rho), thresh, gamma))


def riemann(kind: int, gamma: float, wl, wr) -> np.ndarray:
    """Flux in the rotated frame (rho, u_n, u_t..., p); kind 0 HLL, 1 HLLC."""
    wl = np.ascontiguousarray(wl, dtype=np.float64)
    wr = np.ascontiguousarray(wr, dtype=np.float64)
    f = np.empty_like(wl)
    lib().oracle_riemann(kind, wl.size, gamma, _dp(wl), _dp(wr), _dp(f))
    return f


def dt_raw(cfg, U) -> float:
    cfg = _as_cfg(cfg)
    U = np.ascontiguousarray(U, dtype=np.float64)
    c = cfg.c()
    return lib().oracle_dt_raw(ctypes.byref(c), _dp(U))


def dt(cfg, U, t=0.0, t_end=0.0) -> float:
    cfg = _as_cfg(cfg)
    U = np.ascontiguousarray(U, dtype=np.float64)
    c = cfg.c()
    return lib().oracle_dt(ctypes.byref(c), _dp(U), t, t_end)


def rk_coeffs(stages: int, s: int):
    a, b = ctypes.c_double(), ctypes.c_double()
    lib().oracle_rk_coeffs(stages, s, ctypes.byref(a), ctypes.byref(b))
    return a.value, b.value


def stage(cfg, Uprev, Un, a, b, dt_) -> np.ndarray:
    cfg = _as_cfg(cfg)
    Uprev = np.ascontiguousarray(Uprev, dtype=np.float64)
    Un = np.ascontiguousarray(Un, dtype=np.float64)
    out = np.empty_like(Uprev)
    c = cfg.c()
    _chk(lib().oracle_stage(ctypes.byref(c), _dp(Uprev), _dp(Un), a, b, dt_, _dp(out)), "stage")
    return out


def stage_padded(cfg, P, Un, a, b, dt_) -> np.ndarray:
    cfg = _as_cfg(cfg)
    P = np.ascontiguousarray(P, dtype=np.float64)
    Un = np.ascontiguousarray(Un, dtype=np.float64)
    out = np.empty((cfg.nvar, cfg.nblocks) + tuple(reversed(cfg.nb)), dtype=np.float64)
    c = cfg.c()
    _chk(lib().oracle_stage_padded(ctypes.byref(c), _dp(P), _dp(Un), a, b, dt_, _dp(out)), "stage_padded")
    return out


def step(cfg, U, t=0.0, t_end=0.0, dt_fixed=0.0):
    """One SSP-RK step; returns (U_new, dt_used)."""
    cfg = _as_cfg(cfg)
    U = np.array(U, dtype=np.float64, copy=True, order="C")
    d = ctypes.c_double()
    c = cfg.c()
    _chk(lib().oracle_step(ctypes.byref(c), _dp(U), t, t_end, dt_fixed, ctypes.byref(d)), "step")
    return U, d.value


def step_telescoping(cfg, U, t=0.0, t_end=0.0, dt_fixed=0.0):
    """One telescoping SSP-RK step: one thick guard fill, all
    stages per block on the shrinking halo; returns (U_new, dt_used)."""
    cfg = _as_cfg(cfg)
    U = np.array(U, dtype=np.float64, copy=True, order="C")
    d = ctypes.c_double()
    c = cfg.c()
    _chk(lib().oracle_step_telescoping(ctypes.byref(c), _dp(U), t, t_end, dt_fixed, ctypes.byref(d)),
         "step_telescoping")
    return U, d.value


def run(cfg, U, t_end=0.0, max_steps=0, t0=0.0):
    """Advance to t_end and/or max_steps; returns (U, t, nsteps)."""
    cfg = _as_cfg(cfg)
    U = np.array(U, dtype=np.float64, copy=True, order="C")
    t = ctypes.c_double(t0)
    n = ctypes.c_long(0)
    c = cfg.c()
    _chk(lib().oracle_run(ctypes.byref(c), _dp(U), t_end, max_steps, ctypes.byref(t), ctypes.byref(n)), "run")
    return U, t.value, n.value


def num_threads() -> int:
    return lib().oracle_num_threads()


def set_threads(n: int) -> None:
    """OpenMP threads of the oracle (n <= 0: all cores)."""
    lib().oracle_set_threads(int(n))


# ------------------------------------------------ NEXT N3: static two-level AMR
def _amr(cfg, rlo, rhi) -> _Amr:
    a = _Amr()
    a.c = _as_cfg(cfg).c()
    for d in range(3):
        a.rlo[d] = int(rlo[d])
        a.rhi[d] = int(rhi[d])
    return a


def amr_leaves(cfg, rlo, rhi):
    """(coarse leaves, fine leaves) of the refinement of coarse blocks [rlo, rhi)."""
    a = _amr(cfg, rlo, rhi)
    nc, nf = ctypes.c_long(), ctypes.c_long()
    _chk(lib().oracle_amr_leaves(ctypes.byref(a), ctypes.byref(nc), ctypes.byref(nf)), "amr_leaves")
    return nc.value, nf.value


def amr_fill(cfg, rlo, rhi, U) -> np.ndarray:
    cfg = _as_cfg(cfg)
    a = _amr(cfg, rlo, rhi)
    nl = sum(amr_leaves(cfg, rlo, rhi))
    U = np.ascontiguousarray(U, dtype=np.float64)
    g = [cfg.ng if d < cfg.ndim else 0 for d in range(3)]
    P = np.empty((cfg.nvar, nl, cfg.nb[2] + 2 * g[2], cfg.nb[1] + 2 * g[1], cfg.nb[0] + 2 * g[0]))
    _chk(lib().oracle_amr_fill(ctypes.byref(a), _dp(U), _dp(P)), "amr_fill")
    return P


def amr_dt(cfg, rlo, rhi, U, t=0.0, t_end=0.0) -> float:
    a = _amr(cfg, rlo, rhi)
    return lib().oracle_amr_dt(ctypes.byref(a), _dp(np.ascontiguousarray(U, dtype=np.float64)), t, t_end)


def amr_step(cfg, rlo, rhi, U, t=0.0, t_end=0.0, dt_fixed=0.0, correct=True):
    """One composite step (fluxBuff + flux correction); returns (U, dt)."""
    a = _amr(cfg, rlo, rhi)
    U = np.array(U, dtype=np.float64, copy=True, order="C")
    dt = ctypes.c_double()
    _chk(lib().oracle_amr_step(ctypes.byref(a), _dp(U), t, t_end, dt_fixed, int(correct), ctypes.byref(dt)),
         "amr_step")
    return U, dt.value


def amr_run(cfg, rlo, rhi, U, t_end=0.0, max_steps=0):
    a = _amr(cfg, rlo, rhi)
    U = np.array(U, dtype=np.float64, copy=True, order="C")
    t, n = ctypes.c_double(0.0), ctypes.c_long(0)
    _chk(lib().oracle_amr_run(ctypes.byref(a), _dp(U), t_end, max_steps, ctypes.byref(t), ctypes.byref(n)),
         "amr_run")
    return U, t.value, n.value
