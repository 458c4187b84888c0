"""CPU tests of the CUDA path's arithmetic (spark_device.cuh compiled for the
host) against the oracle: the per-face Riemann solvers, the cell-centric
reconstruction, the integer-pipe limiter and the Newton reciprocal / sqrt.
These pin the GPU formulations without a GPU (the GPU parity tests then pin
the kernels that call them)."""
import ctypes
import os
import subprocess

import numpy as np
import pytest

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "devmath_shim.cu")
DEV = os.path.join(os.path.dirname(HERE), "paper_2401_03378_b200", "csrc", "spark_device.cuh")


@pytest.fixture(scope="module")
def shim(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("shim") / "devmath.so")
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-x", "cu", "-O2", "-std=c++17", "-Xcompiler", "-fPIC",
                           "-shared", "-o", out, SRC])
    L = ctypes.CDLL(out)
    dp = ctypes.POINTER(ctypes.c_double)
    L.shim_riemann.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double, dp, dp, dp]
    L.shim_recon.argtypes = [ctypes.c_int, dp, dp, dp]
    L.shim_minmod.argtypes = [ctypes.c_double, ctypes.c_double]
    L.shim_minmod.restype = ctypes.c_double
    L.shim_rcp.argtypes = [ctypes.c_double]
    L.shim_rcp.restype = ctypes.c_double
    L.shim_sqrt.argtypes = [ctypes.c_double]
    L.shim_sqrt.restype = ctypes.c_double
    L.shim_cons_to_prim.argtypes = [ctypes.c_int, ctypes.c_double, dp, dp]
    return L


def _p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def test_rcp_sqrt(shim):
    g = np.random.Generator(np.random.PCG64(0))
    for x in np.exp(g.uniform(-40, 40, 2000)):
        assert abs(shim.shim_rcp(x) * x - 1.0) < 4e-16
        assert abs(shim.shim_sqrt(x) / np.sqrt(x) - 1.0) < 4e-16
        assert abs(shim.shim_rcp(-x) * x + 1.0) < 4e-16


def test_minmod_bitwise(shim):
    g = np.random.Generator(np.random.PCG64(1))
    vals = list(g.normal(size=200)) + [0.0, -0.0, 1.0, -1.0, 1e-300, -1e-300]
    def rule(a, b):  # reading R2, as the oracle's comparison form states it
        if a > 0 and b > 0:
            return a if a < b else b
        if a < 0 and b < 0:
            return a if a > b else b
        return 0.0

    for a in vals:
        for b in vals:
            d = shim.shim_minmod(a, b)
            assert d == rule(a, b) and np.signbit(d) == np.signbit(rule(a, b)) or d == 0.0 == rule(a, b)


@pytest.mark.parametrize("recon", [1, 2, 3, 4])
def test_recon_cell_matches_faces(shim, recon):
    """Cell-centric edges == the oracle's per-face states."""
    g = np.random.Generator(np.random.PCG64(2))
    R = 1 if recon in (1, 3) else 2  # stencil radius of the cell-centric form
    for _ in range(500):
        w = g.uniform(0.1, 2.0, 2 * R + 3) * np.where(g.random(2 * R + 3) < 0.3, 10.0, 1.0)
        # cell c = w[R+1]; its hi edge is W_L of face c+1/2, its lo edge is W_R of face c-1/2
        c = R + 1
        s = np.ascontiguousarray(w[c - R:c + R + 1])
        lo, hi = ctypes.c_double(), ctypes.c_double()
        shim.shim_recon(recon, _p(s), ctypes.byref(lo), ctypes.byref(hi))
        if recon in (1, 3):
            face = oracle.plm_face if recon == 1 else oracle.mc_face
            oL, _ = face(w[c - 1], w[c], w[c + 1], w[c + 2])
            _, oR = face(w[c - 2], w[c - 1], w[c], w[c + 1])
            assert hi.value == oL and lo.value == oR  # bitwise (exact arithmetic)
        else:
            edge = oracle.weno5_edge if recon == 2 else oracle.weno5z_edge
            oL = edge(*w[c - 2:c + 3])
            oR = edge(*w[c + 2:c - 3:-1])
            assert abs(hi.value - oL) <= 1e-14 * abs(oL) and abs(lo.value - oR) <= 1e-14 * abs(oR)


def test_minmod3_rule(shim):
    """Integer-pipe three-argument minmod == the comparison form, incl. zeros."""
    L = shim
    L.shim_minmod3.argtypes = [ctypes.c_double] * 3
    L.shim_minmod3.restype = ctypes.c_double

    def rule(a, b, c):
        if a > 0 and b > 0 and c > 0:
            return min(a, b, c)
        if a < 0 and b < 0 and c < 0:
            return max(a, b, c)
        return 0.0

    g = np.random.Generator(np.random.PCG64(3))
    vals = list(g.normal(size=60)) + [0.0, -0.0, 1.0, -1.0, 2.0, 1e-300, -1e-300]
    for _ in range(20000):
        a, b, c = (vals[i] for i in g.integers(0, len(vals), 3))
        assert L.shim_minmod3(a, b, c) == rule(a, b, c)


def _rot(W, d, ndim):
    """unrotated (rho, u_x.., p) -> oracle frame (rho, u_d, others in axis order, p)."""
    order = [0, 1 + d] + [1 + e for e in range(ndim) if e != d] + [ndim + 1]
    return W[order], order


@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("ndim", [1, 2, 3])
def test_riemann_matches_oracle(shim, kind, ndim):
    g = np.random.Generator(np.random.PCG64(3 + kind + 10 * ndim))
    nv = ndim + 2
    for n in range(600):
        wl = np.empty(nv)
        wr = np.empty(nv)
        for w in (wl, wr):
            w[0] = g.uniform(0.05, 5.0)
            w[1:nv - 1] = g.uniform(-3, 3, nv - 2) * (3.0 if n % 5 == 0 else 1.0)
            w[nv - 1] = g.uniform(0.01, 5.0)
        for d in range(ndim):
            f = np.empty(nv)
            shim.shim_riemann(kind, nv, d, 1.4, _p(wl), _p(wr), _p(f))
            rl, order = _rot(wl, d, ndim)
            rr, _ = _rot(wr, d, ndim)
            fo_rot = oracle.riemann(kind, 1.4, rl, rr)
            fo = np.empty(nv)
            fo[order] = fo_rot
            scale = np.max(np.abs(fo)) + 1.0
            assert np.allclose(f, fo, rtol=1e-12, atol=1e-13 * scale), (n, d, f, fo)


def test_cons_to_prim(shim):
    g = np.random.Generator(np.random.PCG64(5))
    for nv in (3, 4, 5):
        W = np.empty((nv, 200))
        W[0] = g.uniform(0.1, 3, 200)
        W[1:nv - 1] = g.uniform(-2, 2, (nv - 2, 200))
        W[nv - 1] = g.uniform(0.1, 3, 200)
        U = oracle.prim_to_cons(nv - 2, 1.4, W)
        for q in range(200):
            u = np.ascontiguousarray(U[:, q])
            w = np.empty(nv)
            assert shim.shim_cons_to_prim(nv, 1.4, _p(u), _p(w)) == 1
            assert np.allclose(w, W[:, q], rtol=1e-13, atol=1e-15)
