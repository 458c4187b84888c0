"""GPU invariants at production block shapes (16^3 / 16^2 compile-time kernels):
properties the mathematics fixes, checked on the CUDA path directly (the oracle
pins the same properties on the CPU, tests/test_oracle_pins.py)."""
import numpy as np
import pytest

import oracle
import spark_inputs as si

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def sp():
    from paper_2401_03378_b200 import spark

    spark.lib()
    return spark


def cons(p, W):
    return oracle.prim_to_cons(p.ndim, p.gamma, W)


def run(sp, p, U0, steps, dt=0.0):
    s = sp.Spark(p.config())
    s.set_state(np.ascontiguousarray(U0))
    for _ in range(steps):
        s.step(dt=dt)
    out = s.get_state().cpu().numpy()
    s.close()
    return out


@pytest.mark.parametrize("recon,rk", [(1, 2), (2, 3)])
def test_3d_sod_along_each_axis_equals_1d(sp, recon, rk):
    """A Sod tube along x, y or z of a 3-D box with 16^3 blocks (periodic across)
    gives the 1-D solution on every line (transverse fluxes cancel exactly)."""
    ng = 3 if recon == 2 else 2
    line = si.Problem("l", 1, (16, 1, 1), (4, 1, 1), ng, recon, 1, rk, 0.3)
    U1 = run(sp, line, cons(line, si.sod_x(line)), 4, dt=2e-3)
    G1 = si.to_global(line, U1)[:, 0, 0, :]
    for axis in range(3):
        nblk = [1, 1, 1]
        nblk[axis] = 4
        bc = [(0, 0), (0, 0), (0, 0)]
        bc[axis] = (1, 1)
        p = si.Problem("s", 3, (16, 16, 16), tuple(nblk), ng, recon, 1, rk, 0.3, bc=tuple(bc))
        x, y, z = si.centres(p)
        c = (x, y, z)[axis]
        rho = np.where(c < 0.5, 1.0, 0.125)
        pres = np.where(c < 0.5, 1.0, 0.1)
        W = np.zeros((5,) + rho.shape)
        W[0], W[4] = rho, pres
        G = si.to_global(p, run(sp, p, cons(p, si.from_global(p, W)), 4, dt=2e-3))
        prof = np.moveaxis(G, 3 - axis, -1).reshape(5, -1, 64)
        for r in range(prof.shape[1]):
            assert np.allclose(prof[0, r], G1[0], rtol=1e-12, atol=1e-15)
            assert np.allclose(prof[1 + axis, r], G1[1], rtol=1e-12, atol=1e-14)
            assert np.allclose(prof[4, r], G1[2], rtol=1e-12, atol=1e-15)


def test_3d_conservation_periodic(sp):
    p = si.Problem("c", 3, (16, 16, 16), (2, 2, 2), 3, 2, 1, 3, 0.3, bc=((0, 0),) * 3)
    U0 = cons(p, si.random_state(p, 4, blocky=True))
    U = run(sp, p, U0, 6)
    for v in range(5):
        scale = np.abs(U0[v]).sum() + np.abs(U[v]).sum()
        assert abs(U[v].sum() - U0[v].sum()) <= 1e-13 * scale


def test_3d_sedov_symmetry_gpu(sp):
    """256^3-block-shape Sedov (4^3 blocks of 16^3): the x<->y transposition and
    the mirror x -> 1-x hold to round-off on the GPU."""
    p = si.PRESETS["c4_sedov3d_weno"].with_(nblk=(4, 4, 4))
    G = si.to_global(p, run(sp, p, cons(p, si.initial_primitive(p)), 5))
    T = np.swapaxes(G, -1, -2).copy()
    T[[1, 2]] = T[[2, 1]]
    M = G[..., ::-1].copy()
    M[1] = -M[1]
    scale = np.abs(G).max(axis=(1, 2, 3), keepdims=True)
    assert np.all(np.abs(T - G) <= 1e-12 * scale)
    assert np.all(np.abs(M - G) <= 1e-10 * scale)


def test_rank_count_invariance_3d_production_shape(sp):
    """4 virtual ranks of 16^3 blocks == 1 rank, bit for bit, over 3 steps."""
    p = si.Problem("v", 3, (16, 16, 16), (2, 2, 2), 2, 1, 1, 2, 0.3, bc=((1, 1), (0, 0), (2, 1)))
    U0 = cons(p, si.random_state(p, 9, blocky=True))
    one = sp.Spark(p.config())
    one.set_state(U0)
    grp = sp.LocalGroup(p.config(), 4)
    G0 = si.to_global(p, U0)
    boxes = [sp.rank_box(p.config(), r, 4) for r in range(4)]
    for s, (lo, n) in zip(grp.ranks, boxes):
        sl = tuple(slice(lo[d] * 16, (lo[d] + n[d]) * 16) for d in (2, 1, 0))
        s.set_state(si.from_global(p.with_(nblk=tuple(n)), np.ascontiguousarray(G0[(slice(None),) + sl])))
    for _ in range(3):
        assert one.step(sync=True) == grp.step(sync=True)
    G1 = si.to_global(p, one.get_state().cpu().numpy())
    for s, (lo, n) in zip(grp.ranks, boxes):
        sl = tuple(slice(lo[d] * 16, (lo[d] + n[d]) * 16) for d in (2, 1, 0))
        Gr = si.to_global(p.with_(nblk=tuple(n)), s.get_state().cpu().numpy())
        assert np.array_equal(Gr, G1[(slice(None),) + sl])
    grp.close()
