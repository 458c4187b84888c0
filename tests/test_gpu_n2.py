"""GPU parity for the NEXT-N2 additions (PLM-MC, WENO5-Z, grvAccel) through
the C ABI, against the oracle pinned in tests/test_oracle_n2.py; R15
tolerance.  Cases cover generic and 16x16 compile-time shapes, 1-3-D, every
boundary type, HLL/HLLC, stage-wise and telescoping steps."""
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


def assert_parity(g, o, rel=1e-12, absf=1e-15, what=""):
    g, o = np.asarray(g), np.asarray(o)
    assert g.shape == o.shape
    for v in range(o.shape[0]):
        scale = np.max(np.abs(o[v]))
        err = np.abs(g[v] - o[v])
        bad = err > rel * np.abs(o[v]) + absf * scale
        assert not bad.any(), f"{what} var {v}: {bad.sum()} cells, max err {err.max():.3e}"


G2 = (0.4, -1.3, 0.0)
G3 = (0.3, -0.8, 1.1)
CASES = [
    si.Problem("1d_mc_hllc", 1, (8, 1, 1), (5, 1, 1), 2, 3, 1, 2, 0.8, bc=((2, 1), (1, 1), (1, 1))),
    si.Problem("1d_wz_hll_grav", 1, (7, 1, 1), (3, 1, 1), 3, 4, 0, 3, 0.8, bc=((0, 0), (1, 1), (1, 1)),
               grav=(-0.7, 0.0, 0.0)),
    si.Problem("2d_mc_hllc_grav", 2, (16, 16, 1), (3, 2, 1), 2, 3, 1, 2, 0.4, bc=((1, 2), (0, 0), (1, 1)),
               grav=G2),
    si.Problem("2d_wz_hllc", 2, (12, 10, 1), (3, 3, 1), 3, 4, 1, 3, 0.4, bc=((2, 2), (0, 0), (1, 1))),
    si.Problem("2d_wz16_hll_grav", 2, (16, 16, 1), (2, 3, 1), 3, 4, 0, 3, 0.4, bc=((0, 0), (2, 1), (1, 1)),
               grav=G2),
    si.Problem("3d_mc16_hllc_grav", 3, (16, 16, 16), (2, 2, 2), 2, 3, 1, 2, 0.3, bc=((1, 1), (0, 0), (2, 1)),
               grav=G3),
    si.Problem("3d_wz16_hllc", 3, (16, 16, 16), (2, 1, 2), 3, 4, 1, 3, 0.3, bc=((0, 0), (1, 2), (1, 1))),
    si.Problem("3d_wz_hll_odd_grav", 3, (6, 5, 7), (3, 2, 2), 3, 4, 0, 3, 0.3, bc=((2, 1), (0, 0), (0, 0)),
               grav=G3),
    si.Problem("3d_plm16_hllc_grav", 3, (16, 16, 16), (2, 2, 1), 2, 1, 1, 2, 0.3, bc=((2, 2), (1, 1), (0, 0)),
               grav=G3),
]


@pytest.mark.parametrize("p", CASES, ids=lambda p: p.name)
def test_single_stage(sp, p):
    Up = cons(p, si.random_state(p, 30, blocky=True))
    Un = cons(p, si.random_state(p, 31, blocky=True))
    dt = 0.2 * p.cfl * oracle.dt_raw(p.config(), Up)
    s = sp.Spark(p.config())
    s.set_state(Up)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    for a, b in [(0.0, 1.0), (0.75, 0.25)]:
        g = s.stage_apply(dev(Up), dev(Un), a, b, dt).cpu().numpy()
        assert_parity(g, oracle.stage(p.config(), Up, Un, a, b, dt), what=f"{p.name} a={a}")


@pytest.mark.parametrize("p", CASES, ids=lambda p: p.name)
def test_steps_cfl(sp, p):
    U0 = cons(p, si.random_state(p, 32, blocky=True))
    s = sp.Spark(p.config())
    s.set_state(U0)
    Uo = U0
    for _ in range(3):
        dg = s.step(sync=True)
        Uo, do = oracle.step(p.config(), Uo)
        assert abs(dg - do) <= 1e-13 * do
    assert_parity(s.get_state().cpu().numpy(), Uo, what=p.name)


@pytest.mark.parametrize("ndim,rk", [(1, 2), (2, 3), (3, 2)])
def test_free_fall_gpu(sp, ndim, rk):
    """Uniform periodic state in uniform gravity on the GPU: exact quadratic
    free fall (the oracle pins the same closed form)."""
    nb = (16, 16 if ndim > 1 else 1, 16 if ndim > 2 else 1)
    nblk = (2, 2 if ndim > 1 else 1, 2 if ndim > 2 else 1)
    g = G3[:ndim] + (0.0,) * (3 - ndim)
    p = si.Problem("ff", ndim, nb, nblk, 2, 1, 1, rk, 0.3, bc=((0, 0),) * 3, grav=g)
    U0 = cons(p, si.uniform_state(p, 12))
    s = sp.Spark(p.config())
    s.set_state(U0)
    dt, t = 1e-2, 0.0
    for _ in range(6):
        s.step(dt=dt)
        t += dt
    U = s.get_state().cpu().numpy()
    rho = U0[0].flat[0]
    m0 = [U0[1 + d].flat[0] for d in range(ndim)]
    assert np.all(U[0] == rho)
    for d in range(ndim):
        assert np.allclose(U[1 + d], m0[d] + rho * g[d] * t, rtol=1e-13, atol=1e-15)
    E = U0[ndim + 1].flat[0] + sum(m0[d] * g[d] for d in range(ndim)) * t + 0.5 * rho * sum(x * x for x in g) * t * t
    assert np.allclose(U[ndim + 1], E, rtol=1e-13)
    for v in range(p.nvar):  # still uniform, bit for bit
        assert np.all(U[v] == U[v].flat[0])


TELE = [
    si.Problem("t1_mc_grav", 1, (8, 1, 1), (6, 1, 1), 2, 3, 1, 2, 0.8, bc=((1, 2), (1, 1), (1, 1)),
               grav=(0.9, 0.0, 0.0)),
    si.Problem("t2_wz", 2, (16, 16, 1), (2, 3, 1), 3, 4, 1, 3, 0.4, bc=((2, 1), (1, 2), (1, 1))),
    si.Problem("t2_mc_grav", 2, (16, 16, 1), (3, 2, 1), 2, 3, 0, 2, 0.4, bc=((0, 0), (2, 2), (1, 1)), grav=G2),
]


@pytest.mark.parametrize("p", TELE, ids=lambda p: p.name)
def test_telescoping(sp, p):
    U0 = cons(p, si.random_state(p, 33, blocky=True))
    s = sp.Spark(p.config())
    s.set_state(U0)
    Uo = U0
    for _ in range(3):
        dg = s.step_telescoping(sync=True)
        Uo, do = oracle.step_telescoping(p.config(), Uo)
        assert abs(dg - do) <= 1e-13 * do
    assert_parity(s.get_state().cpu().numpy(), Uo, what=p.name)


@pytest.mark.parametrize("recon", [3, 4])
def test_sedov3d_production_shape(sp, recon):
    """3-D Sedov on 4^3 blocks of 16^3 (the bench kernel shape) with MC / WENO-Z,
    three steps vs the oracle."""
    base = si.PRESETS["c4_sedov3d_weno" if recon == 4 else "c4_sedov3d_plm"]
    p = base.with_(nblk=(4, 4, 4), recon=recon)
    U0 = cons(p, si.initial_primitive(p))
    s = sp.Spark(p.config())
    s.set_state(U0)
    Uo = U0
    for _ in range(3):
        s.step()
        Uo, _ = oracle.step(p.config(), Uo)
    assert_parity(s.get_state().cpu().numpy(), Uo, what=f"sedov recon {recon}")


def test_rank_count_invariance_with_gravity(sp):
    p = si.Problem("vg", 3, (16, 16, 16), (2, 2, 2), 3, 4, 1, 3, 0.3, bc=((2, 2), (0, 0), (1, 1)), grav=G3)
    U0 = cons(p, si.random_state(p, 34, blocky=True))
    one = sp.Spark(p.config())
    one.set_state(U0)
    grp = sp.LocalGroup(p.config(), 4)
    G0 = si.to_global(p, U0)
    boxes = [sp.rank_box(p.config(), r, 4) for r in range(4)]
    for s, (lo, n) in zip(grp.ranks, boxes):
        sl = tuple(slice(lo[d] * 16, (lo[d] + n[d]) * 16) for d in (2, 1, 0))
        s.set_state(si.from_global(p.with_(nblk=tuple(n)), np.ascontiguousarray(G0[(slice(None),) + sl])))
    for _ in range(2):
        assert one.step(sync=True) == grp.step(sync=True)
    G1 = si.to_global(p, one.get_state().cpu().numpy())
    for s, (lo, n) in zip(grp.ranks, boxes):
        sl = tuple(slice(lo[d] * 16, (lo[d] + n[d]) * 16) for d in (2, 1, 0))
        assert np.array_equal(si.to_global(p.with_(nblk=tuple(n)), s.get_state().cpu().numpy()),
                              G1[(slice(None),) + sl])
    grp.close()
