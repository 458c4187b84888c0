"""GPU parity for shockDet + the hybrid Riemann solver (NEXT N2: Alg. 7
P:1815; reading R21) through the C ABI, against the oracle pinned in
tests/test_oracle_shockdet.py, at the R15 tolerance.

Cases cover every KB1 code path the sensor enters: the face-centric 16x16
path (3-D PLM, the bench kernel: own x/y faces, warp 0's block-boundary faces,
the carried z flag), the paired-solve path (3-D WENO5/MC 16^3), generic
shapes, 1-D/2-D, all boundary types, rank-boundary slabs (virtual ranks) and
the telescoping kernel.  Each case also checks, with the oracle, that the
inputs flag shock faces (the hybrid result differs from pure HLLC).
"""
import numpy as np
import pytest

import oracle
import spark_inputs as si

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
HY, THR = si.RIEMANN_HYBRID, 0.5


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


def P(name, ndim, nb, nblk, ng, recon, rk, cfl, bc):
    return si.Problem(name, ndim, nb, nblk, ng, recon, HY, rk, cfl, bc=bc, shock_thresh=THR)


CASES = [
    P("1d_plm", 1, (8, 1, 1), (5, 1, 1), 2, 1, 2, 0.8, ((2, 1), (1, 1), (1, 1))),
    P("1d_weno", 1, (7, 1, 1), (3, 1, 1), 3, 2, 3, 0.8, ((0, 0), (1, 1), (1, 1))),
    P("2d_plm16", 2, (16, 16, 1), (3, 2, 1), 2, 1, 2, 0.4, ((1, 2), (0, 0), (1, 1))),
    P("2d_mc_odd", 2, (12, 10, 1), (3, 3, 1), 2, 3, 2, 0.4, ((2, 2), (0, 0), (1, 1))),
    P("2d_weno16", 2, (16, 16, 1), (2, 3, 1), 3, 2, 3, 0.4, ((0, 0), (2, 1), (1, 1))),
    P("3d_plm16", 3, (16, 16, 16), (2, 2, 2), 2, 1, 2, 0.3, ((1, 1), (0, 0), (2, 1))),
    P("3d_weno16", 3, (16, 16, 16), (2, 1, 2), 3, 2, 3, 0.3, ((0, 0), (1, 2), (1, 1))),
    P("3d_mc16", 3, (16, 16, 16), (1, 2, 2), 2, 3, 2, 0.3, ((2, 2), (1, 1), (0, 0))),
    P("3d_wz_odd", 3, (6, 5, 7), (3, 2, 2), 3, 4, 3, 0.3, ((2, 1), (0, 0), (0, 0))),
]


def shocked(p, U, Un, dt):
    """The oracle flags shock faces in these inputs: hybrid != HLLC."""
    a = oracle.stage(p.config(), U, Un, 0.0, 1.0, dt)
    b = oracle.stage(p.with_(riemann=1).config(), U, Un, 0.0, 1.0, dt)
    return not np.array_equal(a, b)


def blocky(p):
    # the blocky jumps (rho x10, p x100) defeat HLL under WENO5/RK3 at the CFL
    # dt (the oracle itself reports rho or p <= 0): plain random data there
    # (rho, p ~ U[0.5, 1.5], u ~ U[-0.5, 0.5] per cell still flag many faces)
    return p.recon not in (2, 4)


@pytest.mark.parametrize("p", CASES, ids=lambda p: p.name)
def test_single_stage(sp, p):
    Up = cons(p, si.random_state(p, 40, blocky=blocky(p)))
    Un = cons(p, si.random_state(p, 41, blocky=blocky(p)))
    dt = 0.2 * p.cfl * oracle.dt_raw(p.config(), Up)
    assert shocked(p, Up, Un, dt)
    s = sp.Spark(p.config())
    s.set_state(Up)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    for a, b in [(0.0, 1.0), (0.75, 0.25)]:
        g = s.stage_apply(dev(Up), dev(Un), a, b, dt).cpu().numpy()
        assert_parity(g, oracle.stage(p.config(), Up, Un, a, b, dt), what=f"{p.name} a={a}")


@pytest.mark.parametrize("p", CASES, ids=lambda p: p.name)
def test_steps_cfl(sp, p):
    U0 = cons(p, si.random_state(p, 42, blocky=blocky(p)))
    s = sp.Spark(p.config())
    s.set_state(U0)
    Uo = U0
    for _ in range(3):
        dg = s.step(sync=True)
        Uo, do = oracle.step(p.config(), Uo)
        assert abs(dg - do) <= 1e-13 * do
    assert_parity(s.get_state().cpu().numpy(), Uo, what=p.name)


@pytest.mark.parametrize("name", ["c4_sedov3d_plm", "c4_sedov3d_weno"])
def test_sedov3d_hybrid(sp, name):
    """3-D Sedov at the bench block shape (16^3 blocks, 2x2x2 of them), 4 steps."""
    p = si.PRESETS[name].with_(nblk=(2, 2, 2), riemann=HY, shock_thresh=THR)
    U0 = cons(p, si.initial_primitive(p))
    s = sp.Spark(p.config())
    s.set_state(U0)
    Uo = U0
    for _ in range(4):
        s.step()
        Uo, _ = oracle.step(p.config(), Uo)
    assert_parity(s.get_state().cpu().numpy(), Uo, what=name)
    assert shocked(p, Uo, Uo, 0.2 * p.cfl * oracle.dt_raw(p.config(), Uo))


def test_sod_full_run(sp):
    p = si.PRESETS["c1_sod1d"].with_(riemann=HY, shock_thresh=THR)
    U0 = cons(p, si.initial_primitive(p))
    Uo, to, no = oracle.run(p.config(), U0, t_end=p.t_end)
    s = sp.Spark(p.config())
    s.set_state(U0)
    s.advance(10_000, t_end=p.t_end, check_every=32)
    t, n, _ = s.time()
    assert n == no and abs(t - to) <= 1e-14
    assert_parity(s.get_state().cpu().numpy(), Uo, absf=1e-14, what="sod hybrid")


@pytest.mark.parametrize("nranks", [2, 4, 8])
def test_virtual_ranks_bitwise(sp, nranks):
    p = P("v3", 3, (8, 8, 8), (2, 2, 2), 2, 1, 2, 0.3, ((0, 0), (1, 2), (1, 1)))
    cfg = p.config()
    U0 = cons(p, si.random_state(p, 43, blocky=True))
    one = sp.Spark(cfg)
    one.set_state(U0)
    grp = sp.LocalGroup(cfg, nranks)
    G0 = si.to_global(p, U0)
    for r, s in enumerate(grp.ranks):
        lo, n = sp.rank_box(cfg, r, nranks)
        sub = G0[:, lo[2] * 8:(lo[2] + n[2]) * 8, lo[1] * 8:(lo[1] + n[1]) * 8, lo[0] * 8:(lo[0] + n[0]) * 8]
        s.set_state(si.from_global(p.with_(nblk=tuple(n)), np.ascontiguousarray(sub)))
    for _ in range(3):
        assert one.step(sync=True) == grp.step(sync=True)
    G1 = si.to_global(p, one.get_state().cpu().numpy())
    for r, s in enumerate(grp.ranks):
        lo, n = sp.rank_box(cfg, r, nranks)
        Gr = si.to_global(p.with_(nblk=tuple(n)), s.get_state().cpu().numpy())
        assert np.array_equal(Gr, G1[:, lo[2] * 8:(lo[2] + n[2]) * 8, lo[1] * 8:(lo[1] + n[1]) * 8,
                                     lo[0] * 8:(lo[0] + n[0]) * 8])
    grp.close()


@pytest.mark.parametrize("p", [
    P("t1", 1, (16, 1, 1), (4, 1, 1), 2, 1, 2, 0.8, ((1, 1), (1, 1), (1, 1))),
    P("t2", 2, (16, 16, 1), (2, 2, 1), 3, 2, 3, 0.4, ((0, 0), (2, 1), (1, 1))),
], ids=lambda p: p.name)
def test_telescoping(sp, p):
    U0 = cons(p, si.random_state(p, 44, blocky=True))
    s = sp.Spark(p.config())
    s.set_state(U0)
    Uo = U0
    for _ in range(3):
        dg = s.step_telescoping(sync=True)
        Uo, do = oracle.step_telescoping(p.config(), Uo)
        assert abs(dg - do) <= 1e-13 * do
    assert_parity(s.get_state().cpu().numpy(), Uo, what=p.name)


def test_config_rejects_bad_hybrid(sp):
    p = si.PRESETS["c1_sod1d"]
    assert not sp.check_config(p.with_(riemann=HY).config(), 1)                          # threshold 0
    assert not sp.check_config(p.with_(riemann=HY, recon=0, ng=1, shock_thresh=THR).config(), 1)
    assert sp.check_config(p.with_(riemann=HY, shock_thresh=THR).config(), 1)
