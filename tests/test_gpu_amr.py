"""GPU parity for NEXT N3 (fluxBuff + flux correction on a static two-level
refinement, spark_amr_*) through the C ABI against the oracle pinned in
tests/test_oracle_amr.py: the coarse-fine guard fill bit for bit, single and
multi-step composite updates at the R15 tolerance, and the invariants
(uniform state, conservation to round-off) on the GPU itself."""
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
    nv, nl = W.shape[0], W.shape[1]
    return oracle.prim_to_cons(p.ndim, p.gamma, W.reshape(nv, nl, -1)).reshape(W.shape)


def assert_parity(g, o, rel=1e-12, absf=1e-15, what=""):
    g, o = np.asarray(g), np.asarray(o)
    assert g.shape == o.shape
    for v in range(o.shape[0]):
        scale = np.max(np.abs(o[v]))
        err = np.abs(g[v] - o[v])
        bad = err > rel * np.abs(o[v]) + absf * scale
        assert not bad.any(), f"{what} var {v}: {bad.sum()} cells, max err {err.max():.3e}"


def P(name, ndim, nb, nblk, ng, recon, riemann, rk, cfl, bc, thr=0.0):
    return si.Problem(name, ndim, nb, nblk, ng, recon, riemann, rk, cfl, bc=bc, shock_thresh=thr)


CASES = [
    (P("1d_plm", 1, (8, 1, 1), (6, 1, 1), 2, 1, 1, 2, 0.8, ((0, 0), (1, 1), (1, 1))), (2, 0, 0), (4, 1, 1)),
    (P("1d_weno_edge", 1, (8, 1, 1), (5, 1, 1), 3, 2, 1, 3, 0.8, ((2, 1), (1, 1), (1, 1))), (0, 0, 0), (2, 1, 1)),
    (P("2d_plm16", 2, (16, 16, 1), (4, 3, 1), 2, 1, 1, 2, 0.4, ((0, 0), (1, 2), (1, 1))), (1, 1, 0), (3, 2, 1)),
    (P("2d_weno_rk3", 2, (8, 8, 1), (4, 4, 1), 3, 2, 1, 3, 0.4, ((0, 0), (0, 0), (1, 1))), (1, 0, 0), (3, 2, 1)),
    (P("2d_mc_hll", 2, (8, 6, 1), (3, 4, 1), 2, 3, 0, 2, 0.4, ((2, 2), (1, 1), (1, 1))), (0, 1, 0), (2, 3, 1)),
    (P("2d_hybrid", 2, (8, 8, 1), (4, 4, 1), 2, 1, 2, 2, 0.4, ((1, 1), (1, 1), (1, 1)), 0.5), (1, 1, 0), (3, 3, 1)),
    (P("3d_plm", 3, (8, 8, 8), (3, 3, 3), 2, 1, 1, 2, 0.3, ((0, 0), (1, 2), (2, 1))), (1, 1, 1), (2, 2, 2)),
    (P("3d_weno", 3, (6, 6, 6), (2, 3, 2), 3, 2, 1, 3, 0.3, ((0, 0), (0, 0), (0, 0))), (0, 1, 0), (1, 2, 2)),
    # 16^3 leaves: the fused leaf kernel (face-centric schemes), every BC kind
    (P("3d_plm16", 3, (16, 16, 16), (3, 3, 3), 2, 1, 1, 2, 0.3, ((0, 0), (1, 2), (2, 1))), (1, 1, 1), (2, 2, 2)),
    (P("3d_mc16_hll", 3, (16, 16, 16), (2, 3, 2), 2, 3, 0, 3, 0.3, ((2, 2), (0, 0), (1, 1))), (0, 1, 0), (1, 2, 2)),
    (P("3d_first16", 3, (16, 16, 16), (3, 2, 2), 2, 0, 1, 2, 0.3, ((1, 1), (2, 2), (0, 0))), (1, 0, 1), (3, 1, 2)),
    (P("3d_hybrid16", 3, (16, 16, 16), (2, 2, 3), 2, 1, 2, 2, 0.3, ((0, 0), (0, 0), (2, 2)), 0.5), (0, 0, 1),
     (2, 1, 2)),
]


@pytest.mark.parametrize("p,rlo,rhi", CASES, ids=lambda x: getattr(x, "name", str(x)))
def test_fill_bitexact(sp, p, rlo, rhi):
    """The padded leaves (interior + face guards across coarse-fine faces and
    physical boundaries) equal the oracle's bit for bit; index-encoded and
    random states."""
    nl = sum(oracle.amr_leaves(p.config(), rlo, rhi))
    assert (nl,) == (sum(sp.amr_leaves(p.config(), rlo, rhi)),)
    enc = np.stack([v * 2.0 ** 32 + np.arange(nl * int(np.prod(p.nb)), dtype=np.float64).reshape(
        (nl,) + tuple(reversed(p.nb))) for v in range(p.nvar)])
    for U in (enc, cons(p, si.amr_primitive(p, rlo, rhi, "random", seed=1))):
        a = sp.Amr(p.config(), rlo, rhi)
        a.set_state(U)
        g = a.fill_guardcells().cpu().numpy()
        o = oracle.amr_fill(p.config(), rlo, rhi, U)
        face = ~np.isnan(o)
        assert np.array_equal(np.isnan(g), ~face)
        assert np.array_equal(g[face], o[face])
        a.close()


@pytest.mark.parametrize("p,rlo,rhi", CASES, ids=lambda x: getattr(x, "name", str(x)))
def test_steps_vs_oracle(sp, p, rlo, rhi):
    kind = "random" if p.riemann != 0 else "pulse"
    U0 = cons(p, si.amr_primitive(p, rlo, rhi, kind, seed=2))
    a = sp.Amr(p.config(), rlo, rhi)
    a.set_state(U0)
    Uo = U0
    for _ in range(3):
        dg = a.step(sync=True)
        Uo, do = oracle.amr_step(p.config(), rlo, rhi, Uo)
        assert abs(dg - do) <= 1e-13 * do
    assert_parity(a.get_state(), Uo, what=p.name)
    a.close()


def test_uniform_state_and_conservation_on_gpu(sp):
    p = P("inv", 3, (8, 8, 8), (3, 3, 3), 2, 1, 1, 2, 0.3, ((0, 0),) * 3)
    rlo, rhi = (1, 1, 1), (2, 3, 2)
    a = sp.Amr(p.config(), rlo, rhi)
    a.set_state(cons(p, si.amr_primitive(p, rlo, rhi, "uniform", seed=3)))
    for _ in range(3):
        a.step()
    U = a.get_state()
    for v in range(p.nvar):
        assert np.all(U[v] == U[v].flat[0])
    U0 = cons(p, si.amr_primitive(p, rlo, rhi, "pulse"))
    a.set_state(U0)
    for _ in range(6):
        a.step()
    U = a.get_state()
    _, _, _, fac = si.amr_centres(p, rlo, rhi)
    tot = lambda X: np.einsum("vl,l->v", X.reshape(p.nvar, X.shape[1], -1).sum(-1), fac ** 3)
    T0, T1 = tot(U0), tot(U)
    assert np.all(np.abs(T1 - T0) <= 1e-13 * (np.abs(T0) + np.abs(T0).max()))
    a.close()


def test_sod_full_run(sp):
    p = P("sod", 1, (8, 1, 1), (16, 1, 1), 2, 1, 1, 2, 0.8, ((1, 1), (1, 1), (1, 1)))
    rlo, rhi = (8, 0, 0), (16, 1, 1)
    U0 = cons(p, si.amr_primitive(p, rlo, rhi, "sod_x"))
    Uo, to, no = oracle.amr_run(p.config(), rlo, rhi, U0, t_end=0.2)
    a = sp.Amr(p.config(), rlo, rhi)
    a.set_state(U0)
    for _ in range(no):
        a.step(t_end=0.2)
    t, n, _ = a.time()
    assert n == no and abs(t - to) <= 1e-14
    assert_parity(a.get_state(), Uo, absf=1e-14, what="amr sod")
    a.close()


def test_failure_rolls_back(sp):
    p = P("bad", 2, (8, 8, 1), (4, 4, 1), 2, 1, 1, 2, 0.4, ((0, 0), (0, 0), (1, 1)))
    rlo, rhi = (1, 1, 0), (3, 3, 1)
    U0 = cons(p, si.amr_primitive(p, rlo, rhi, "random", seed=4))
    a = sp.Amr(p.config(), rlo, rhi)
    a.set_state(U0)
    with pytest.raises(sp.NonPhysicalError, match="rolled back"):
        a.step(dt=1.0, sync=True)
    assert np.array_equal(a.get_state(), U0)
    assert a.time()[:2] == (0.0, 0)
    a.step(sync=True)
    a.close()


@pytest.mark.parametrize("nranks", [2, 3, 5])
@pytest.mark.parametrize("p,rlo,rhi", [CASES[2], CASES[5], CASES[6], CASES[7], CASES[8], CASES[11]],
                         ids=lambda x: getattr(x, "name", str(x)))
def test_virtual_ranks_bitwise(sp, p, rlo, rhi, nranks):
    """The leaf list split into nranks contiguous ranges: guard values and the
    fine-face fluxBuff values cross ranks through packed exchange buffers
    (fill_guardcells, communicate_fluxes); the result equals one rank's bit
    for bit, with the same global dt."""
    U0 = cons(p, si.amr_primitive(p, rlo, rhi, "random", seed=7))
    one = sp.Amr(p.config(), rlo, rhi)
    one.set_state(U0)
    grp = sp.AmrGroup(p.config(), rlo, rhi, nranks)
    for (first, count), a in zip(grp.leaves, grp.ranks):
        a.set_state(np.ascontiguousarray(U0[:, first:first + count]))
    for _ in range(3):
        assert one.step(sync=True) == grp.step(sync=True)
    ref = one.get_state()
    for (first, count), a in zip(grp.leaves, grp.ranks):
        assert np.array_equal(a.get_state(), ref[:, first:first + count])
    grp.close()
    one.close()
