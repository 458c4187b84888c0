"""NEXT N1 beyond one rank and two dimensions: telescoping SSP-RK through
HBM tiles (spark_telescope_tile.cu) — 3-D blocks, virtual ranks and NCCL
(self-exchange) with ONE shell exchange per step — against the oracle's
telescoping step (pinned in tests/test_oracle_telescoping.py) at the R15
tolerance, and bitwise invariant under the rank count."""
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
    for v in range(o.shape[0]):
        scale = np.max(np.abs(o[v]))
        err = np.abs(g[v] - o[v])
        bad = err > rel * np.abs(o[v]) + absf * scale
        assert not bad.any(), f"{what} var {v}: {bad.sum()} cells, max err {err.max():.3e}"


CASES = [
    si.Problem("t3_plm16", 3, (16, 16, 16), (2, 2, 2), 2, 1, 1, 2, 0.3, bc=((1, 1), (0, 0), (2, 1))),
    si.Problem("t3_weno16", 3, (16, 16, 16), (1, 2, 1), 3, 2, 1, 3, 0.3, bc=((0, 0), (2, 2), (1, 1))),
    si.Problem("t3_mc_odd", 3, (6, 5, 7), (3, 3, 2), 2, 3, 0, 2, 0.3, bc=((2, 1), (0, 0), (0, 0))),
    si.Problem("t3_hybrid", 3, (8, 8, 8), (2, 2, 2), 2, 1, 2, 2, 0.3, bc=((1, 1), (1, 1), (2, 2)), shock_thresh=0.5),
    si.Problem("t2_tiles", 2, (16, 16, 1), (3, 2, 1), 3, 2, 1, 3, 0.4, bc=((0, 0), (2, 1), (1, 1))),
]


@pytest.mark.parametrize("p", CASES, ids=lambda p: p.name)
def test_tile_telescoping_vs_oracle(sp, p):
    U0 = cons(p, si.random_state(p, 50, blocky=p.recon not in (2, 4)))
    s = sp.Spark(p.config())
    s.set_state(U0)
    s.enable_tiles()
    Uo = U0
    for _ in range(3):
        dg = s.step_telescoping(sync=True)
        Uo, do = oracle.step_telescoping(p.config(), Uo)
        assert abs(dg - do) <= 1e-13 * do
    assert_parity(s.get_state().cpu().numpy(), Uo, what=p.name)
    s.close()


def test_periodic_tile_telescoping_equals_stagewise(sp):
    p = si.Problem("per", 3, (16, 16, 16), (2, 2, 2), 2, 1, 1, 2, 0.3, bc=((0, 0),) * 3)
    U0 = cons(p, si.random_state(p, 51, blocky=True))
    a, b = sp.Spark(p.config()), sp.Spark(p.config())
    a.set_state(U0)
    b.set_state(U0)
    for _ in range(3):
        assert a.step_telescoping(sync=True) == b.step(sync=True)
    assert_parity(a.get_state().cpu().numpy(), b.get_state().cpu().numpy(), what="periodic")


@pytest.mark.parametrize("nranks", [2, 4, 8])
def test_virtual_ranks_bitwise(sp, nranks):
    p = si.Problem("vr", 3, (8, 8, 8), (2, 2, 2), 2, 1, 1, 2, 0.3, bc=((0, 0), (1, 2), (0, 0)))
    cfg = p.config()
    U0 = cons(p, si.random_state(p, 52, blocky=True))
    one = sp.Spark(cfg)
    one.set_state(U0)
    grp = sp.LocalGroup(cfg, nranks)
    G0 = si.to_global(p, U0)
    for r, s in enumerate(grp.ranks):
        lo, n = sp.rank_box(cfg, r, nranks)
        sub = G0[:, lo[2] * 8:(lo[2] + n[2]) * 8, lo[1] * 8:(lo[1] + n[1]) * 8, lo[0] * 8:(lo[0] + n[0]) * 8]
        s.set_state(si.from_global(p.with_(nblk=tuple(n)), np.ascontiguousarray(sub)))
    for _ in range(3):
        assert one.step_telescoping(sync=True) == grp.step_telescoping(sync=True)
    G1 = si.to_global(p, one.get_state().cpu().numpy())
    for r, s in enumerate(grp.ranks):
        lo, n = sp.rank_box(cfg, r, nranks)
        Gr = si.to_global(p.with_(nblk=tuple(n)), s.get_state().cpu().numpy())
        assert np.array_equal(Gr, G1[:, lo[2] * 8:(lo[2] + n[2]) * 8, lo[1] * 8:(lo[1] + n[1]) * 8,
                                     lo[0] * 8:(lo[0] + n[0]) * 8])
    grp.close()


@pytest.mark.parametrize("p", [
    si.Problem("s3", 3, (16, 16, 16), (2, 2, 2), 2, 1, 1, 2, 0.3, bc=((0, 0),) * 3),
    si.Problem("s3m", 3, (8, 8, 8), (2, 3, 2), 3, 2, 1, 3, 0.3, bc=((0, 0), (1, 2), (0, 0))),
], ids=lambda p: p.name)
def test_nccl_self_exchange_bitwise(sp, p):
    """One rank with an NCCL communicator: the periodic shell goes through
    pack -> 26-message grouped ncclSend/ncclRecv to self -> gather; bitwise
    equal to the local-wrap tile path."""
    U0 = cons(p, si.random_state(p, 53, blocky=p.recon != 2))
    plain = sp.Spark(p.config())
    plain.set_state(U0)
    plain.enable_tiles()
    viaccl = sp.Spark(p.config(), nccl_id=sp.nccl_unique_id())
    viaccl.set_state(U0)
    for _ in range(3):
        assert plain.step_telescoping(sync=True) == viaccl.step_telescoping(sync=True)
    assert np.array_equal(plain.get_state().cpu().numpy(), viaccl.get_state().cpu().numpy())
    viaccl.close()
