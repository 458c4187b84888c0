"""GPU telescoping SSP-RK (NEXT N1, spark_step_telescoping) against the oracle's
telescoping step (tests/test_oracle_telescoping.py pins that oracle), at the
R15 tolerance; and, with periodic boundaries, against the GPU non-telescoping
step (mathematically identical)."""
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
    for v in range(o.shape[0]):
        scale = np.max(np.abs(o[v]))
        err = np.abs(g[v] - o[v])
        bad = err > rel * np.abs(o[v]) + absf * scale
        assert not bad.any(), f"{what} var {v}: {bad.sum()} cells, max err {err.max():.3e}"


CASES = [
    si.Problem("t1p", 1, (8, 1, 1), (6, 1, 1), 2, 1, 1, 2, 0.8, bc=((1, 2), (1, 1), (1, 1))),
    si.Problem("t1w", 1, (7, 1, 1), (5, 1, 1), 3, 2, 0, 3, 0.8, bc=((0, 0), (1, 1), (1, 1))),
    si.Problem("t2p", 2, (16, 16, 1), (3, 2, 1), 2, 1, 1, 2, 0.4, bc=((1, 1), (0, 0), (1, 1))),
    si.Problem("t2w", 2, (16, 16, 1), (2, 3, 1), 3, 2, 1, 3, 0.4, bc=((2, 1), (1, 2), (1, 1))),
    si.Problem("t2f", 2, (12, 10, 1), (3, 2, 1), 1, 0, 0, 2, 0.4, bc=((0, 0), (2, 2), (1, 1))),
]


@pytest.mark.parametrize("p", CASES, ids=lambda p: p.name)
def test_telescoping_vs_oracle(sp, p):
    U0 = cons(p, si.random_state(p, 21, blocky=True))
    s = sp.Spark(p.config())
    s.set_state(U0)
    Uo = U0
    for _ in range(3):
        dg = s.step_telescoping(sync=True)
        Uo, do = oracle.step_telescoping(p.config(), Uo)
        assert abs(dg - do) <= 1e-13 * do
    assert_parity(s.get_state().cpu().numpy(), Uo, what=p.name)


@pytest.mark.parametrize("p", [c.with_(bc=((0, 0),) * 3) for c in CASES], ids=lambda p: p.name + "_per")
def test_periodic_telescoping_equals_stagewise_gpu(sp, p):
    U0 = cons(p, si.random_state(p, 22, blocky=True))
    a, b = sp.Spark(p.config()), sp.Spark(p.config())
    a.set_state(U0)
    b.set_state(U0)
    for _ in range(3):
        a.step()
        b.step_telescoping()
    ga, gb = a.get_state().cpu().numpy(), b.get_state().cpu().numpy()
    assert_parity(gb, ga, rel=1e-13, absf=1e-16, what="periodic")


def test_c3_telescoping_reduced(sp):
    """configs[2]'s scheme (2-D Sedov, WENO5 + HLLC, SSP-RK3, 16^2 blocks) on a
    256^2 grid: 3 telescoped steps vs the oracle."""
    p = si.PRESETS["c3_sedov2d"].with_(nblk=(16, 16, 1))
    U0 = cons(p, si.initial_primitive(p))
    s = sp.Spark(p.config())
    s.set_state(U0)
    Uo = U0
    for _ in range(3):
        s.step_telescoping()
        Uo, _ = oracle.step_telescoping(p.config(), Uo)
    assert_parity(s.get_state().cpu().numpy(), Uo, what="c3 telescoping")


def test_telescoping_3d_needs_a_scratch(sp):
    """3-D telescoping runs through HBM tiles (tests/test_gpu_telescoping3d.py);
    at the ABI, without spark_set_scratch the call is refused (SPARK_ERR_STATE)."""
    p = si.PRESETS["c4_sedov3d_plm"].with_(nblk=(2, 2, 2))
    s = sp.Spark(p.config())
    s.set_primitive(si.initial_primitive(p))
    assert sp.lib().spark_step_telescoping(s.ctx, 0.0, 0.0, None) == sp.SPARK_ERR_STATE
