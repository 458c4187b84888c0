"""Rank-consistent failure handling and bitwise resume (spark.h: spark_step,
spark_step_group, spark_set_time; SURVEY §8(b) errors; P:1542-1546 — every
stage's exchange couples the ranks, so a failure on one rank must stop all).

A stage that produces rho <= 0, p <= 0 or NaN writes the step number into the
failure word, which the per-step collective min-reduces with the CFL minimum;
every rank therefore rolls back (failing step = the checked one) or freezes and
reports (an earlier unchecked step) identically.
"""
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


P2 = si.Problem("e2", 2, (8, 8, 1), (4, 2, 1), 2, 1, 1, 2, 0.4, bc=((0, 0), (0, 0), (1, 1)))


def colliding_state(p: si.Problem, x0: float, x1: float):
    """Physical state whose cells x0 <= x < x1 move apart at Mach ~ 20: a step
    with a dt far beyond the CFL limit empties them (rho < 0 or p < 0)."""
    X = si.centres(p)[0]
    W = np.zeros((p.nvar,) + X.shape)
    W[0] = 1.0
    W[-1] = 1.0
    inside = (X >= x0) & (X < x1)
    W[1] = np.where(inside, np.where(X < 0.5 * (x0 + x1), -25.0, 25.0), 0.0)
    return oracle.prim_to_cons(p.ndim, p.gamma, si.from_global(p, W))


def local(p, G, cfg, sp, r, nranks):
    lo, n = sp.rank_box(cfg, r, nranks)
    sub = G[:, lo[2] * p.nb[2]:(lo[2] + n[2]) * p.nb[2], lo[1] * p.nb[1]:(lo[1] + n[1]) * p.nb[1],
            lo[0] * p.nb[0]:(lo[0] + n[0]) * p.nb[0]]
    return si.from_global(p.with_(nblk=tuple(n)), np.ascontiguousarray(sub))


def test_failing_step_rolls_back(sp):
    U0 = colliding_state(P2, 0.55, 0.7)
    s = sp.Spark(P2.config())
    s.set_state(U0)
    with pytest.raises(sp.NonPhysicalError, match="rolled back"):
        s.step(dt=0.05, sync=True)
    assert np.array_equal(s.get_state().cpu().numpy(), U0)
    t, n, _ = s.time()
    assert t == 0.0 and n == 0
    # a CFL step from the restored state is fine and bitwise the fresh one
    fresh = sp.Spark(P2.config())
    fresh.set_state(U0)
    assert s.step(sync=True) == fresh.step(sync=True)
    assert np.array_equal(s.get_state().cpu().numpy(), fresh.get_state().cpu().numpy())


def test_unchecked_failure_freezes_and_reports(sp):
    U0 = colliding_state(P2, 0.55, 0.7)
    s = sp.Spark(P2.config())
    s.set_state(U0)
    s.step(dt=0.05)             # fails, unchecked
    s.step(dt=1e-4)             # frozen
    with pytest.raises(sp.NonPhysicalError, match="step 1.*not rolled back"):
        s.step(dt=1e-4, sync=True)
    t, n, _ = s.time()
    assert n == 1 and t == 0.05  # time stopped after the failing step


@pytest.mark.parametrize("nranks", [2, 4])
def test_group_failure_rolls_back_every_rank(sp, nranks):
    """The collision lies in the x > 0.5 ranks' sub-boxes only; every rank
    rolls back to its own U^n with identical t and step counts."""
    cfg = P2.config()
    G0 = si.to_global(P2, colliding_state(P2, 0.55, 0.7))
    grp = sp.LocalGroup(cfg, nranks)
    U0 = [local(P2, G0, cfg, sp, r, nranks) for r in range(nranks)]
    for r, s in enumerate(grp.ranks):
        s.set_state(U0[r])
    for _ in range(2):          # two good steps first
        grp.step(dt=1e-5, sync=True)
    Un = [s.get_state().cpu().numpy() for s in grp.ranks]
    with pytest.raises(sp.NonPhysicalError, match="rolled back"):
        grp.step(dt=0.05, sync=True)
    times = set()
    for r, s in enumerate(grp.ranks):
        assert np.array_equal(s.get_state().cpu().numpy(), Un[r])
        times.add(s.time()[:2])
    assert times == {(2e-5, 2)}
    grp.step(dt=1e-5, sync=True)  # and the group steps on
    grp.close()


def test_nccl_self_exchange_failure_rolls_back(sp):
    p = si.Problem("e3", 3, (8, 8, 8), (2, 2, 2), 2, 1, 1, 2, 0.3, bc=((0, 0),) * 3)
    U0 = colliding_state(p, 0.55, 0.7)
    s = sp.Spark(p.config(), nccl_id=sp.nccl_unique_id())
    s.set_state(U0)
    with pytest.raises(sp.NonPhysicalError, match="rolled back"):
        s.step(dt=0.05, sync=True)
    assert np.array_equal(s.get_state().cpu().numpy(), U0)
    assert s.time()[:2] == (0.0, 0)
    s.step(sync=True)
    s.close()


@pytest.mark.parametrize("name", ["c1_sod1d", "c2b_sod2d"])
def test_resume_is_bitwise(sp, name):
    """Checkpoint after k steps (get_state + time), restart in a new context
    (set_state + set_time): the continued run equals the uninterrupted one bit
    for bit, including the t_end clip of the last step."""
    p = si.PRESETS[name]
    U0 = oracle.prim_to_cons(p.ndim, p.gamma, si.initial_primitive(p))
    a = sp.Spark(p.config())
    a.set_state(U0)
    a.advance(10_000, t_end=p.t_end, check_every=16)
    ta, na, _ = a.time()
    b = sp.Spark(p.config())
    b.set_state(U0)
    for _ in range(na // 2):
        b.step(t_end=p.t_end)
    Uk = b.get_state().cpu().numpy()
    tk, nk, _ = b.time()
    c = sp.Spark(p.config())
    c.set_state(Uk)
    c.set_time(tk, nk)
    c.advance(10_000, t_end=p.t_end, check_every=16)
    tc, nc, _ = c.time()
    assert (tc, nc) == (ta, na)
    assert np.array_equal(c.get_state().cpu().numpy(), a.get_state().cpu().numpy())


def test_group_with_a_finalized_member_refuses_to_step(sp):
    """Finalizing one member of a local group leaves the others unable to
    exchange: stepping or filling guards on what is left is a state error,
    not a silent exchange with a missing rank."""
    import ctypes

    cfg = P2.config()
    grp = sp.LocalGroup(cfg, 2)
    G0 = si.to_global(P2, colliding_state(P2, 0.55, 0.7))
    for r, s in enumerate(grp.ranks):
        s.set_state(local(P2, G0, cfg, sp, r, 2))
    h0 = grp._handles[0]
    grp.ranks[1].close()
    st = sp.lib().spark_step_group((ctypes.c_void_p * 1)(h0), 1, 1e-5, 0.0, None)
    assert st == sp.SPARK_ERR_STATE
    assert "finalized" in sp.lib().spark_last_error(ctypes.c_void_p(h0)).decode()
    with pytest.raises(sp.SparkError, match="finalized"):
        grp.ranks[0].fill_guardcells()
    grp.ranks[0].close()

    p = si.Problem("g", 2, (8, 8, 1), (4, 4, 1), 2, 1, 1, 2, 0.4, bc=((0, 0), (0, 0), (1, 1)))
    rlo, rhi = (1, 1, 0), (3, 3, 1)
    ag = sp.AmrGroup(p.config(), rlo, rhi, 2)
    h0 = ag._handles[0]
    ag.ranks[1].close()
    st = sp.lib().spark_amr_step_group((ctypes.c_void_p * 1)(h0), 1, 1e-5, 0.0, None)
    assert st == sp.SPARK_ERR_STATE
    ag.ranks[0].close()
