"""Pins for the telescoping SSP-RK oracle (PAPER.md P:1549-1561,
lst:spark-telescoping P:1598-1604): one thick guard fill per step, all stages
per block on the shrinking halo.

* periodic boundaries: every halo cell is some other block's interior cell, so
  the telescoped stage values are the same arithmetic on the same inputs as the
  non-telescoping step -> bitwise equal (any dimension, scheme, RK order);
* physical boundaries (reading R17: guards beyond the boundary are filled once
  and then evolved): the results differ only within (S-1)*NGK cells of the
  boundary after one step, and the whole scheme still converges to the exact
  Sod solution.
"""
import numpy as np
import pytest

import oracle
import spark_inputs as si
from tests import exact_riemann as er


def cons(p, W):
    return oracle.prim_to_cons(p.ndim, p.gamma, W)


NGK = {0: 1, 1: 2, 2: 3}

PERIODIC = [
    si.Problem("t1w", 1, (8, 1, 1), (4, 1, 1), 3, 2, 1, 3, 0.8, bc=((0, 0),) * 3),
    si.Problem("t1f", 1, (5, 1, 1), (3, 1, 1), 1, 0, 0, 2, 0.8, bc=((0, 0),) * 3),
    si.Problem("t2p", 2, (8, 8, 1), (3, 2, 1), 2, 1, 1, 2, 0.4, bc=((0, 0),) * 3),
    si.Problem("t2w", 2, (6, 7, 1), (2, 3, 1), 3, 2, 0, 3, 0.4, bc=((0, 0),) * 3),
    si.Problem("t3p", 3, (4, 4, 4), (2, 2, 3), 2, 1, 1, 3, 0.3, bc=((0, 0),) * 3),
]


@pytest.mark.parametrize("p", PERIODIC, ids=lambda p: p.name)
def test_periodic_telescoping_equals_nontelescoping(p):
    U = cons(p, si.random_state(p, 3, blocky=True))
    Ua, Ub = U, U
    for _ in range(3):
        Ua, da = oracle.step(p.config(), Ua)
        Ub, db = oracle.step_telescoping(p.config(), Ub)
        assert da == db
    assert np.array_equal(Ua, Ub)


@pytest.mark.parametrize("p", [
    si.Problem("o2", 2, (8, 8, 1), (3, 3, 1), 3, 2, 1, 3, 0.4, bc=((1, 2), (2, 1), (1, 1))),
    si.Problem("o3", 3, (4, 4, 4), (3, 2, 2), 2, 1, 1, 2, 0.3, bc=((1, 1), (2, 2), (1, 2))),
    si.Problem("o1", 1, (8, 1, 1), (4, 1, 1), 2, 1, 0, 3, 0.8, bc=((2, 1), (1, 1), (1, 1))),
], ids=lambda p: p.name)
def test_boundary_differences_confined(p):
    """Outflow / reflect: one telescoped step differs from the non-telescoping
    step only within (S-1)*NGK cells of a physical boundary."""
    U = cons(p, si.random_state(p, 7, blocky=True))
    Ua, da = oracle.step(p.config(), U)
    Ub, db = oracle.step_telescoping(p.config(), U)
    assert da == db
    Ga, Gb = si.to_global(p, Ua), si.to_global(p, Ub)
    w = (p.rk_stages - 1) * NGK[p.recon]
    N = [p.nblk[d] * p.nb[d] for d in range(3)]
    sl = [slice(None)]
    for d in (2, 1, 0):
        sl.append(slice(w, N[d] - w) if d < p.ndim else slice(None))
    assert np.array_equal(Ga[tuple(sl)], Gb[tuple(sl)])
    assert not np.array_equal(Ga, Gb)  # the boundary layer does differ
    scale = np.abs(Ga).max(axis=(1, 2, 3), keepdims=True)
    assert np.all(np.abs(Ga - Gb) <= 0.05 * scale)


def test_uniform_state_telescoping():
    # 12 cells per dimension >= the 9-cell telescoped halo (the oracle refuses less)
    p = si.Problem("u", 3, (4, 4, 4), (3, 3, 3), 3, 2, 1, 3, 0.3, bc=((1, 1), (2, 2), (0, 0)))
    W = si.uniform_state(p, 2)
    W[1:4] = 0.0  # at rest: reflect walls keep it uniform too
    U0 = cons(p, W)
    U = U0
    for _ in range(2):
        U, _ = oracle.step_telescoping(p.config(), U)
    for v in range(p.nvar):
        assert np.all(U[v] == U[v].flat[0])


def test_sod_telescoping_vs_exact():
    """configs[0] in telescoping mode: plateaus within 1 % of the exact solution."""
    p = si.PRESETS["c1_sod1d"]
    U = cons(p, si.initial_primitive(p))
    t = 0.0
    while t < 0.2 * (1 - 1e-14):
        U, dt = oracle.step_telescoping(p.config(), U, t, 0.2)
        t += dt
    W = si.to_global(p, oracle.cons_to_prim(1, 1.4, U))[:, 0, 0, :]
    x = (np.arange(256) + 0.5) / 256
    WL, WR = (1.0, 0.0, 1.0), (0.125, 0.0, 0.1)
    ex = er.sample(WL, WR, (x - 0.5) / 0.2)
    assert np.mean(np.abs(W[0] - ex[0])) < 0.01
    head, tail, contact, shock = er.wave_positions(WL, WR, 0.2)
    ps, us = er.star_state(WL, WR)
    rl, rr = er.star_densities(WL, WR, ps)
    h = 1 / 256
    sel = (x > contact + 4 * h) & (x < shock - 4 * h)
    assert abs(W[0, sel].mean() - rr) < 0.01 * rr


def test_halo_deeper_than_domain_refused():
    """S*NGK guard layers need that many cells per dimension (a reflect map of
    a deeper guard would leave the domain); the GPU refuses the same case."""
    p = si.Problem("d", 3, (4, 4, 4), (2, 2, 2), 3, 2, 1, 3, 0.3, bc=((1, 1), (2, 2), (0, 0)))
    with pytest.raises(oracle.OracleError):
        oracle.step_telescoping(p.config(), cons(p, si.uniform_state(p, 2)))
