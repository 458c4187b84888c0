"""Pins for the NEXT-N2 additions to the oracle: the
monotonized-central PLM limiter, WENO5-Z, and the grvAccel gravity source.

The paper gives no formula for any of them (P:1815, P:1831 name the nodes
only); readings R18-R20 fix the textbook forms.  Each pin is a
closed form, a convergence order, a bound or an exact invariant, chosen so a
dropped factor, a wrong sign or a swapped stencil fails it.
"""
import math

import numpy as np
import pytest

import oracle
import spark_inputs as si


def cons(p, W):
    return oracle.prim_to_cons(p.ndim, p.gamma, W)


# ------------------------------------------------------------------ PLM-MC
def test_mc_linear_data_exact():
    """Slopes of linear data are the data's slope (2d, d, 2d -> d)."""
    for a, d in [(0.0, 1.0), (3.0, -0.25), (-1.0, 2.5)]:
        w = [a + k * d for k in range(4)]
        l, r = oracle.mc_face(*w)
        assert l == pytest.approx(a + 1.5 * d, rel=1e-15) and r == pytest.approx(a + 1.5 * d, rel=1e-15)


def test_mc_closed_forms():
    # centred slope inside the 2x bounds: (0, 1, 3): dl = 1, dr = 2 -> 1.5
    l, _ = oracle.mc_face(0.0, 1.0, 3.0, 6.0)
    assert l == 1.75
    # 2 dl binds: (0, 1, 5): min(2, 2.5, 8) = 2
    l, _ = oracle.mc_face(0.0, 1.0, 5.0, 9.0)
    assert l == 2.0
    # right state of the face uses cell i+1's slope: (1, 5, 9) -> dl = 4, dr = 4 -> 4
    _, r = oracle.mc_face(0.0, 1.0, 5.0, 9.0)
    assert r == 5.0 - 2.0
    # extremum: zero slope; plateau: zero slope
    assert oracle.mc_face(0.0, 1.0, 0.0, 1.0) == (1.0, 0.0)
    assert oracle.mc_face(1.0, 1.0, 2.0, 2.0) == (1.0, 2.0)
    # negative monotone data mirror the positive case
    l, _ = oracle.mc_face(0.0, -1.0, -3.0, -6.0)
    assert l == -1.75


def test_mc_is_between_plm_and_the_bounds():
    """|MC slope| >= |minmod slope| and the face value stays within the two
    neighbouring cell values (the TVD bound |slope| <= 2 min(|dl|, |dr|))."""
    g = np.random.default_rng(5)
    for _ in range(4000):
        w = g.normal(size=4) * g.choice([1e-3, 1.0, 1e3])
        l, r = oracle.mc_face(*w)
        lp, rp = oracle.plm_face(*w)
        assert abs(l - w[1]) >= abs(lp - w[1]) * (1 - 1e-15)
        assert abs(w[2] - r) >= abs(w[2] - rp) * (1 - 1e-15)
        lo, hi = min(w[1], w[2]), max(w[1], w[2])
        assert lo - 1e-12 * abs(hi) <= l <= hi + 1e-12 * abs(hi)
        assert lo - 1e-12 * abs(hi) <= r <= hi + 1e-12 * abs(hi)


def test_mc_second_order_convergence():
    """Smooth monotone data: face-value error falls 4x per halving of h."""
    def err(n):
        h = 1.0 / n
        x = (np.arange(-2, n + 2) + 0.5) * h
        avg = (np.cos(x - h / 2) - np.cos(x + h / 2)) / h  # cell averages of sin (monotone on [0, 1])
        e = 0.0
        for i in range(2, n + 1):
            l, _ = oracle.mc_face(avg[i - 1], avg[i], avg[i + 1], avg[i + 2])
            e = max(e, abs(l - math.sin(x[i] + h / 2)))
        return e

    r = err(64) / err(128)
    assert 3.5 < r < 4.6


# ----------------------------------------------------------------- WENO5-Z
def test_wenoz_linear_and_constant_exact():
    assert oracle.weno5z_edge(1.0, 2.0, 3.0, 4.0, 5.0) == pytest.approx(3.5, rel=1e-15)
    assert oracle.weno5z_edge(2.0, 2.0, 2.0, 2.0, 2.0) == 2.0
    # linear data: all beta equal -> tau5 = 0 -> linear weights -> exact
    for a, d in [(0.3, -0.7), (-5.0, 1e-3)]:
        s = [a + k * d for k in range(5)]
        assert oracle.weno5z_edge(*s) == pytest.approx(a + 2.5 * d, rel=1e-14, abs=1e-15)


def test_wenoz_linear_weights_closed_form():
    """Data symmetric about c give beta_0 = beta_2, so tau5 = 0 and WENO-Z
    takes the linear weights (0.1, 0.6, 0.3): the edge value is then the fixed
    5-point formula (2a - 13b + 47c + 27d - 3e) / 60 (JS weights would not be)."""
    a, b, c, d, e = 1.0, 4.0, 2.0, 4.0, 1.0
    ref = (2 * a - 13 * b + 47 * c + 27 * d - 3 * e) / 60.0
    assert oracle.weno5z_edge(a, b, c, d, e) == pytest.approx(ref, rel=1e-14)
    # WENO5-JS differs there (its weights depend on beta_k individually)
    assert abs(oracle.weno5_edge(a, b, c, d, e) - ref) > 1e-3


def test_wenoz_discontinuity_is_eno():
    """A jump between c and d, (0,0,0,1,1), at the right edge of c: the smooth
    stencil (a, b, c) takes all the weight -> the edge value is ~0."""
    v = oracle.weno5z_edge(0.0, 0.0, 0.0, 1.0, 1.0)
    assert 0.0 <= v < 1e-30
    v = oracle.weno5z_edge(1.0, 1.0, 1.0, 0.0, 0.0)
    assert abs(v - 1.0) < 1e-30


def test_wenoz_fifth_order():
    """Cell averages of sin(2 pi x): edge error falls ~32x per halving of h."""
    def err(n):
        h = 1.0 / n
        k = 2 * math.pi
        x = (np.arange(-3, n + 3) + 0.5) * h
        avg = (np.cos(k * (x - h / 2)) - np.cos(k * (x + h / 2))) / (k * h)
        e = 0.0
        for i in range(3, n + 3):
            v = oracle.weno5z_edge(*avg[i - 2:i + 3])
            e = max(e, abs(v - math.sin(k * (x[i] + h / 2))))
        return e

    r = err(40) / err(80)
    assert r > 24.0


def test_wenoz_face_mirror():
    g = np.random.default_rng(8)
    for _ in range(200):
        s = g.normal(size=6)
        l, r = oracle.weno5z_face(s)
        l2, r2 = oracle.weno5z_face(s[::-1].copy())
        assert l == r2 and r == l2


# ------------------------------------------------------- grvAccel (gravity)
@pytest.mark.parametrize("ndim,rk", [(1, 2), (2, 3), (3, 2), (3, 3)])
def test_gravity_free_fall_exact(ndim, rk):
    """A uniform periodic state in uniform gravity stays uniform; m and E obey
    m' = rho g, E' = m . g, whose solution is quadratic in t, which SSP-RK2/3
    integrate exactly: m = m0 + rho g t, E = E0 + (m0 . g) t + rho |g|^2 t^2 / 2."""
    nb = (8, 8 if ndim > 1 else 1, 8 if ndim > 2 else 1)
    nblk = (2, 2 if ndim > 1 else 1, 2 if ndim > 2 else 1)
    g = (0.3, -1.1, 0.7)[:ndim] + (0.0,) * (3 - ndim)
    p = si.Problem("ff", ndim, nb, nblk, 2, 1, 1, rk, 0.3, bc=((0, 0),) * 3, grav=g)
    W = si.uniform_state(p, 11)
    U0 = cons(p, W)
    U, dt, t = U0, 1e-2, 0.0
    for _ in range(7):
        U, _ = oracle.step(p.config(), U, dt_fixed=dt)
        t += dt
    rho = U0[0].flat[0]
    m0 = [U0[1 + d].flat[0] for d in range(ndim)]
    E0 = U0[ndim + 1].flat[0]
    assert np.all(U[0] == rho)
    for d in range(ndim):
        assert np.allclose(U[1 + d], m0[d] + rho * g[d] * t, rtol=1e-13, atol=1e-15)
    E = E0 + sum(m0[d] * g[d] for d in range(ndim)) * t + 0.5 * rho * sum(x * x for x in g) * t * t
    assert np.allclose(U[ndim + 1], E, rtol=1e-13)


def test_gravity_momentum_budget():
    """Periodic, non-uniform state: fluxes telescope away, so every step adds
    exactly dt g M to the total momentum (M = total mass, itself conserved)."""
    p = si.Problem("gb", 2, (8, 8, 1), (3, 2, 1), 2, 1, 1, 2, 0.3, bc=((0, 0),) * 3, grav=(0.5, -2.0, 0.0))
    U = cons(p, si.random_state(p, 3))
    M = U[0].sum()
    for _ in range(4):
        mx, my = U[1].sum(), U[2].sum()
        U, dt = oracle.step(p.config(), U)
        assert abs(U[0].sum() - M) <= 1e-13 * M
        assert abs(U[1].sum() - (mx + dt * 0.5 * M)) <= 1e-12 * (abs(mx) + M)
        assert abs(U[2].sum() - (my - dt * 2.0 * M)) <= 1e-12 * (abs(my) + M)


def test_gravity_zero_is_identity():
    """g = 0 reproduces the gravity-free operator bit for bit."""
    p = si.Problem("g0", 2, (8, 8, 1), (2, 2, 1), 2, 1, 1, 2, 0.3, bc=((1, 1), (2, 2), (1, 1)))
    U0 = cons(p, si.random_state(p, 4, blocky=True))
    a, _ = oracle.step(p.config(), U0)
    b, _ = oracle.step(p.with_(grav=(0.0, 0.0, 0.0)).config(), U0)
    assert np.array_equal(a, b)
    c, _ = oracle.step(p.with_(grav=(0.0, 1e-3, 0.0)).config(), U0)
    assert not np.array_equal(a[2], c[2])  # the source acts (on y-momentum first)


def test_gravity_telescoping_matches_stagewise_periodic():
    p = si.Problem("gt", 2, (8, 8, 1), (3, 3, 1), 2, 1, 1, 2, 0.3, bc=((0, 0),) * 3, grav=(0.2, 0.4, 0.0))
    U0 = cons(p, si.random_state(p, 6, blocky=True))
    a, da = oracle.step(p.config(), U0)
    b, db = oracle.step_telescoping(p.config(), U0)
    assert da == db
    assert np.allclose(a, b, rtol=1e-13, atol=1e-14)


# ------------------------------------------------------------- config checks
def test_n2_config_validation():
    p = si.PRESETS["c1_sod1d"]
    assert oracle.check_config(p.with_(recon=3).config()) == 0            # MC: ng 2
    assert oracle.check_config(p.with_(recon=4, ng=2).config()) != 0      # WENO-Z needs ng 3
    assert oracle.check_config(p.with_(recon=4, ng=3).config()) == 0
    assert oracle.check_config(p.with_(recon=5, ng=3).config()) != 0


@pytest.mark.parametrize("recon", [0, 1, 2, 3, 4])
def test_extra_guard_layers_change_nothing(recon):
    """ng beyond the reconstruction's reach (NGK) adds guard layers nobody
    reads: the step is bitwise identical (regression: the oracle's stencil
    buffer once held only 6 cells and overflowed for WENO with ng = 4)."""
    ngk = 3 if recon in (2, 4) else (2 if recon in (1, 3) else 1)
    p = si.Problem("xg", 2, (8, 8, 1), (2, 2, 1), ngk, recon, 1, 3, 0.4, bc=((2, 1), (0, 0), (1, 1)))
    U0 = cons(p, si.random_state(p, 9, blocky=True))
    a, _ = oracle.step(p.config(), U0)
    b, _ = oracle.step(p.with_(ng=ngk + 1).config(), U0)
    assert np.array_equal(a, b)
