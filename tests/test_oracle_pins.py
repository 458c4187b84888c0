"""Pins for the CPU oracle against what the mathematics and textbooks fix.

Each test names the property it checks and why a plausible mistake in the
oracle would fail it.  PAPER.md prints no numerical results for Spark, so the
pins are closed forms, invariants, special cases and brute force.
"""
import math
import os

import numpy as np
import pytest

import oracle
import spark_inputs as si
from tests import exact_riemann as er

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def cons(p: si.Problem, W):
    return oracle.prim_to_cons(p.ndim, p.gamma, W)


def ulp_diff(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return np.abs(a - b) / np.spacing(np.maximum(np.abs(a), np.abs(b)))


# --------------------------------------------------------------- config checks
def test_config_validation():
    p = si.PRESETS["c1_sod1d"]
    assert oracle.check_config(p.config()) == 0
    assert oracle.check_config(p.with_(ng=1).config()) != 0          # PLM needs ng >= 2
    assert oracle.check_config(p.with_(recon=2, ng=2).config()) != 0  # WENO5 needs ng >= 3
    assert oracle.check_config(p.with_(rk_stages=4).config()) != 0
    assert oracle.check_config(p.with_(nb=(1, 1, 1)).config()) != 0   # nb < ng


# ------------------------------------------------------- guard fill brute force
def _brute_map(g, N, lo, hi):
    """Per-dimension guard map written independently: returns (index, flip)."""
    if 0 <= g < N:
        return g, False
    bc = lo if g < 0 else hi
    if bc == si.BC_PERIODIC:
        return g % N, False
    if bc == si.BC_OUTFLOW:
        return (0 if g < 0 else N - 1), False
    return (-1 - g if g < 0 else 2 * N - 1 - g), True


GUARD_CASES = [
    si.Problem("g1", 1, (4, 1, 1), (3, 1, 1), 2, 1, 1, 2, 0.8, bc=((0, 1), (1, 1), (1, 1))),
    si.Problem("g1r", 1, (5, 1, 1), (2, 1, 1), 3, 2, 1, 3, 0.8, bc=((2, 0), (1, 1), (1, 1))),
    si.Problem("g2", 2, (4, 3, 1), (2, 3, 1), 2, 1, 1, 2, 0.4, bc=((0, 0), (1, 2), (1, 1))),
    si.Problem("g3", 3, (3, 4, 3), (2, 2, 3), 3, 2, 1, 3, 0.3, bc=((2, 1), (0, 0), (1, 2))),
    si.Problem("g3p", 3, (4, 4, 4), (1, 2, 1), 2, 1, 1, 2, 0.3, bc=((0, 0), (0, 0), (0, 0))),
]


@pytest.mark.parametrize("p", GUARD_CASES, ids=lambda p: p.name)
def test_guard_fill_bruteforce(p):
    """Every padded cell (faces, edges, corners) equals the per-dimension map of
    its global index; reflect negates the normal momentum.  Index-encoded state
    U[v][g] = v 2^32 + g makes any block/cell/variable mix-up visible (bit-exact)."""
    U = si.index_encoded(p)
    P = oracle.fill_guardcells(p.config(), U)
    N = [p.nblk[d] * p.nb[d] for d in range(3)]
    G = si.to_global(p, U)
    g = [p.ng if d < p.ndim else 0 for d in range(3)]
    nb = p.nb
    for b in range(int(np.prod(p.nblk))):
        bx, by, bz = b % p.nblk[0], (b // p.nblk[0]) % p.nblk[1], b // (p.nblk[0] * p.nblk[1])
        for pk in range(nb[2] + 2 * g[2]):
            for pj in range(nb[1] + 2 * g[1]):
                for pi in range(nb[0] + 2 * g[0]):
                    mx, fx = _brute_map(bx * nb[0] + pi - g[0], N[0], *p.bc[0])
                    my, fy = _brute_map(by * nb[1] + pj - g[1], N[1], *p.bc[1])
                    mz, fz = _brute_map(bz * nb[2] + pk - g[2], N[2], *p.bc[2])
                    flips = (fx, fy, fz)
                    for v in range(p.nvar):
                        want = G[v, mz, my, mx]
                        if 1 <= v <= p.ndim and flips[v - 1]:
                            want = -want
                        assert P[v, b, pk, pj, pi] == want


# ------------------------------------------------------------------------- EOS
def test_eos_hand_values():
    # 1-D: W = (rho, u, p) = (1, 0.5, 2): E = 2/0.4 + 0.5*1*0.25 = 5.125
    U = oracle.prim_to_cons(1, 1.4, np.array([1.0, 0.5, 2.0]))
    # (1.4 - 1 is not exactly 0.4 in binary: allow a few ulp)
    assert np.allclose(U, [1.0, 0.5, 5.125], rtol=1e-15, atol=0)
    # 3-D: W = (2, 1, -1, 0.5, 0.4): m = (2,-2,1), E = 0.4/0.4 + 0.5*2*2.25 = 3.25
    U = oracle.prim_to_cons(3, 1.4, np.array([2.0, 1.0, -1.0, 0.5, 0.4]))
    assert np.allclose(U, [2.0, 2.0, -2.0, 1.0, 3.25], rtol=1e-15, atol=0)
    W = oracle.cons_to_prim(3, 1.4, U)
    assert np.allclose(W, [2.0, 1.0, -1.0, 0.5, 0.4], rtol=1e-14, atol=0)


@pytest.mark.parametrize("ndim", [1, 2, 3])
def test_eos_roundtrip(ndim):
    g = np.random.Generator(np.random.PCG64(7))
    n = 2000
    W = np.empty((ndim + 2, n))
    W[0] = g.uniform(0.1, 10.0, n)
    W[1:ndim + 1] = g.uniform(-2, 2, (ndim, n))
    W[ndim + 1] = g.uniform(0.1, 10.0, n)
    W2 = oracle.cons_to_prim(ndim, 1.4, oracle.prim_to_cons(ndim, 1.4, W))
    assert np.all(ulp_diff(W2[0], W[0]) <= 0)
    assert np.max(np.abs(W2 - W) / np.abs(W)) < 1e-13


# -------------------------------------------------------------- reconstruction
def test_plm_linear_exact_and_extrema():
    g = np.random.Generator(np.random.PCG64(1))
    for _ in range(200):
        a, s = g.uniform(-3, 3), g.uniform(-3, 3)
        w = [a + s * m for m in range(4)]  # W_{i-1..i+2}, exactly representable-ish
        l, r = oracle.plm_face(*w)
        face = a + s * 1.5
        assert abs(l - face) <= 4 * np.spacing(abs(face) + 3 * abs(s))
        assert abs(r - face) <= 4 * np.spacing(abs(face) + 3 * abs(s))
    # constant: unchanged
    assert oracle.plm_face(2.0, 2.0, 2.0, 2.0) == (2.0, 2.0)
    # local extremum in cell i -> zero slope there -> W_L = W_i; same for i+1
    assert oracle.plm_face(1.0, 3.0, 2.0, 4.0)[0] == 3.0
    assert oracle.plm_face(1.0, 3.0, 2.0, 4.0)[1] == 2.0
    # minmod picks the smaller slope: W = (0, 1, 3, 4) -> slopes (1,2)->1, (2,1)->1
    assert oracle.plm_face(0.0, 1.0, 3.0, 4.0) == (1.5, 2.5)


def test_weno5_quadratic_exact():
    """Cell averages of any quadratic -> exact edge value (each candidate stencil
    reproduces quadratics, so any convex combination does)."""
    g = np.random.Generator(np.random.PCG64(2))
    for _ in range(200):
        c0, c1, c2 = g.uniform(-2, 2, 3)
        # average of q over [m-1/2, m+1/2] (unit cells) = q(m) + c2/12
        avg = [c0 + c1 * m + c2 * (m * m + 1.0 / 12.0) for m in range(-2, 4)]  # W_{i-2..i+3}, i = 0
        face = c0 + c1 * 0.5 + c2 * 0.25
        l, r = oracle.weno5_face(np.array(avg))
        scale = abs(c0) + abs(c1) + abs(c2) + 1
        assert abs(l - face) < 1e-13 * scale
        assert abs(r - face) < 1e-13 * scale


def test_weno5_order_smooth():
    """Reconstruction-only error on sin(2 pi x) averages: observed order well above
    any second-order scheme (JS weights lose some order near critical points)."""
    errs = []
    Ns = [32, 64, 128, 256]
    for N in Ns:
        h = 1.0 / N
        xl = np.arange(N) * h
        avg = (np.cos(2 * np.pi * xl) - np.cos(2 * np.pi * (xl + h))) / (2 * np.pi * h)
        e = 0.0
        for i in range(N):
            s = [avg[(i + m) % N] for m in range(-2, 4)]
            l, r = oracle.weno5_face(np.array(s))
            exact = math.sin(2 * math.pi * (i + 1) * h)
            e += (abs(l - exact) + abs(r - exact)) * h
        errs.append(e)
    orders = [math.log2(errs[n] / errs[n + 1]) for n in range(len(Ns) - 1)]
    assert min(orders[1:]) > 3.5, orders
    assert orders[-1] > 4.5, orders


# -------------------------------------------------------------------- Riemann
def phys_flux_1d(W, g=1.4):
    r, u, p = W
    E = p / (g - 1) + 0.5 * r * u * u
    return np.array([r * u, r * u * u + p, u * (E + p)])


@pytest.mark.parametrize("kind", [0, 1])
def test_riemann_consistency_hand_value(kind):
    # W = (1, 0.5, 1): f = (0.5, 1.25, 0.5*(2.5 + 0.125 + 1) = 1.8125)
    f = oracle.riemann(kind, 1.4, [1.0, 0.5, 1.0], [1.0, 0.5, 1.0])
    assert np.allclose(f, [0.5, 1.25, 1.8125], rtol=1e-15, atol=1e-16)


@pytest.mark.parametrize("kind", [0, 1])
def test_riemann_consistency_random(kind):
    g = np.random.Generator(np.random.PCG64(3))
    for _ in range(200):
        W = np.array([g.uniform(0.1, 5), g.uniform(-3, 3), g.uniform(-1, 1), g.uniform(-1, 1), g.uniform(0.1, 5)])
        f = oracle.riemann(kind, 1.4, W, W)
        r, u, v, w, p = W
        E = p / 0.4 + 0.5 * r * (u * u + v * v + w * w)
        want = np.array([r * u, r * u * u + p, r * u * v, r * u * w, u * (E + p)])
        assert np.allclose(f, want, rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("kind", [0, 1])
def test_riemann_supersonic_upwind(kind):
    # both states move right faster than sound: S_L >= 0 -> F = f(W_L) exactly
    WL, WR = [1.0, 3.0, 1.0], [0.5, 2.9, 0.4]
    f = oracle.riemann(kind, 1.4, WL, WR)
    assert np.array_equal(f, oracle.riemann(kind, 1.4, WL, WL))
    WL, WR = [1.0, -3.0, 1.0], [0.5, -2.9, 0.4]
    f = oracle.riemann(kind, 1.4, WL, WR)
    assert np.array_equal(f, oracle.riemann(kind, 1.4, WR, WR))


def test_hllc_stationary_contact():
    # HLLC resolves an isolated stationary contact exactly: no mass or energy
    # flux, momentum flux = p; transverse velocity jump is carried passively.
    f = oracle.riemann(1, 1.4, [1.0, 0.0, 0.3, 1.0], [0.125, 0.0, -0.7, 1.0])
    assert abs(f[0]) < 1e-15 and abs(f[2]) < 1e-15 and abs(f[3]) < 1e-15
    assert abs(f[1] - 1.0) < 1e-15


@pytest.mark.parametrize("kind", [0, 1])
def test_riemann_mirror_antisymmetry(kind):
    """F(sigma W_R, sigma W_L) = -sigma F(W_L, W_R), sigma flips u_n."""
    g = np.random.Generator(np.random.PCG64(4))
    for _ in range(300):
        WL = np.array([g.uniform(0.1, 5), g.uniform(-2, 2), g.uniform(-1, 1), g.uniform(0.1, 5)])
        WR = np.array([g.uniform(0.1, 5), g.uniform(-2, 2), g.uniform(-1, 1), g.uniform(0.1, 5)])
        sig = np.array([1.0, -1.0, 1.0, 1.0])
        f = oracle.riemann(kind, 1.4, WL, WR)
        fm = oracle.riemann(kind, 1.4, sig * WR, sig * WL)
        scale = np.max(np.abs(f)) + 1.0
        assert np.allclose(fm, -sig * f, rtol=0, atol=1e-13 * scale)


def test_hll_vs_hllc_differ_only_inside_fan():
    # inside the fan with a contact, HLL smears it (nonzero mass flux) while HLLC does not
    fh = oracle.riemann(0, 1.4, [1.0, 0.0, 1.0], [0.125, 0.0, 1.0])
    fc = oracle.riemann(1, 1.4, [1.0, 0.0, 1.0], [0.125, 0.0, 1.0])
    assert abs(fh[0]) > 1e-3 and abs(fc[0]) < 1e-15


# ------------------------------------------------------------------ RK coeffs
def test_rk_coeffs_consistency():
    # each stage is a convex combination (a + b = 1) and the scheme is consistent:
    # for L = const the Shu-Osher stages reproduce U^n + dt L exactly in reals.
    for S in (2, 3):
        for s in range(1, S + 1):
            a, b = oracle.rk_coeffs(S, s)
            assert abs(a + b - 1.0) < 1e-16 and a >= 0 and b > 0
    # RK3 literals (Gottlieb & Shu 1998, Eq. 4.2)
    assert oracle.rk_coeffs(3, 2) == (0.75, 0.25)
    assert oracle.rk_coeffs(3, 3) == (1.0 / 3.0, 2.0 / 3.0)
    assert oracle.rk_coeffs(2, 2) == (0.5, 0.5)


# ----------------------------------------------------------------------- Sod
def _golden_sod():
    vals = {}
    with open(os.path.join(GOLDEN, "toro_sod_test1.txt")) as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                k, v = line.split()
                vals[k] = float(v)
    return vals


def test_exact_solver_matches_toro_table():
    gold = _golden_sod()
    WL, WR = (1.0, 0.0, 1.0), (0.125, 0.0, 0.1)
    ps, us = er.star_state(WL, WR)
    rl, rr = er.star_densities(WL, WR, ps)
    assert abs(ps - gold["p_star"]) < 1e-5
    assert abs(us - gold["u_star"]) < 1e-5
    assert abs(rl - gold["rho_star_L"]) < 1e-5
    assert abs(rr - gold["rho_star_R"]) < 1e-5


def _sod_run(N, recon=1, rk=2, ng=2):
    p = si.PRESETS["c1_sod1d"].with_(nblk=(N // 8, 1, 1), recon=recon, rk_stages=rk, ng=ng)
    U0 = cons(p, si.initial_primitive(p))
    U, t, n = oracle.run(p.config(), U0, t_end=0.2)
    W = oracle.cons_to_prim(1, 1.4, U)
    return p, si.to_global(p, W)[:, 0, 0, :], t, n


def test_sod_vs_exact_c1():
    """configs[0]: plateau means within 1 %, wave locations within 3 dx."""
    p, W, t, n = _sod_run(256)
    assert abs(t - 0.2) < 1e-12 and n > 10
    N = 256
    h = 1.0 / N
    x = (np.arange(N) + 0.5) * h
    WL, WR = (1.0, 0.0, 1.0), (0.125, 0.0, 0.1)
    head, tail, contact, shock = er.wave_positions(WL, WR, 0.2)
    ps, us = er.star_state(WL, WR)
    rl, rr = er.star_densities(WL, WR, ps)
    away = lambda a, b: (x > a + 4 * h) & (x < b - 4 * h)
    # star-left plateau (tail..contact), star-right plateau (contact..shock)
    for sel, want in [(away(tail, contact), (rl, us, ps)), (away(contact, shock), (rr, us, ps))]:
        assert sel.sum() >= 4
        for v in range(3):
            assert abs(W[v, sel].mean() - want[v]) < 0.01 * abs(want[v]), (v, W[v, sel].mean(), want[v])
    # shock location: where rho crosses the mid value between rho*_R and rho_R
    mid = 0.5 * (rr + 0.125)
    xs = x[np.argmax((W[0][:-1] > mid) & (W[0][1:] <= mid) & (x[:-1] > contact))]
    assert abs(xs - shock) < 3 * h
    # contact: rho crosses the mean of the star densities
    midc = 0.5 * (rl + rr)
    xc = x[np.argmax((W[0][:-1] > midc) & (W[0][1:] <= midc) & (x[:-1] > tail))]
    assert abs(xc - contact) < 4 * h
    # exact solution L1 error
    ex = er.sample(WL, WR, (x - 0.5) / 0.2)
    assert np.mean(np.abs(W[0] - ex[0])) < 0.01


def test_sod_convergence():
    """L1(rho) error against the exact solution decreases under refinement."""
    WL, WR = (1.0, 0.0, 1.0), (0.125, 0.0, 0.1)
    errs = []
    for N in (128, 256, 512, 1024):
        _, W, _, _ = _sod_run(N)
        x = (np.arange(N) + 0.5) / N
        ex = er.sample(WL, WR, (x - 0.5) / 0.2)
        errs.append(np.mean(np.abs(W[0] - ex[0])))
    assert all(errs[n + 1] < 0.8 * errs[n] for n in range(3)), errs


def test_sod_weno5_rk3_and_hll():
    WL, WR = (1.0, 0.0, 1.0), (0.125, 0.0, 0.1)
    x = (np.arange(256) + 0.5) / 256
    ex = er.sample(WL, WR, (x - 0.5) / 0.2)
    _, W, _, _ = _sod_run(256, recon=2, rk=3, ng=3)
    assert np.mean(np.abs(W[0] - ex[0])) < 0.01
    p = si.PRESETS["c1_sod1d"].with_(riemann=0)
    U, _, _ = oracle.run(p.config(), cons(p, si.initial_primitive(p)), t_end=0.2)
    Wh = si.to_global(p, oracle.cons_to_prim(1, 1.4, U))[0, 0, 0]
    assert np.mean(np.abs(Wh - ex[0])) < 0.015


# -------------------------------------------------------------- invariants
@pytest.mark.parametrize("case", [
    si.Problem("u2", 2, (8, 8, 1), (3, 2, 1), 2, 1, 1, 2, 0.4, bc=((0, 0),) * 3),
    si.Problem("u3w", 3, (6, 5, 4), (2, 2, 2), 3, 2, 1, 3, 0.3, bc=((0, 0),) * 3),
    si.Problem("u3h", 3, (4, 4, 4), (2, 2, 2), 2, 1, 0, 2, 0.3, bc=((0, 0),) * 3),
], ids=lambda p: p.name)
def test_uniform_state_preserved(case):
    """Every face flux is identical, so F+ - F- == 0 exactly: the state stays
    spatially bitwise uniform; RK2 changes no value at all."""
    U0 = cons(case, si.uniform_state(case, 11))
    U, _, n = oracle.run(case.config(), U0, max_steps=3)
    for v in range(case.nvar):
        assert np.all(U[v] == U[v].flat[0])
    if case.rk_stages == 2:
        assert np.array_equal(U, U0)
    else:
        assert np.max(ulp_diff(U, U0)) <= 3


def test_conservation_periodic_c2b():
    """configs[1] reading C2b: sum U dV conserved to round-off with periodic BCs."""
    p = si.PRESETS["c2b_sod2d"]
    U0 = cons(p, si.initial_primitive(p))
    U, t, n = oracle.run(p.config(), U0, max_steps=40)
    assert n == 40
    for v in range(p.nvar):
        s0, s1 = U0[v].sum(), U[v].sum()
        scale = np.abs(U0[v]).sum() + np.abs(U[v]).sum()
        assert abs(s1 - s0) <= 1e-13 * scale, (v, s0, s1)


def test_2d_rows_equal_1d_c2a():
    """configs[1] reading C2a: each row of the x-aligned 2-D Sod equals a 1-D run
    with the same cells and CFL number, bitwise (y-fluxes cancel exactly)."""
    p2 = si.PRESETS["c2a_sod2d"]
    U2, t2, n2 = oracle.run(p2.config(), cons(p2, si.initial_primitive(p2)), t_end=0.2)
    p1 = si.PRESETS["c1_sod1d"].with_(nblk=(16, 1, 1), nb=(8, 1, 1), cfl=p2.cfl)
    U1, t1, n1 = oracle.run(p1.config(), cons(p1, si.initial_primitive(p1)), t_end=0.2)
    assert n1 == n2 and t1 == t2
    G2 = si.to_global(p2, U2)
    G1 = si.to_global(p1, U1)
    for row in range(G2.shape[2]):
        assert np.array_equal(G2[0, 0, row], G1[0, 0, 0])
        assert np.array_equal(G2[1, 0, row], G1[1, 0, 0])
        assert np.array_equal(G2[3, 0, row], G1[2, 0, 0])
        assert np.all(G2[2, 0, row] == 0.0)


def test_block_decomposition_invariance():
    """The same global state split into different block shapes gives bitwise the
    same result and the same dt (blocks are indistinguishable from the domain,
    P:361-364) — pins block indexing and the guard fill inside the stage."""
    base = si.Problem("d", 2, (8, 8, 1), (4, 3, 1), 3, 2, 1, 3, 0.4,
                      bc=((1, 2), (0, 0), (1, 1)), ic="blocky")
    W = si.to_global(base, si.random_state(base, 5, blocky=True))
    outs = []
    for nb, nblk in [((8, 8, 1), (4, 3, 1)), ((4, 6, 1), (8, 4, 1)), ((32, 3, 1), (1, 8, 1))]:
        p = base.with_(nb=nb, nblk=nblk)
        U0 = cons(p, si.from_global(p, W))
        U, dt = oracle.step(p.config(), U0)
        outs.append((si.to_global(p, U), dt))
    for G, dt in outs[1:]:
        assert dt == outs[0][1]
        assert np.array_equal(G, outs[0][0])


@pytest.mark.parametrize("ndim", [2, 3])
def test_sedov_symmetry(ndim):
    """Sedov (configs[2], [3] shapes, reduced): x<->y transposition is bitwise
    (summation order (x+y)+z, reading R9); mirror x -> 1-x holds to 1e-10."""
    if ndim == 2:
        p = si.PRESETS["c3_sedov2d"].with_(nblk=(4, 4, 1))
    else:
        p = si.PRESETS["c4_sedov3d_weno"].with_(nb=(8, 8, 8), nblk=(2, 2, 2))
    U, t, n = oracle.run(p.config(), cons(p, si.initial_primitive(p)), max_steps=4)
    G = si.to_global(p, U)
    # transposition x <-> y: swap axes and the two momenta
    T = np.swapaxes(G, -1, -2).copy()
    T[[1, 2]] = T[[2, 1]]
    assert np.array_equal(T, G)
    # mirror x -> 1 - x: flip x, negate x-momentum
    M = G[..., ::-1].copy()
    M[1] = -M[1]
    scale = np.abs(G).max(axis=(1, 2, 3), keepdims=True)
    assert np.all(np.abs(M - G) <= 1e-10 * scale)


def test_sedov_energy_and_growth():
    """2-D Sedov: mass/energy conserved while the shock is inside the box;
    shock radius R ~ t^(1/2) (dimensional analysis: R = xi (E t^2/rho)^(1/4)),
    fitted exponent within 5 %.  R = peak of the angle-averaged density profile
    (parabolic sub-bin refinement)."""
    p = si.PRESETS["c3_sedov2d"].with_(nblk=(8, 8, 1), recon=1, ng=2, rk_stages=2)
    U0 = cons(p, si.initial_primitive(p))
    x, y, _ = si.centres(p)
    r = np.hypot(x - 0.5, y - 0.5)
    h = 1.0 / 128
    bins = np.arange(0, 0.5 + h, h)
    idx = np.digitize(r.ravel(), bins) - 1
    cnt = np.maximum(np.bincount(idx, minlength=len(bins)), 1)
    radii, times = [], []
    U, t = U0, 0.0
    for t_target in (0.01, 0.06):
        U, t, _ = oracle.run(p.config(), U, t_end=t_target, t0=t)
        rho = si.to_global(p, U)[0, 0]
        prof = np.bincount(idx, weights=rho.ravel(), minlength=len(bins)) / cnt
        k = int(np.argmax(prof))
        a, b, c = prof[k - 1], prof[k], prof[k + 1]
        radii.append((k + 0.5 + 0.5 * (a - c) / (a - 2 * b + c)) * h)
        times.append(t)
    for v in (0, 3):
        assert abs(U[v].sum() - U0[v].sum()) <= 1e-12 * abs(U0[v].sum())
    expo = math.log(radii[1] / radii[0]) / math.log(times[1] / times[0])
    assert abs(expo - 0.5) < 0.025, expo


# ---------------------------------------------------------- convergence order
def _wave_error(N, recon, rk, ng, cfl):
    p = si.Problem("w", 1, (8, 1, 1), (N // 8, 1, 1), ng, recon, 1, rk, cfl, bc=((0, 0),) * 3)
    U0 = cons(p, si.density_wave_avg(p, 0.0))
    U, t, _ = oracle.run(p.config(), U0, t_end=0.25)
    rho = si.to_global(p, U)[0, 0, 0]
    ex = si.to_global(p, si.density_wave_avg(p, t))[0, 0, 0]
    return np.mean(np.abs(rho - ex))


def test_density_wave_order_plm_rk2():
    """Exact solution: a density wave advected at u = 1 (pure contact)."""
    e = [_wave_error(N, 1, 2, 2, 0.8) for N in (32, 64, 128, 256)]
    orders = [math.log2(e[n] / e[n + 1]) for n in range(3)]
    assert orders[-1] > 1.7, orders


def test_density_wave_order_weno5_rk3():
    e = [_wave_error(N, 2, 3, 3, 0.8) for N in (32, 64, 128)]
    orders = [math.log2(e[n] / e[n + 1]) for n in range(2)]
    assert orders[-1] > 2.7, orders


def test_dt_min_is_exact_min():
    """dt = C min over cells of dx/(|u|+c): compare with a brute-force min."""
    p = si.Problem("dt", 2, (8, 8, 1), (2, 3, 1), 2, 1, 1, 2, 0.4, bc=((0, 0),) * 3, hi=(1.0, 1.5, 1.0))
    W = si.random_state(p, 9)
    U = cons(p, W)
    Wg = si.to_global(p, W)
    c = np.sqrt(1.4 * Wg[3] / Wg[0])
    dx, dy = 1.0 / 16, 1.5 / 24
    m = min((dx / (np.abs(Wg[1]) + c)).min(), (dy / (np.abs(Wg[2]) + c)).min())
    assert abs(oracle.dt_raw(p.config(), U) - m) <= 2 * np.spacing(m)
    assert oracle.dt(p.config(), U, 0.0, 0.0) == pytest.approx(0.4 * m, rel=1e-15)
    # clip to t_end - t
    assert oracle.dt(p.config(), U, 0.99, 1.0) == pytest.approx(0.01, rel=1e-12)


def test_nonphysical_detected():
    p = si.Problem("np", 1, (8, 1, 1), (2, 1, 1), 2, 1, 1, 2, 0.8)
    W = si.random_state(p, 1)
    U = cons(p, W)
    U[0, 0, 0, 0, 3] = -1.0  # negative density
    with pytest.raises(oracle.OracleError):
        oracle.step(p.config(), U, dt_fixed=1e-3)


def test_rotation_invariance_3d():
    """A 1-D profile with constant transverse velocities, laid along x, y or z of
    a 3-D periodic box, evolves identically (to round-off) in each orientation:
    pins the rotated frame of every direction (normal / transverse components and
    the full |u|^2 in the energy)."""
    N = 32
    g = np.random.Generator(np.random.PCG64(21))
    rho = g.uniform(0.5, 1.5, N) * np.where(np.arange(N) % 11 < 5, 1.0, 4.0)
    pres = g.uniform(0.5, 1.5, N) * np.where(np.arange(N) % 7 < 3, 1.0, 10.0)
    un = g.uniform(-0.5, 0.5, N)
    ut1, ut2 = 0.3, -0.45
    res = []
    for axis in range(3):
        nb = [4, 4, 4]
        nblk = [1, 1, 1]
        nb[axis], nblk[axis] = 8, N // 8
        p = si.Problem("rot", 3, tuple(nb), tuple(nblk), 3, 2, 1, 3, 0.3, bc=((0, 0),) * 3)
        shape = [4, 4, 4]
        shape[axis] = N
        sh = (shape[2], shape[1], shape[0])
        bshape = [1, 1, 1]
        bshape[2 - axis] = N
        line = lambda a: np.broadcast_to(np.asarray(a, dtype=float).reshape(bshape) if np.ndim(a) else a, sh)
        vel = [None, None, None]
        tr = iter([ut1, ut2])
        for d in range(3):
            vel[d] = line(un) if d == axis else line(next(tr))
        W = np.stack([line(rho), vel[0], vel[1], vel[2], line(pres)]).astype(float)
        U0 = cons(p, si.from_global(p, W))
        U, _ = oracle.step(p.config(), U0, dt_fixed=2e-3)
        U, _ = oracle.step(p.config(), U, dt_fixed=2e-3)
        G = si.to_global(p, U)
        idx = [0, 0, 0]
        idx[2 - axis] = slice(None)
        prof = G[(slice(None),) + tuple(idx)]          # [v][N]
        order = [0, 1 + axis] + [1 + d for d in range(3) if d != axis] + [4]
        res.append(prof[order])
    for r in res[1:]:
        assert np.allclose(r, res[0], rtol=1e-13, atol=1e-14)
