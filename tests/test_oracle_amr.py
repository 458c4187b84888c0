"""Pins for the oracle's NEXT-N3 path: fluxBuff + flux correction on a static
two-level refinement, the all-levels variant (lst:spark-all-levels
P:1510-1523; Alg. 8 fluxBuff P:1834; readings R22/R23 in DESIGN.md §2).

What fixes the composite scheme without retyping it:
* guard cells: an independent formulation through two global arrays (the
  composite at fine resolution, coarse cells injected; at coarse resolution,
  fine cells averaged) on an index-encoded state (exact in FP64);
* limits: an empty refined box is the uniform coarse scheme, a box covering
  the domain is the uniform fine scheme — bit for bit;
* conservation to round-off over many steps with periodic boundaries (and a
  drift of order 1e-6 without the correction: the correction is what makes
  the composite update conservative);
* a uniform state stays bitwise uniform; x<->y transposition symmetry;
* Sod through a coarse-fine interface against the exact solution.
"""
import numpy as np
import pytest

import oracle
import spark_inputs as si
from tests import exact_riemann as er


def cons(p, W):
    nv, nl = W.shape[0], W.shape[1]
    return oracle.prim_to_cons(p.ndim, p.gamma, W.reshape(nv, nl, -1)).reshape(W.shape)


def mapped(g, N, bc_lo, bc_hi):
    """Per-dimension boundary map (periodic / outflow / reflect) -> (index, flip)."""
    if 0 <= g < N:
        return g, False
    bc = bc_lo if g < 0 else bc_hi
    if bc == si.BC_PERIODIC:
        return g % N, False
    if bc == si.BC_OUTFLOW:
        return (0 if g < 0 else N - 1), False
    return (-1 - g if g < 0 else 2 * N - 1 - g), True


def composite_globals(p, rlo, rhi, U):
    """(fine-resolution array with coarse cells injected, coarse-resolution
    array with fine cells averaged) of a leaf state U[v][leaf][k][j][i]."""
    leaves = si.amr_leaf_blocks(p, rlo, rhi)
    nv = U.shape[0]
    N = [p.nblk[d] * p.nb[d] for d in range(3)]
    r = [2 if d < p.ndim else 1 for d in range(3)]
    F = np.full((nv, N[2] * r[2], N[1] * r[1], N[0] * r[0]), np.nan)
    C = np.full((nv, N[2], N[1], N[0]), np.nan)
    nb = p.nb
    for q, (lev, b) in enumerate(leaves):
        if lev == 0:
            sl = tuple(slice(b[d] * nb[d], (b[d] + 1) * nb[d]) for d in (2, 1, 0))
            C[(slice(None),) + sl] = U[:, q]
            blk = U[:, q]
            for d in range(p.ndim):
                blk = np.repeat(blk, 2, axis=3 - d)
            slf = tuple(slice(b[d] * nb[d] * r[d], (b[d] + 1) * nb[d] * r[d]) for d in (2, 1, 0))
            F[(slice(None),) + slf] = blk
        else:
            slf = tuple(slice(b[d] * nb[d], (b[d] + 1) * nb[d]) for d in (2, 1, 0))
            F[(slice(None),) + slf] = U[:, q]
    # restriction of the refined box
    lo = [rlo[d] * nb[d] for d in range(3)]
    hi = [rhi[d] * nb[d] for d in range(3)]
    if all(rhi[d] > rlo[d] for d in range(3)):
        sub = F[:, lo[2] * r[2]:hi[2] * r[2], lo[1] * r[1]:hi[1] * r[1], lo[0] * r[0]:hi[0] * r[0]]
        sh = sub.shape
        m = sub.reshape(nv, sh[1] // r[2], r[2], sh[2] // r[1], r[1], sh[3] // r[0], r[0]).mean(axis=(2, 4, 6))
        C[:, lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]] = m
    return F, C


CASES_FILL = [
    (si.Problem("f2", 2, (4, 4, 1), (4, 3, 1), 2, 1, 1, 2, 0.4, bc=((0, 0), (1, 2), (1, 1))), (1, 1, 0), (3, 2, 1)),
    (si.Problem("f2e", 2, (4, 4, 1), (3, 3, 1), 2, 1, 1, 2, 0.4, bc=((2, 1), (0, 0), (1, 1))), (0, 0, 0), (2, 3, 1)),
    (si.Problem("f3", 3, (4, 4, 4), (3, 3, 2), 2, 1, 1, 2, 0.3, bc=((0, 0), (1, 1), (2, 0 + 2))), (1, 0, 0), (2, 2, 1)),
    (si.Problem("f1", 1, (6, 1, 1), (5, 1, 1), 3, 2, 1, 3, 0.8, bc=((0, 0), (1, 1), (1, 1))), (3, 0, 0), (5, 1, 1)),
]


@pytest.mark.parametrize("p,rlo,rhi", CASES_FILL, ids=lambda x: getattr(x, "name", str(x)))
def test_fill_against_composite_arrays(p, rlo, rhi):
    """Every face guard of every leaf equals the boundary-mapped cell of the
    composite array of its own level (index-encoded state: exact)."""
    leaves = si.amr_leaf_blocks(p, rlo, rhi)
    nc, nf = oracle.amr_leaves(p.config(), rlo, rhi)
    assert nc + nf == len(leaves)
    nl = len(leaves)
    U = np.stack([v * 2.0 ** 32 + np.arange(nl * int(np.prod(p.nb)), dtype=np.float64).reshape(
        (nl,) + tuple(reversed(p.nb))) for v in range(p.nvar)])
    P = oracle.amr_fill(p.config(), rlo, rhi, U)
    F, C = composite_globals(p, rlo, rhi, U)
    g = [p.ng if d < p.ndim else 0 for d in range(3)]
    r = [2 if d < p.ndim else 1 for d in range(3)]
    N = [p.nblk[d] * p.nb[d] for d in range(3)]
    checked = 0
    for q, (lev, b) in enumerate(leaves):
        A = F if lev else C
        NL = [N[d] * (r[d] if lev else 1) for d in range(3)]
        for d in range(p.ndim):
            tr = [e for e in range(p.ndim) if e != d]  # transverse dimensions
            for side in (0, 1):
                for depth in range(g[d]):
                    loc_d = -1 - depth if side == 0 else p.nb[d] + depth
                    for t2 in range(p.nb[tr[1]] if len(tr) > 1 else 1):
                        for t1 in range(p.nb[tr[0]] if len(tr) > 0 else 1):
                            loc = [0, 0, 0]
                            loc[d] = loc_d
                            if len(tr) > 0:
                                loc[tr[0]] = t1
                            if len(tr) > 1:
                                loc[tr[1]] = t2
                            gc = [b[e] * p.nb[e] + loc[e] for e in range(3)]
                            gm, flip = mapped(gc[d], NL[d], p.bc[d][0], p.bc[d][1])
                            gc[d] = gm
                            want = A[:, gc[2], gc[1], gc[0]].copy()
                            if flip:
                                want[1 + d] = -want[1 + d]
                            got = P[:, q, loc[2] + g[2], loc[1] + g[1], loc[0] + g[0]]
                            assert np.array_equal(got, want), (q, lev, b, d, side, loc)
                            checked += 1
        # interior copied
        inner = P[:, q, g[2]:g[2] + p.nb[2], g[1]:g[1] + p.nb[1], g[0]:g[0] + p.nb[0]]
        assert np.array_equal(inner, U[:, q])
    nface = sum(2 * g[d] * int(np.prod([p.nb[e] for e in range(p.ndim) if e != d])) for d in range(p.ndim))
    assert checked == nface * nl


def test_empty_box_is_the_uniform_coarse_scheme():
    p = si.Problem("e", 2, (8, 8, 1), (3, 2, 1), 2, 1, 1, 2, 0.4, bc=((0, 0), (1, 2), (1, 1)))
    W = si.amr_primitive(p, (0, 0, 0), (0, 0, 0), "random", seed=3)
    U = cons(p, W)
    Ua, dta = oracle.amr_step(p.config(), (0, 0, 0), (0, 0, 0), U)
    Uu, dtu = oracle.step(p.config(), U)
    assert dta == dtu and np.array_equal(Ua, Uu)


@pytest.mark.parametrize("ndim", [1, 2, 3])
def test_full_box_is_the_uniform_fine_scheme(ndim):
    nb = {1: (8, 1, 1), 2: (8, 8, 1), 3: (4, 4, 4)}[ndim]
    nblk = {1: (3, 1, 1), 2: (2, 2, 1), 3: (2, 1, 2)}[ndim]
    p = si.Problem("fb", ndim, nb, nblk, 2, 1, 1, 2, [0.8, 0.4, 0.3][ndim - 1], bc=((0, 0), (1, 2), (2, 1)))
    rlo, rhi = (0, 0, 0), nblk
    W = si.amr_primitive(p, rlo, rhi, "random", seed=4)
    U = cons(p, W)
    Ua, dta = oracle.amr_step(p.config(), rlo, rhi, U)
    q = p.with_(nblk=tuple(2 * nblk[d] if d < ndim else 1 for d in range(3)))
    Uu, dtu = oracle.step(q.config(), U)
    assert dta == dtu and np.array_equal(Ua, Uu)


@pytest.mark.parametrize("ndim", [1, 2, 3])
def test_uniform_state_stays_bitwise_uniform(ndim):
    nb = {1: (8, 1, 1), 2: (8, 8, 1), 3: (4, 4, 4)}[ndim]
    nblk = {1: (4, 1, 1), 2: (4, 3, 1), 3: (3, 3, 2)}[ndim]
    p = si.Problem("u", ndim, nb, nblk, 2, 1, 1, 3 if ndim == 2 else 2, [0.8, 0.4, 0.3][ndim - 1],
                   bc=((0, 0),) * 3)
    rlo = (1, 1 if ndim > 1 else 0, 0)
    rhi = (3, 2 if ndim > 1 else 1, 1)
    U0 = cons(p, si.amr_primitive(p, rlo, rhi, "uniform", seed=5))
    U = U0
    for _ in range(3):
        U, _ = oracle.amr_step(p.config(), rlo, rhi, U)
    for v in range(p.nvar):
        assert np.all(U[v] == U[v].flat[0])


def totals(p, rlo, rhi, U):
    _, _, _, fac = si.amr_centres(p, rlo, rhi)
    vol = fac ** p.ndim  # cell volume in units of the coarse cell
    return np.einsum("vl,l->v", U.reshape(U.shape[0], U.shape[1], -1).sum(axis=-1), vol)


@pytest.mark.parametrize("ndim,recon,rk", [(1, 1, 2), (2, 1, 2), (2, 2, 3), (3, 1, 2)])
def test_conservation_and_the_correction_matters(ndim, recon, rk):
    nb = {1: (8, 1, 1), 2: (8, 8, 1), 3: (4, 4, 4)}[ndim]
    nblk = {1: (6, 1, 1), 2: (4, 4, 1), 3: (4, 3, 3)}[ndim]
    p = si.Problem("c", ndim, nb, nblk, 3 if recon == 2 else 2, recon, 1, rk, [0.8, 0.4, 0.3][ndim - 1],
                   bc=((0, 0),) * 3)
    rlo = (1, 1 if ndim > 1 else 0, 1 if ndim > 2 else 0)
    rhi = (3, 3 if ndim > 1 else 1, 2 if ndim > 2 else 1)
    U0 = cons(p, si.amr_primitive(p, rlo, rhi, "pulse"))
    T0 = totals(p, rlo, rhi, U0)
    U, Un = U0, U0
    for _ in range(8):
        U, _ = oracle.amr_step(p.config(), rlo, rhi, U)
        Un, _ = oracle.amr_step(p.config(), rlo, rhi, Un, correct=False)
    scale = np.abs(T0) + np.abs(T0).max()
    drift = np.abs(totals(p, rlo, rhi, U) - T0) / scale
    drift_nc = np.abs(totals(p, rlo, rhi, Un) - T0) / scale
    assert drift.max() < 1e-14, drift
    assert drift_nc.max() > 1e-8, drift_nc


def test_transposition_symmetry_2d():
    p = si.Problem("s", 2, (8, 8, 1), (4, 4, 1), 2, 1, 1, 2, 0.4, bc=((1, 1), (1, 1), (1, 1)))
    rlo, rhi = (1, 1, 0), (3, 3, 1)
    x, y, _, _ = si.amr_centres(p, rlo, rhi)
    W = np.zeros((4,) + x.shape)
    r2 = (x - 0.5) ** 2 + (y - 0.5) ** 2
    W[0] = 1.0
    W[3] = 1.0 + 50.0 * np.exp(-r2 / 0.005)
    U = cons(p, W)
    for _ in range(5):
        U, _ = oracle.amr_step(p.config(), rlo, rhi, U)
    F, _ = composite_globals(p, rlo, rhi, U)
    T = np.swapaxes(F, -1, -2).copy()
    T[[1, 2]] = T[[2, 1]]
    assert np.array_equal(T, F)


def test_sod_through_refined_region():
    """1-D Sod with the right half refined: plateaus and shock against the
    exact solution; the fine region lowers the error there."""
    p = si.Problem("sod", 1, (8, 1, 1), (16, 1, 1), 2, 1, 1, 2, 0.8, bc=((1, 1),) * 3)
    rlo, rhi = (8, 0, 0), (16, 1, 1)
    U0 = cons(p, si.amr_primitive(p, rlo, rhi, "sod_x"))
    U, t, n = oracle.amr_run(p.config(), rlo, rhi, U0, t_end=0.2)
    assert abs(t - 0.2) < 1e-12
    x, _, _, _ = si.amr_centres(p, rlo, rhi)
    W = oracle.cons_to_prim(1, 1.4, U.reshape(3, -1))
    xs = x.reshape(-1)
    WL, WR = (1.0, 0.0, 1.0), (0.125, 0.0, 0.1)
    ex = er.sample(WL, WR, (xs - 0.5) / 0.2)
    fine = xs > 0.5
    err_f = np.mean(np.abs(W[0][fine] - ex[0][fine]))
    # the same problem without refinement, on the same right half
    Uc, _, _ = oracle.run(p.config(), cons(p, si.amr_primitive(p, (0, 0, 0), (0, 0, 0), "sod_x")), t_end=0.2)
    Wc = oracle.cons_to_prim(1, 1.4, Uc.reshape(3, -1))
    xc = (np.arange(128) + 0.5) / 128
    exc = er.sample(WL, WR, (xc - 0.5) / 0.2)
    err_c = np.mean(np.abs(Wc[0][xc > 0.5] - exc[0][xc > 0.5]))
    assert err_f < 0.75 * err_c, (err_f, err_c)
    head, tail, contact, shock = er.wave_positions(WL, WR, 0.2)
    ps, us = er.star_state(WL, WR)
    sel = (xs > contact + 0.03) & (xs < shock - 0.03)
    assert abs(W[2][sel].mean() - ps) < 0.01 * ps


def test_amr_config_validation():
    p = si.Problem("v", 2, (7, 8, 1), (3, 3, 1), 2, 1, 1, 2, 0.4)
    with pytest.raises(oracle.OracleError):   # nb must be even with a refined box
        oracle.amr_leaves(p.config(), (1, 1, 0), (2, 2, 1))
    q = p.with_(nb=(8, 8, 1))
    with pytest.raises(oracle.OracleError):   # box outside the block grid
        oracle.amr_leaves(q.config(), (1, 1, 0), (4, 2, 1))
