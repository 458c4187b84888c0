"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the method (no EOS, reconstruction, Riemann
solver, divergence or RK).  It only produces:

* problem descriptions (``PRESETS``: the five BASELINE.json configs),
* primitive initial states ``W[v][b][k][j][i]`` (rho, u_1..u_ndim, p) — each side
  converts them to conserved variables with its own EOS,
* index permutations between the canonical block layout and a global
  ``[v][z][y][x]`` array (pure reshapes),
* seeded random states (numpy ``Generator(PCG64(seed))``).

Input recipes:
  Sod    (rho,u,p) = (1,0,1) for x < 0.5, (0.125,0,0.1) otherwise  [Toro 2009 Test 1]
  Sedov  rho = 1, u = 0, p_amb = 1e-5; E_blast = 1 deposited uniformly as
         internal energy in the cells whose centres lie within r0 = 3.5 dx of
         the domain centre
  random rho, p ~ U[0.5, 1.5], u_d ~ U[-0.5, 0.5]; "blocky" adds jumps of
         rho x10 and p x100 every 5-13 cells along x (limiter branches)
"""
from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np

BC_PERIODIC, BC_OUTFLOW, BC_REFLECT = 0, 1, 2
RECON_FIRST, RECON_PLM, RECON_WENO5, RECON_PLM_MC, RECON_WENO5Z = 0, 1, 2, 3, 4
RIEMANN_HLL, RIEMANN_HLLC, RIEMANN_HYBRID = 0, 1, 2


@dataclass(frozen=True)
class Problem:
    """A problem description: the fields of spark_config plus the IC name."""

    name: str
    ndim: int
    nb: tuple
    nblk: tuple
    ng: int
    recon: int
    riemann: int
    rk_stages: int
    cfl: float
    bc: tuple = ((BC_OUTFLOW, BC_OUTFLOW),) * 3
    lo: tuple = (0.0, 0.0, 0.0)
    hi: tuple = (1.0, 1.0, 1.0)
    gamma: float = 1.4
    ic: str = "sod"
    t_end: float = 0.0
    grav: tuple = (0.0, 0.0, 0.0)
    shock_thresh: float = 0.0

    def config(self) -> dict:
        return dict(ndim=self.ndim, nb=tuple(self.nb), nblk=tuple(self.nblk), ng=self.ng, lo=tuple(self.lo),
                    hi=tuple(self.hi), bc=tuple(tuple(x) for x in self.bc), recon=self.recon,
                    riemann=self.riemann, rk_stages=self.rk_stages, gamma=self.gamma, cfl=self.cfl,
                    grav=tuple(self.grav), shock_thresh=self.shock_thresh)

    def with_(self, **kw) -> "Problem":
        return replace(self, **kw)

    @property
    def nvar(self):
        return self.ndim + 2

    @property
    def ncells(self):
        return int(np.prod(self.nb)) * int(np.prod(self.nblk))


_OUT = ((BC_OUTFLOW, BC_OUTFLOW),) * 3
_PER = ((BC_PERIODIC, BC_PERIODIC),) * 3

# The five BASELINE.json configs.
PRESETS = {
    # configs[0]: 1-D Sod, 256 cells = 32 blocks x 8, RK2 + PLM + HLLC, t = 0.2
    "c1_sod1d": Problem("c1_sod1d", 1, (8, 1, 1), (32, 1, 1), 2, RECON_PLM, RIEMANN_HLLC, 2, 0.8,
                        bc=_OUT, ic="sod_x", t_end=0.2),
    # configs[1] reading C2a: x-aligned Sod, outflow in x, periodic in y
    "c2a_sod2d": Problem("c2a_sod2d", 2, (16, 16, 1), (8, 8, 1), 2, RECON_PLM, RIEMANN_HLLC, 2, 0.4,
                         bc=((BC_OUTFLOW, BC_OUTFLOW), (BC_PERIODIC, BC_PERIODIC), (BC_OUTFLOW, BC_OUTFLOW)),
                         ic="sod_x", t_end=0.2),
    # configs[1] reading C2b: fully periodic square Sod (conservation)
    "c2b_sod2d": Problem("c2b_sod2d", 2, (16, 16, 1), (8, 8, 1), 2, RECON_PLM, RIEMANN_HLLC, 2, 0.4,
                         bc=_PER, ic="sod_square", t_end=0.1),
    # configs[2]: 2-D Sedov 1024^2 in 16^2 blocks, RK3 + WENO5 + HLLC
    "c3_sedov2d": Problem("c3_sedov2d", 2, (16, 16, 1), (64, 64, 1), 3, RECON_WENO5, RIEMANN_HLLC, 3, 0.4,
                          bc=_OUT, ic="sedov", t_end=0.05),
    # configs[3]: 3-D Sedov 256^3 in 16^3 blocks (PLM/RK2 and WENO5/RK3 variants)
    "c4_sedov3d_plm": Problem("c4_sedov3d_plm", 3, (16, 16, 16), (16, 16, 16), 2, RECON_PLM, RIEMANN_HLLC, 2,
                              0.3, bc=_OUT, ic="sedov", t_end=0.05),
    "c4_sedov3d_weno": Problem("c4_sedov3d_weno", 3, (16, 16, 16), (16, 16, 16), 3, RECON_WENO5, RIEMANN_HLLC,
                               3, 0.3, bc=_OUT, ic="sedov", t_end=0.05),
    # configs[4]: 3-D Sedov 1024^3 in 16^3 blocks over 2/4/8 GPUs
    "c5_sedov3d_plm": Problem("c5_sedov3d_plm", 3, (16, 16, 16), (64, 64, 64), 2, RECON_PLM, RIEMANN_HLLC, 2,
                              0.3, bc=_OUT, ic="sedov", t_end=0.05),
    "c5_sedov3d_weno": Problem("c5_sedov3d_weno", 3, (16, 16, 16), (64, 64, 64), 3, RECON_WENO5, RIEMANN_HLLC,
                               3, 0.3, bc=_OUT, ic="sedov", t_end=0.05),
}


# ----------------------------------------------------------------- layouts
def to_global(p: Problem, A: np.ndarray) -> np.ndarray:
    """Canonical [v][b][k][j][i] (b lexicographic over blocks) -> [v][Z][Y][X]."""
    nv = A.shape[0]
    nbx, nby, nbz = p.nblk
    ni, nj, nk = p.nb
    A = A.reshape(nv, nbz, nby, nbx, nk, nj, ni)
    return A.transpose(0, 1, 4, 2, 5, 3, 6).reshape(nv, nbz * nk, nby * nj, nbx * ni)


def from_global(p: Problem, G: np.ndarray) -> np.ndarray:
    """[v][Z][Y][X] -> canonical [v][b][k][j][i]."""
    nv = G.shape[0]
    nbx, nby, nbz = p.nblk
    ni, nj, nk = p.nb
    G = G.reshape(nv, nbz, nk, nby, nj, nbx, ni)
    return np.ascontiguousarray(G.transpose(0, 1, 3, 5, 2, 4, 6).reshape(nv, nbz * nby * nbx, nk, nj, ni))


def centres(p: Problem, box=None):
    """Cell-centre coordinates (x, y, z) as [Z][Y][X] arrays of the whole grid, or
    of the sub-box ``box = ((lo_x, lo_y, lo_z), (n_x, n_y, n_z))`` in cells."""
    n = [p.nblk[d] * p.nb[d] for d in range(3)]
    lo_c, n_c = box if box is not None else ((0, 0, 0), n)
    ax = []
    for d in range(3):
        h = (p.hi[d] - p.lo[d]) / n[d]
        ax.append(p.lo[d] + (np.arange(lo_c[d], lo_c[d] + n_c[d]) + 0.5) * h)
    z, y, x = np.meshgrid(ax[2], ax[1], ax[0], indexing="ij")
    return x, y, z


def _prim_global(p: Problem, rho, vel, pres, box=None) -> np.ndarray:
    shape = rho.shape
    W = np.zeros((p.nvar,) + shape, dtype=np.float64)
    W[0] = rho
    for d in range(p.ndim):
        W[1 + d] = vel[d] if vel is not None else 0.0
    W[p.ndim + 1] = pres
    if box is not None:  # canonical layout of the sub-box (its own block grid)
        q = replace(p, nblk=tuple(box[1][d] // p.nb[d] for d in range(3)))
        return from_global(q, W)
    return from_global(p, W)


# -------------------------------------------------------------- generators
def sod_x(p: Problem) -> np.ndarray:
    """Sod along x (Toro 2009, Test 1): primitive W, canonical layout."""
    x, _, _ = centres(p)
    left = x < 0.5
    rho = np.where(left, 1.0, 0.125)
    pres = np.where(left, 1.0, 0.1)
    return _prim_global(p, rho, None, pres)


def sod_square(p: Problem) -> np.ndarray:
    """Periodic square Sod: (1,0,1) inside |x-1/2|,|y-1/2| < 1/4, else (0.125,0,0.1)."""
    x, y, _ = centres(p)
    inside = (np.abs(x - 0.5) < 0.25) & (np.abs(y - 0.5) < 0.25)
    rho = np.where(inside, 1.0, 0.125)
    pres = np.where(inside, 1.0, 0.1)
    return _prim_global(p, rho, None, pres)


def sedov(p: Problem, e_blast: float = 1.0, p_amb: float = 1e-5, r0_cells: float = 3.5, box=None) -> np.ndarray:
    """Sedov blast: E_blast deposited as uniform internal energy within r0 of the centre.

    p_dep = (gamma-1) E_blast / (n_dep dV) is the IC's definition of the deposit
    (an input recipe, not the method's EOS).  ``box`` (cells) restricts the
    output to one rank's sub-box; n_dep is always counted on the whole grid."""
    x, y, z = centres(p, box)
    dxs = [(p.hi[d] - p.lo[d]) / (p.nblk[d] * p.nb[d]) for d in range(3)]
    c = [0.5 * (p.lo[d] + p.hi[d]) for d in range(3)]
    r2 = (x - c[0]) ** 2
    if p.ndim >= 2:
        r2 = r2 + (y - c[1]) ** 2
    if p.ndim >= 3:
        r2 = r2 + (z - c[2]) ** 2
    r0 = r0_cells * dxs[0]
    dep = r2 < r0 * r0
    n_dep = _sedov_ndep(p, r0) if box is not None else int(dep.sum())
    dV = float(np.prod(dxs[: p.ndim]))
    rho = np.ones_like(x)
    pres = np.full_like(x, p_amb)
    pres[dep] = (p.gamma - 1.0) * e_blast / (n_dep * dV)
    return _prim_global(p, rho, None, pres, box)


def _sedov_ndep(p: Problem, r0: float) -> int:
    """Number of deposit cells on the whole grid (only the neighbourhood of the centre)."""
    n = [p.nblk[d] * p.nb[d] for d in range(3)]
    k = int(np.ceil(r0 / ((p.hi[0] - p.lo[0]) / n[0]))) + 2
    lo = [max(0, n[d] // 2 - k) if d < p.ndim else 0 for d in range(3)]
    hi = [min(n[d], n[d] // 2 + k) if d < p.ndim else 1 for d in range(3)]
    x, y, z = centres(p, (tuple(lo), tuple(hi[d] - lo[d] for d in range(3))))
    c = [0.5 * (p.lo[d] + p.hi[d]) for d in range(3)]
    r2 = (x - c[0]) ** 2
    if p.ndim >= 2:
        r2 = r2 + (y - c[1]) ** 2
    if p.ndim >= 3:
        r2 = r2 + (z - c[2]) ** 2
    return int((r2 < r0 * r0).sum())


def sedov_deposit(p: Problem, e_blast: float = 1.0, p_amb: float = 1e-5, r0_cells: float = 3.5):
    """The Sedov IC in sparse form: (global (x, y, z) cell indices of the deposit,
    p_dep, p_amb).  Same membership test and p_dep expression as ``sedov``, so
    ``sedov_device`` is bit-identical to ``sedov`` (tests/test_inputs.py)."""
    n = [p.nblk[d] * p.nb[d] for d in range(3)]
    dxs = [(p.hi[d] - p.lo[d]) / n[d] for d in range(3)]
    r0 = r0_cells * dxs[0]
    k = int(np.ceil(r0 / dxs[0])) + 2
    lo = [max(0, n[d] // 2 - k) if d < p.ndim else 0 for d in range(3)]
    hi = [min(n[d], n[d] // 2 + k) if d < p.ndim else 1 for d in range(3)]
    x, y, z = centres(p, (tuple(lo), tuple(hi[d] - lo[d] for d in range(3))))
    c = [0.5 * (p.lo[d] + p.hi[d]) for d in range(3)]
    r2 = (x - c[0]) ** 2
    if p.ndim >= 2:
        r2 = r2 + (y - c[1]) ** 2
    if p.ndim >= 3:
        r2 = r2 + (z - c[2]) ** 2
    kz, jy, ix = np.nonzero(r2 < r0 * r0)
    cells = np.stack([ix + lo[0], jy + lo[1], kz + lo[2]], axis=1)
    dV = float(np.prod(dxs[: p.ndim]))
    p_dep = (p.gamma - 1.0) * e_blast / (len(cells) * dV)
    return cells, p_dep, p_amb


def sedov_device(p: Problem, box=None, device="cuda"):
    """``sedov(p, box)`` built directly in device memory (torch), canonical block
    layout of the sub-box: a fill plus a scatter of the ~200 deposit cells.  For
    grids whose host copy would not fit (configs[4]: 1024^3 x 5 x 8 B = 40 GiB)."""
    import torch

    n = [p.nblk[d] * p.nb[d] for d in range(3)]
    lo_c, n_c = box if box is not None else ((0, 0, 0), tuple(n))
    nbk = [n_c[d] // p.nb[d] for d in range(3)]
    nblocks = nbk[0] * nbk[1] * nbk[2]
    W = torch.zeros((p.nvar, nblocks, p.nb[2], p.nb[1], p.nb[0]), dtype=torch.float64, device=device)
    cells, p_dep, p_amb = sedov_deposit(p)
    W[0].fill_(1.0)
    W[p.ndim + 1].fill_(p_amb)
    loc = cells - np.asarray(lo_c)[None, :]
    inside = np.all((loc >= 0) & (loc < np.asarray(n_c)[None, :]), axis=1)
    loc = loc[inside]
    if len(loc):
        nb = np.asarray(p.nb)
        bq, r = loc // nb, loc % nb
        b = bq[:, 0] + nbk[0] * (bq[:, 1] + nbk[1] * bq[:, 2])
        idx = ((b * p.nb[2] + r[:, 2]) * p.nb[1] + r[:, 1]) * p.nb[0] + r[:, 0]
        W[p.ndim + 1].view(-1)[torch.from_numpy(idx).to(W.device)] = p_dep
    return W


def random_state(p: Problem, seed: int, blocky: bool = False) -> np.ndarray:
    """rho, p ~ U[0.5,1.5]; u_d ~ U[-0.5,0.5]; 'blocky' adds x-jumps (rho x10, p x100)."""
    g = np.random.Generator(np.random.PCG64(seed))
    n = [p.nblk[d] * p.nb[d] for d in range(3)]
    shape = (n[2], n[1], n[0])
    rho = g.uniform(0.5, 1.5, shape)
    vel = [g.uniform(-0.5, 0.5, shape) for _ in range(p.ndim)]
    pres = g.uniform(0.5, 1.5, shape)
    if blocky:
        edges, pos = [], 0
        while pos < n[0]:
            pos += int(g.integers(5, 14))
            edges.append(pos)
        seg = np.searchsorted(np.array(edges), np.arange(n[0]), side="right")
        hi = (seg % 2 == 1)[None, None, :]
        rho = np.where(hi, rho * 10.0, rho)
        pres = np.where(hi, pres * 100.0, pres)
    return _prim_global(p, rho, vel, pres)


def uniform_state(p: Problem, seed: int) -> np.ndarray:
    """A random constant (rho, u, p) everywhere."""
    g = np.random.Generator(np.random.PCG64(seed))
    n = [p.nblk[d] * p.nb[d] for d in range(3)]
    shape = (n[2], n[1], n[0])
    rho = np.full(shape, g.uniform(0.5, 1.5))
    vel = [np.full(shape, g.uniform(-0.5, 0.5)) for _ in range(p.ndim)]
    pres = np.full(shape, g.uniform(0.5, 1.5))
    return _prim_global(p, rho, vel, pres)


def density_wave_avg(p: Problem, t: float = 0.0, amp: float = 0.2):
    """Cell averages of rho = 1 + amp sin 2 pi (x - t), u = 1, p = 1 on [0,1] (1-D).

    Returned as primitive W whose rho is the exact cell average (u, p are
    constant, so the conserved cell averages follow linearly)."""
    n = p.nblk[0] * p.nb[0]
    h = (p.hi[0] - p.lo[0]) / n
    xl = p.lo[0] + np.arange(n) * h
    xr = xl + h
    avg = 1.0 + amp * (np.cos(2 * math.pi * (xl - t)) - np.cos(2 * math.pi * (xr - t))) / (2 * math.pi * h)
    rho = avg.reshape(1, 1, n)
    vel = [np.ones_like(rho)]
    pres = np.ones_like(rho)
    return _prim_global(p, rho, vel, pres)


def index_encoded(p: Problem) -> np.ndarray:
    """U[v][g] = v * 2**32 + g (g = global cell index x + NX*(y + NY*z)); exact in fp64.

    Used to prove guard-cell / block indexing bit-exact."""
    n = [p.nblk[d] * p.nb[d] for d in range(3)]
    g = np.arange(n[0] * n[1] * n[2], dtype=np.float64).reshape(n[2], n[1], n[0])
    G = np.stack([v * 2.0 ** 32 + g for v in range(p.nvar)])
    return from_global(p, G)


def initial_primitive(p: Problem, seed: int = 0, box=None) -> np.ndarray:
    if p.ic == "sedov":
        return sedov(p, box=box)
    assert box is None, "sub-box generation only for sedov"
    if p.ic == "sod_x":
        return sod_x(p)
    if p.ic == "sod_square":
        return sod_square(p)
    if p.ic == "random":
        return random_state(p, seed)
    if p.ic == "blocky":
        return random_state(p, seed, blocky=True)
    raise ValueError(p.ic)


# ------------------------------------------ NEXT N3: static two-level refinement
# Layout only (no method arithmetic): the leaf list of a refinement of the
# coarse blocks [rlo, rhi) by 2 — coarse blocks outside the box, then the fine
# blocks of the box, each lexicographic with x fastest — and primitive states
# evaluated at the leaves' cell centres.  Leaf states are [v][leaf][k][j][i].
def amr_leaf_blocks(p: Problem, rlo, rhi):
    """[(level, (bx, by, bz))] in leaf order (fine block coordinates are on the
    global fine block grid)."""
    has_box = all(rhi[d] > rlo[d] for d in range(3))
    out = []
    for bz in range(p.nblk[2]):
        for by in range(p.nblk[1]):
            for bx in range(p.nblk[0]):
                inside = has_box and all(rlo[d] <= b < rhi[d] for d, b in enumerate((bx, by, bz)))
                if not inside:
                    out.append((0, (bx, by, bz)))
    if has_box:
        f = [2 * (rhi[d] - rlo[d]) if d < p.ndim else 1 for d in range(3)]
        o = [2 * rlo[d] if d < p.ndim else 0 for d in range(3)]
        for bz in range(f[2]):
            for by in range(f[1]):
                for bx in range(f[0]):
                    out.append((1, (o[0] + bx, o[1] + by, o[2] + bz)))
    return out


def amr_centres(p: Problem, rlo, rhi):
    """Cell centres (x, y, z) of every leaf cell, arrays [leaf][k][j][i], and
    the cell spacing factor of each leaf (1 coarse, 1/2 fine)."""
    leaves = amr_leaf_blocks(p, rlo, rhi)
    dx = [(p.hi[d] - p.lo[d]) / (p.nblk[d] * p.nb[d]) for d in range(3)]
    X = np.zeros((3, len(leaves), p.nb[2], p.nb[1], p.nb[0]))
    fac = np.ones(len(leaves))
    for q, (lev, b) in enumerate(leaves):
        f = 0.5 if lev else 1.0
        fac[q] = f
        for d in range(3):
            h = dx[d] * (f if d < p.ndim else 1.0)
            c = p.lo[d] + (b[d] * p.nb[d] + np.arange(p.nb[d]) + 0.5) * h
            shape = [1, 1, 1]
            shape[2 - d] = p.nb[d]
            X[d, q] = c.reshape(shape)
    return X[0], X[1], X[2], fac


def amr_primitive(p: Problem, rlo, rhi, kind: str, seed: int = 0) -> np.ndarray:
    """Primitive leaf state W[v][leaf][k][j][i]:
    'random'  rho, p ~ U[0.5, 1.5], u ~ U[-0.5, 0.5] per cell (seeded);
    'uniform' one random constant state;
    'pulse'   rho = 1 + 0.5 g, p = 1 + 2 g, u_d = 0.3 (d+1)/ndim,
              g = exp(-|x - x0|^2 / 0.01), x0 = 0.4 per dim (crosses the box);
    'sod_x'   Toro Test 1 along x (x < 0.5 left state)."""
    x, y, z, _ = amr_centres(p, rlo, rhi)
    nl = x.shape[0]
    W = np.zeros((p.nvar,) + x.shape)
    g = np.random.Generator(np.random.PCG64(seed))
    if kind == "random":
        W[0] = g.uniform(0.5, 1.5, x.shape)
        for d in range(p.ndim):
            W[1 + d] = g.uniform(-0.5, 0.5, x.shape)
        W[-1] = g.uniform(0.5, 1.5, x.shape)
    elif kind == "uniform":
        W[0] = g.uniform(0.5, 1.5)
        for d in range(p.ndim):
            W[1 + d] = g.uniform(-0.5, 0.5)
        W[-1] = g.uniform(0.5, 1.5)
    elif kind == "pulse":
        r2 = (x - 0.4) ** 2 + ((y - 0.4) ** 2 if p.ndim > 1 else 0.0) + ((z - 0.4) ** 2 if p.ndim > 2 else 0.0)
        gg = np.exp(-r2 / 0.01)
        W[0] = 1.0 + 0.5 * gg
        for d in range(p.ndim):
            W[1 + d] = 0.3 * (d + 1) / p.ndim
        W[-1] = 1.0 + 2.0 * gg
    elif kind == "sod_x":
        W[0] = np.where(x < 0.5, 1.0, 0.125)
        W[-1] = np.where(x < 0.5, 1.0, 0.1)
    else:
        raise ValueError(kind)
    assert W.shape[1] == nl
    return W
