"""Exact Riemann solver for the 1-D Euler equations with an ideal gas.

Independent textbook pin for the oracle (not used by the oracle or the CUDA
path): E. F. Toro, Riemann Solvers and Numerical Methods for Fluid Dynamics,
3rd ed., Ch. 4 — pressure function f_K(p) (Eqs. 4.6-4.8), Newton iteration
for p* (Sec. 4.3.2), star velocity (Eq. 4.9) and the sampling procedure of
Sec. 4.5 (shock / rarefaction fans on both sides).
"""
from __future__ import annotations

import math

import numpy as np


def _fk(p, rho, pk, g):
    a = math.sqrt(g * pk / rho)
    if p > pk:  # shock
        A = 2.0 / ((g + 1.0) * rho)
        B = (g - 1.0) / (g + 1.0) * pk
        f = (p - pk) * math.sqrt(A / (p + B))
        df = math.sqrt(A / (B + p)) * (1.0 - (p - pk) / (2.0 * (B + p)))
    else:  # rarefaction
        f = 2.0 * a / (g - 1.0) * ((p / pk) ** ((g - 1.0) / (2.0 * g)) - 1.0)
        df = 1.0 / (rho * a) * (p / pk) ** (-(g + 1.0) / (2.0 * g))
    return f, df


def star_state(WL, WR, g=1.4, tol=1e-15):
    """Return (p*, u*) for primitive states (rho, u, p)."""
    rl, ul, pl = WL
    rr, ur, pr = WR
    # two-rarefaction initial guess (Toro Eq. 4.46)
    al, ar = math.sqrt(g * pl / rl), math.sqrt(g * pr / rr)
    z = (g - 1.0) / (2.0 * g)
    p = ((al + ar - 0.5 * (g - 1.0) * (ur - ul)) / (al / pl ** z + ar / pr ** z)) ** (1.0 / z)
    for _ in range(100):
        fl, dfl = _fk(p, rl, pl, g)
        fr, dfr = _fk(p, rr, pr, g)
        pn = p - (fl + fr + ur - ul) / (dfl + dfr)
        pn = max(pn, 1e-14)
        if abs(pn - p) / (0.5 * (pn + p)) < tol:
            p = pn
            break
        p = pn
    fl, _ = _fk(p, rl, pl, g)
    fr, _ = _fk(p, rr, pr, g)
    u = 0.5 * (ul + ur) + 0.5 * (fr - fl)
    return p, u


def star_densities(WL, WR, p, g=1.4):
    rl, _, pl = WL
    rr, _, pr = WR
    gm = (g - 1.0) / (g + 1.0)

    def rho_star(r, pk):
        if p > pk:
            return r * (p / pk + gm) / (gm * p / pk + 1.0)
        return r * (p / pk) ** (1.0 / g)

    return rho_star(rl, pl), rho_star(rr, pr)


def sample(WL, WR, xi, g=1.4):
    """Primitive solution (rho, u, p) at similarity coordinate xi = (x - x0)/t."""
    rl, ul, pl = WL
    rr, ur, pr = WR
    ps, us = star_state(WL, WR, g)
    rsl, rsr = star_densities(WL, WR, ps, g)
    al, ar = math.sqrt(g * pl / rl), math.sqrt(g * pr / rr)
    out = np.empty((3, len(xi)))
    for n, s in enumerate(xi):
        if s <= us:  # left of contact
            if ps > pl:  # left shock
                sl = ul - al * math.sqrt((g + 1) / (2 * g) * ps / pl + (g - 1) / (2 * g))
                out[:, n] = (rl, ul, pl) if s <= sl else (rsl, us, ps)
            else:  # left rarefaction
                shl = ul - al
                asl = al * (ps / pl) ** ((g - 1) / (2 * g))
                stl = us - asl
                if s <= shl:
                    out[:, n] = (rl, ul, pl)
                elif s >= stl:
                    out[:, n] = (rsl, us, ps)
                else:
                    c = 2 / (g + 1) + (g - 1) / ((g + 1) * al) * (ul - s)
                    out[:, n] = (rl * c ** (2 / (g - 1)), 2 / (g + 1) * (al + (g - 1) / 2 * ul + s),
                                 pl * c ** (2 * g / (g - 1)))
        else:  # right of contact
            if ps > pr:  # right shock
                sr = ur + ar * math.sqrt((g + 1) / (2 * g) * ps / pr + (g - 1) / (2 * g))
                out[:, n] = (rr, ur, pr) if s >= sr else (rsr, us, ps)
            else:  # right rarefaction
                shr = ur + ar
                asr = ar * (ps / pr) ** ((g - 1) / (2 * g))
                str_ = us + asr
                if s >= shr:
                    out[:, n] = (rr, ur, pr)
                elif s <= str_:
                    out[:, n] = (rsr, us, ps)
                else:
                    c = 2 / (g + 1) - (g - 1) / ((g + 1) * ar) * (ur - s)
                    out[:, n] = (rr * c ** (2 / (g - 1)), 2 / (g + 1) * (-ar + (g - 1) / 2 * ur + s),
                                 pr * c ** (2 * g / (g - 1)))
    return out


def wave_positions(WL, WR, t, x0=0.5, g=1.4):
    """Head / tail of the left rarefaction, contact and right shock (Sod-type)."""
    rl, ul, pl = WL
    rr, ur, pr = WR
    ps, us = star_state(WL, WR, g)
    al, ar = math.sqrt(g * pl / rl), math.sqrt(g * pr / rr)
    asl = al * (ps / pl) ** ((g - 1) / (2 * g))
    sr = ur + ar * math.sqrt((g + 1) / (2 * g) * ps / pr + (g - 1) / (2 * g))
    return (x0 + (ul - al) * t, x0 + (us - asl) * t, x0 + us * t, x0 + sr * t)
