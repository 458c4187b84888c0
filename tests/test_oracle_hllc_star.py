"""HLLC star-region pin (calcFlux, Alg. 8; reading R5/R6, Toro 2009 §10.4).

Inside the fan (S_L < 0 < S_R) the HLLC flux is F*_K = F_K + S_K (U*_K - U_K)
for the side K that S* selects, and the star states are built so that F*_K is
the physical flux of a state moving at S* under the common star pressure
p* = p_K + rho_K (S_K - u_K)(S* - u_K) (the Rankine-Hugoniot conditions across
the K wave, Toro eqs. 10.26-10.36).  From the returned flux alone:

  mass      F0 = rho* S*
  momentum  F1 = rho* S*^2 + p*           -> S* = (F1 - p_K + q_K u_K)/(F0 + q_K)
  energy    F_E = S* (E*_K + p*)          with E*_K = E_K + (F_E - F_K,E)/S_K
  transv.   F_t = F0 v_t

(q_K = rho_K (S_K - u_K)).  The energy line does not appear in the oracle's
closed form of U*_K; a dropped or misplaced term there fails it.
"""
import numpy as np
import pytest

import oracle

GAMMA = 1.4


def phys(W):
    r, un = W[0], W[1]
    vt = W[2:-1]
    p = W[-1]
    E = p / (GAMMA - 1) + 0.5 * r * (un * un + float(np.sum(vt * vt)))
    U = np.concatenate([[r, r * un], r * vt, [E]])
    F = np.concatenate([[r * un, r * un * un + p], r * un * vt, [un * (E + p)]])
    return U, F


@pytest.mark.parametrize("nv", [3, 4, 5])
def test_hllc_star_flux_is_physical_flux_of_star_state(nv):
    g = np.random.Generator(np.random.PCG64(21 + nv))
    checked = 0
    for _ in range(4000):
        wl = np.concatenate([[g.uniform(0.2, 2.0)], g.uniform(-1.0, 1.0, nv - 2), [g.uniform(0.1, 3.0)]])
        wr = np.concatenate([[g.uniform(0.2, 2.0)], g.uniform(-1.0, 1.0, nv - 2), [g.uniform(0.1, 3.0)]])
        cl, cr = np.sqrt(GAMMA * wl[-1] / wl[0]), np.sqrt(GAMMA * wr[-1] / wr[0])
        sl, sr = min(wl[1] - cl, wr[1] - cr), max(wl[1] + cl, wr[1] + cr)
        if not (sl < -1e-3 and sr > 1e-3):
            continue
        F = oracle.riemann(1, GAMMA, wl, wr)
        ok_sides = []
        for W, S in ((wl, sl), (wr, sr)):
            U, FK = phys(W)
            q = W[0] * (S - W[1])
            sstar = (F[1] - W[-1] + q * W[1]) / (F[0] + q)
            pstar = W[-1] + q * (sstar - W[1])
            Estar = U[-1] + (F[-1] - FK[-1]) / S
            e_ok = abs(F[-1] - sstar * (Estar + pstar)) <= 1e-11 * (1 + abs(F[-1]))
            t_ok = all(abs(F[2 + m] - F[0] * W[2 + m]) <= 1e-12 * (1 + abs(F[2 + m])) for m in range(nv - 3))
            # the mass flux is rho* S* with rho* = rho_K (S_K - u_K)/(S_K - S*)
            m_ok = abs(F[0] - W[0] * (S - W[1]) / (S - sstar) * sstar) <= 1e-11 * (1 + abs(F[0]))
            ok_sides.append(e_ok and t_ok and m_ok)
        # exactly the side selected by S* satisfies its relations (the other
        # generally does not); at least one must
        assert any(ok_sides), (wl, wr, F)
        checked += 1
    assert checked > 1000
