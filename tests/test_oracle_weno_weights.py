"""Dedicated pins for the WENO5-JS nonlinear weights of the oracle.

The oracle's ``oracle_weno5_edge`` (calcLims, Alg. 8; reading R3 =
Jiang & Shu 1996) writes the smoothness indicators as closed forms with the
constants 13/12 and 1/4, the weights as d_k / (eps + beta_k)^2 and the linear
weights as (0.1, 0.6, 0.3).  None of those constants is retyped here.  They are
re-derived from the definitions in exact rational arithmetic:

* candidate k is the quadratic p_k whose averages over the three cells of
  stencil k equal the data (a 3x3 linear solve);
* beta_k = sum_{l=1,2} int_cell h^(2l-1) (d^l p_k / dx^l)^2 dx
  (Jiang & Shu's definition of the indicator, integrated exactly);
* the linear weights d_k are the unique convex weights for which
  sum_k d_k p_k(x_{i+1/2}) equals the edge value of the quartic through all
  five cell averages, for every data set (a linear solve on unit data);
* alpha_k = d_k / (eps + beta_k)^p with p = 2 and eps = 1e-6 (reading R3).

A mutation of any indicator coefficient, of the exponent or of a linear weight
changes the edge value of non-smooth data far beyond round-off, so one of the
tests below fails.  ``test_mutations_are_visible`` checks that the data sets
used are discriminating in exactly that sense.
"""
from fractions import Fraction as Fr

import numpy as np
import pytest

import oracle

EPS = Fr(1, 10**6)
P = 2


def cell_avg_row(m):
    """[1, avg x, avg x^2] over the unit cell centred at m."""
    return [Fr(1), Fr(m), Fr(m * m) + Fr(1, 12)]


def solve(A, b):
    """Gauss-Jordan elimination in exact rationals."""
    n = len(A)
    M = [list(map(Fr, A[r])) + [Fr(b[r])] for r in range(n)]
    for c in range(n):
        piv = next(r for r in range(c, n) if M[r][c] != 0)
        M[c], M[piv] = M[piv], M[c]
        M[c] = [x / M[c][c] for x in M[c]]
        for r in range(n):
            if r != c and M[r][c] != 0:
                M[r] = [x - M[r][c] * y for x, y in zip(M[r], M[c])]
    return [M[r][n] for r in range(n)]


def candidate(k, W):
    """Coefficients (c0, c1, c2) of p_k for data W = W_{i-2..i+2} (cell i at 0)."""
    cells = [k - 2, k - 1, k]
    return solve([cell_avg_row(m) for m in cells], [W[m + 2] for m in cells])


def beta(c):
    """int_{-1/2}^{1/2} (p')^2 + (p'')^2 dx for p = c0 + c1 x + c2 x^2 (h = 1)."""
    c0, c1, c2 = c
    # (p')^2 = c1^2 + 4 c1 c2 x + 4 c2^2 x^2 ; int x = 0, int x^2 = 1/12
    d1 = c1 * c1 + 4 * c2 * c2 * Fr(1, 12)
    d2 = (2 * c2) ** 2
    return d1 + d2


def edge(c):
    c0, c1, c2 = c
    return c0 + c1 * Fr(1, 2) + c2 * Fr(1, 4)


def quartic_edge(W):
    """Edge value at x = 1/2 of the quartic whose 5 cell averages are W."""
    rows = []
    for m in range(-2, 3):
        # average of x^n over [m - 1/2, m + 1/2]
        rows.append([(Fr(2 * m + 1, 2) ** (n + 1) - Fr(2 * m - 1, 2) ** (n + 1)) / (n + 1) for n in range(5)])
    c = solve(rows, W)
    return sum(c[n] * Fr(1, 2) ** n for n in range(5))


def linear_weights():
    """d such that sum_k d_k edge(p_k) == quartic edge for all data: solve on the
    unit vectors (5 equations, 3 unknowns; consistent by construction)."""
    A, b = [], []
    for j in range(5):
        W = [Fr(int(j == m)) for m in range(5)]
        A.append([edge(candidate(k, W)) for k in range(3)])
        b.append(quartic_edge(W))
    d = solve(A[:3], b[:3])
    for r in range(3, 5):  # the two remaining equations hold too
        assert sum(A[r][k] * d[k] for k in range(3)) == b[r]
    return d


D = linear_weights()


def weno_js_edge(W, eps=EPS, p=P, d=None, beta_fn=beta):
    d = D if d is None else d
    cands = [candidate(k, W) for k in range(3)]
    alpha = [d[k] / (eps + beta_fn(cands[k])) ** p for k in range(3)]
    s = sum(alpha)
    return sum(alpha[k] / s * edge(cands[k]) for k in range(3)), [a / s for a in alpha]


# stencils with jumps, kinks and extrema: weights far from linear
ROUGH = [
    (0, 0, 1, 3, 2),
    (1, -2, 3, 0, 5),
    (4, 4, 1, 1, 1),
    (0, 1, 0, 1, 0),
    (Fr(1, 2), Fr(3, 4), 2, Fr(-1, 8), 7),
    (10, 9, 7, 4, 0),
    (1, 1, 1, 2, 4),
    (-3, Fr(5, 2), Fr(1, 3), 1, -1),
]


def test_linear_weights_derived():
    """The derivation reproduces the textbook optimal weights (0.1, 0.6, 0.3)
    — a check on the derivation machinery, not on the oracle."""
    assert D == [Fr(1, 10), Fr(6, 10), Fr(3, 10)]


@pytest.mark.parametrize("W", ROUGH)
def test_weno5js_edge_matches_definition(W):
    """Oracle edge value == the value built from the defining integrals."""
    W = [Fr(x) for x in W]
    ref, _ = weno_js_edge(W)
    got = oracle.weno5_edge(*[float(x) for x in W])
    scale = max(abs(float(x)) for x in W) + 1.0
    assert abs(got - float(ref)) <= 2e-15 * scale, (got, float(ref))


def test_weno5js_random_stencils_match_definition():
    g = np.random.Generator(np.random.PCG64(11))
    for _ in range(300):
        # dyadic rationals: exact both as doubles and as fractions
        W = [Fr(int(x), 64) for x in g.integers(-256, 256, 5)]
        ref, _ = weno_js_edge(W)
        got = oracle.weno5_edge(*[float(x) for x in W])
        assert abs(got - float(ref)) <= 4e-15 * (max(abs(float(x)) for x in W) + 1.0)


@pytest.mark.parametrize("jump_at", [0, 1, 2, 3])
@pytest.mark.parametrize("mirror", [False, True])
def test_weno5js_eno_at_jump(jump_at, mirror):
    """Essentially non-oscillatory at a jump: the candidates whose stencil
    crosses the jump get weights <= 1e-6 of the smooth candidate, so the edge
    value equals the smooth candidate's value up to that weight (JS, p = 2:
    alpha_smooth / alpha_cross ~ (beta_cross / eps)^2 ~ 1e12)."""
    W = [0.0 if m < jump_at + 1 else 1.0 for m in range(5)]  # jump between cells jump_at, jump_at+1
    if mirror:
        W = [1.0 - x for x in W]
    cands = [candidate(k, [Fr(x) for x in W]) for k in range(3)]
    smooth = [k for k in range(3) if len({W[m + 2] for m in (k - 2, k - 1, k)}) == 1]
    v = oracle.weno5_edge(*W)
    if smooth:
        k = smooth[0]
        assert abs(v - float(edge(cands[k]))) < 1e-10, (W, v)
    # independent of the oracle: the crossing candidates' weights are tiny
    _, w = weno_js_edge([Fr(x) for x in W])
    for k in range(3):
        if smooth and k not in smooth:
            assert w[k] < 1e-6 * w[smooth[0]]


def test_mutations_are_visible():
    """The rough stencils discriminate every plausible misreading: a wrong
    indicator constant, exponent, epsilon or linear weight moves at least one
    edge value by far more than the 2e-15 tolerance used above."""
    def beta_mut(c13, c14):
        # the textbook closed form 13/12 (2nd difference)^2 + 1/4 (1st)^2 is
        # 13/12 (2 c2)^2 + 1/4 (2 c1)^2 in the candidate's coefficients; the
        # mutant replaces its two constants
        return lambda c: c13 * (2 * c[2]) ** 2 + c14 * (2 * c[1]) ** 2

    mutants = {
        "beta 13/12 -> 1/12": dict(beta_fn=beta_mut(Fr(1, 12), Fr(1, 4))),
        "beta 1/4 -> 3/4": dict(beta_fn=beta_mut(Fr(13, 12), Fr(3, 4))),
        "exponent 2 -> 1": dict(p=1),
        "eps 1e-6 -> 1e-40": dict(eps=Fr(1, 10**40)),
        "linear weights swapped": dict(d=[Fr(3, 10), Fr(6, 10), Fr(1, 10)]),
    }
    # sanity: the unmutated closed form reproduces the integral definition
    ident = beta_mut(Fr(13, 12), Fr(1, 4))
    for W in ROUGH:
        Wf = [Fr(x) for x in W]
        for k in range(3):
            assert ident(candidate(k, Wf)) == beta(candidate(k, Wf))
    for name, kw in mutants.items():
        moved = max(abs(float(weno_js_edge([Fr(x) for x in W], **kw)[0] - weno_js_edge([Fr(x) for x in W])[0]))
                    for W in ROUGH)
        assert moved > 1e-9, name
