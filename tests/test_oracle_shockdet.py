"""Pins for shockDet (Alg. 7 block init) and its
consumer, the hybrid Riemann solver (reading R21).

Reading R21: cell i is a shock cell along direction d when the flow converges
across it by more than 1e-6 of the sound speed, u_d(i+1) - u_d(i-1) < -1e-6 c
(a dead band for the exact ties and last-bit noise of symmetric states), and
the pressure jump across it exceeds a
threshold, |p(i+1) - p(i-1)| > thresh * min(p(i-1), p(i+1)); a face is a
shock face when either adjacent cell is one; calcFlux then takes HLL at shock
faces and HLLC elsewhere (the usual cure of HLLC's shock instabilities).  The
sensor reads only the face's own PLM stencil (cells i-1..i+2), so it needs no
edge or corner guard cells and is identical across block and rank faces.

What fixes it beyond the definition: an exact Riemann solution (Toro 2009
Test 1) has exactly one shock; a uniform state and an advected density wave
have none; an infinite threshold reduces the hybrid to HLLC bit for bit.
"""
import numpy as np
import pytest

import oracle
import spark_inputs as si
from tests import exact_riemann as er

THR = 0.5


def cons(p, W):
    return oracle.prim_to_cons(p.ndim, p.gamma, W)


def test_sensor_cases():
    f = oracle.shock_face
    assert not f([0, 0, 0, 0], [1, 1, 1, 1], THR)                # uniform
    assert not f([1, 0.5, 0, -0.5], [1, 1.01, 1.02, 1.03], THR)   # compression, weak p jump
    assert not f([-1, 0, 1, 2], [1, 3, 9, 27], THR)               # expansion, strong p jump
    assert f([1, 0.5, 0, 0], [1, 1, 3, 3], THR)                   # compression + jump at cell i
    assert f([0, 1, 0, 0], [1, 1, 1, 3], THR)                     # ... at cell i+1 only
    # exact velocity ties, and compressions below 1e-6 of the sound speed
    # (c = sqrt(1.4 * 9) here), are not shocks whatever the pressure jump
    c = np.sqrt(1.4 * 9.0)
    assert not f([0.3, 0.3, 0.3, 0.3], [1, 1, 9, 9], THR)
    assert not f([0, 0, -0.9e-6 * c, 0], [1, 1, 9, 9], THR)
    assert f([0, 0, -1.1e-6 * c, 0], [1, 1, 9, 9], THR)
    # the band scales with the sound speed: a denser gas has a smaller c
    assert f([0, 0, -0.9e-6 * c, 0], [1, 1, 9, 9], THR, rho=[1, 1, 4, 4])
    # strict inequality at the threshold: p jump exactly thresh * min
    assert not f([1, 1, 0, 0], [2, 2, 3, 3], THR)
    assert f([1, 1, 0, 0], [2, 2, 3.0000001, 3], THR)
    # mirror symmetry: reversing the stencil and the normal velocity
    g = np.random.Generator(np.random.PCG64(3))
    for _ in range(2000):
        u = g.normal(size=4)
        p = g.uniform(0.1, 2.0, 4)
        r = g.uniform(0.1, 2.0, 4)
        assert f(u, p, THR, rho=r) == f(-u[::-1], p[::-1], THR, rho=r[::-1])


def _sod(N, riemann, thr=THR, t_end=0.2):
    p = si.PRESETS["c1_sod1d"].with_(nb=(8, 1, 1), nblk=(N // 8, 1, 1), riemann=riemann, shock_thresh=thr)
    U, t, n = oracle.run(p.config(), cons(p, si.initial_primitive(p)), t_end=t_end)
    return p, si.to_global(p, oracle.cons_to_prim(1, 1.4, U))[:, 0, 0, :], n


def _flags(W, thr=THR):
    N = W.shape[1]
    return np.array([i for i in range(1, N - 2)
                     if oracle.shock_face(W[1, i - 1:i + 3], W[2, i - 1:i + 3], thr, rho=W[0, i - 1:i + 3])])


@pytest.mark.parametrize("N", [256, 512])
def test_sod_flags_only_the_shock(N):
    """At t = 0.2 the flagged faces sit within 3 dx of the exact shock
    position and nowhere near the contact or the rarefaction."""
    WL, WR = (1.0, 0.0, 1.0), (0.125, 0.0, 0.1)
    head, tail, contact, shock = er.wave_positions(WL, WR, 0.2)
    _, W, _ = _sod(N, si.RIEMANN_HYBRID)
    h = 1.0 / N
    xf = (_flags(W) + 1) * h  # face i+1/2 between cells i and i+1
    assert len(xf) >= 1
    assert np.all(np.abs(xf - shock) < 3 * h), (xf, shock)


def test_hybrid_differs_from_hllc_only_through_shock_faces():
    """The hybrid solution still matches the exact Sod plateaus and shock
    position, and differs from HLLC (the shock faces took HLL)."""
    WL, WR = (1.0, 0.0, 1.0), (0.125, 0.0, 0.1)
    _, Wh, nh = _sod(256, si.RIEMANN_HYBRID)
    _, Wc, nc = _sod(256, si.RIEMANN_HLLC)
    assert not np.array_equal(Wh, Wc)
    x = (np.arange(256) + 0.5) / 256
    ex = er.sample(WL, WR, (x - 0.5) / 0.2)
    assert np.mean(np.abs(Wh[0] - ex[0])) < 0.01
    errs = []
    for N in (128, 256, 512):
        _, W, _ = _sod(N, si.RIEMANN_HYBRID)
        xs = (np.arange(N) + 0.5) / N
        errs.append(np.mean(np.abs(W[0] - er.sample(WL, WR, (xs - 0.5) / 0.2)[0])))
    assert errs[1] < 0.8 * errs[0] and errs[2] < 0.8 * errs[1], errs


def test_no_shock_faces_means_hllc_bitwise():
    """Advected density wave (u = 1, p = 1: a pure contact) and a uniform
    state: no face is ever a shock face, so the hybrid equals HLLC bit for bit;
    an infinite threshold does the same on 2-D Sedov (strong shocks)."""
    p = si.Problem("dw", 1, (16, 1, 1), (8, 1, 1), 2, 1, si.RIEMANN_HYBRID, 2, 0.8, bc=((0, 0),) * 3,
                   shock_thresh=THR)
    x = (np.arange(128) + 0.5) / 128
    W = np.stack([1 + 0.2 * np.sin(2 * np.pi * x), np.ones_like(x), np.ones_like(x)])[:, None, None, :]
    U0 = cons(p, si.from_global(p, W))
    Uh, _, _ = oracle.run(p.config(), U0, max_steps=40)
    Uc, _, _ = oracle.run(p.with_(riemann=1).config(), U0, max_steps=40)
    assert np.array_equal(Uh, Uc)
    q = si.Problem("u3", 3, (4, 4, 4), (2, 2, 2), 2, 1, si.RIEMANN_HYBRID, 2, 0.3, bc=((0, 0),) * 3,
                   shock_thresh=THR)
    U0 = cons(q, si.uniform_state(q, 5))
    assert np.array_equal(oracle.run(q.config(), U0, max_steps=3)[0],
                          oracle.run(q.with_(riemann=1).config(), U0, max_steps=3)[0])
    s = si.PRESETS["c3_sedov2d"].with_(nblk=(4, 4, 1), riemann=si.RIEMANN_HYBRID, shock_thresh=1e300)
    U0 = cons(s, si.initial_primitive(s))
    assert np.array_equal(oracle.run(s.config(), U0, max_steps=4)[0],
                          oracle.run(s.with_(riemann=1).config(), U0, max_steps=4)[0])


@pytest.mark.parametrize("ndim", [2, 3])
def test_sedov_hybrid_symmetry_and_flags(ndim):
    """Sedov with the hybrid solver: x<->y transposition stays bitwise, and the
    blast's shock faces are flagged (the hybrid differs from HLLC)."""
    if ndim == 2:
        p = si.PRESETS["c3_sedov2d"].with_(nblk=(4, 4, 1), riemann=si.RIEMANN_HYBRID, shock_thresh=THR)
    else:
        p = si.PRESETS["c4_sedov3d_plm"].with_(nb=(8, 8, 8), nblk=(2, 2, 2), riemann=si.RIEMANN_HYBRID,
                                               shock_thresh=THR)
    U0 = cons(p, si.initial_primitive(p))
    U, _, _ = oracle.run(p.config(), U0, max_steps=6)
    G = si.to_global(p, U)
    T = np.swapaxes(G, -1, -2).copy()
    T[[1, 2]] = T[[2, 1]]
    assert np.array_equal(T, G)
    Uc, _, _ = oracle.run(p.with_(riemann=1).config(), U0, max_steps=6)
    assert not np.array_equal(U, Uc)


def test_hybrid_config_validation():
    p = si.PRESETS["c1_sod1d"].with_(riemann=si.RIEMANN_HYBRID)
    with pytest.raises(oracle.OracleError):   # threshold must be > 0
        oracle.run(p.config(), cons(p, si.initial_primitive(p)), max_steps=1)
    q = p.with_(recon=0, ng=1, shock_thresh=THR)  # the sensor needs a 2-cell stencil
    with pytest.raises(oracle.OracleError):
        oracle.run(q.config(), cons(q, si.initial_primitive(q)), max_steps=1)
