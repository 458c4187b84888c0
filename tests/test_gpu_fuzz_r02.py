"""Seeded random configurations for the round-2 paths, through the C ABI
against the oracle (R15): the shockDet hybrid solver in every KB1 shape, the
HBM-tile telescoping step (1-3-D, any block shape), and the two-level
refinement with a random refined box, on one rank and on virtual ranks
(bitwise equal to one rank).  One PCG64 stream per case: fixed, reproducible."""
import numpy as np
import pytest

import oracle
import spark_inputs as si

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def draw(i, *, hybrid=False, even=False, ngmin=1):
    g = np.random.Generator(np.random.PCG64(5000 + i))
    ndim = int(g.integers(1, 4))
    recon = int(g.integers(1, 5)) if hybrid else int(g.integers(0, 5))
    ngk = 3 if recon in (2, 4) else (2 if recon in (1, 3) else 1)
    ng = max(ngk, ngmin) + int(g.integers(0, 2))
    nb, nblk, bc = [1, 1, 1], [1, 1, 1], [(1, 1)] * 3
    for d in range(ndim):
        if ndim >= 2 and d < 2 and g.random() < 0.3:
            nb[d] = 16
        else:
            nb[d] = int(g.integers(ng, 13 if ndim < 3 else 9))
        if even and nb[d] % 2:
            nb[d] += 1
        nblk[d] = int(g.integers(1, 4))
        bc[d] = (0, 0) if g.random() < 0.3 else (int(g.integers(1, 3)), int(g.integers(1, 3)))
    if nb[0] * nb[1] > 256:
        nb[1] = 256 // nb[0]
        if even and nb[1] % 2:
            nb[1] -= 1
    cfl = {1: 0.8, 2: 0.4, 3: 0.3}[ndim]
    riemann = 2 if hybrid else int(g.integers(0, 3 if recon else 2))
    return si.Problem(f"f{i}", ndim, tuple(nb), tuple(nblk), ng, recon, riemann, int(g.integers(2, 4)), cfl,
                      bc=tuple(bc), shock_thresh=float(g.uniform(0.2, 1.0)) if riemann == 2 else 0.0), g


def ids(c):
    p = c[0] if isinstance(c, tuple) else c
    return f"{p.name}-{p.ndim}d-nb{'x'.join(map(str, p.nb[:p.ndim]))}-r{p.recon}s{p.riemann}k{p.rk_stages}"


@pytest.fixture(scope="module")
def sp():
    from paper_2401_03378_b200 import spark

    spark.lib()
    return spark


def cons(p, W):
    nv = W.shape[0]
    return oracle.prim_to_cons(p.ndim, p.gamma, W.reshape(nv, -1)).reshape(W.shape)


def assert_parity(g, o, rel=1e-12, absf=1e-15, what=""):
    for v in range(o.shape[0]):
        scale = np.max(np.abs(o[v]))
        err = np.abs(g[v] - o[v])
        bad = err > rel * np.abs(o[v]) + absf * scale
        assert not bad.any(), f"{what} var {v}: {bad.sum()} cells, max err {err.max():.3e}"


def start_state(p, seed, fn):
    """Blocky random data where the oracle can step it, plain random otherwise
    (HLL / the hybrid under WENO5 cannot always step the x100 pressure jumps)."""
    for blocky in (True, False):
        U0 = cons(p, si.random_state(p, seed, blocky=blocky))
        try:
            return U0, fn(U0)
        except oracle.OracleError:
            continue
    pytest.skip("the oracle itself cannot step this random state")


HYB = [draw(i, hybrid=True)[0] for i in range(40)]


@pytest.mark.parametrize("p", HYB, ids=ids)
def test_fuzz_hybrid_steps(sp, p):
    def ref(U):
        Uo = U
        dts = []
        for _ in range(2):
            Uo, do = oracle.step(p.config(), Uo)
            dts.append(do)
        return Uo, dts
    U0, (Uo, dts) = start_state(p, 71, ref)
    s = sp.Spark(p.config())
    s.set_state(U0)
    for do in dts:
        dg = s.step(sync=True)
        assert abs(dg - do) <= 1e-13 * do
    assert_parity(s.get_state().cpu().numpy(), Uo, what=p.name)
    s.close()


TEL = [c for c in (draw(100 + i)[0] for i in range(40))
       if all(c.nb[d] * c.nblk[d] >= c.rk_stages * (3 if c.recon in (2, 4) else (2 if c.recon in (1, 3) else 1))
              for d in range(c.ndim))]


@pytest.mark.parametrize("p", TEL, ids=ids)
def test_fuzz_tile_telescoping(sp, p):
    U0, (Ut, dto) = start_state(p, 72, lambda U: oracle.step_telescoping(p.config(), U))
    s = sp.Spark(p.config())
    s.set_state(U0)
    s.enable_tiles()
    dg = s.step_telescoping(sync=True)
    assert abs(dg - dto) <= 1e-13 * dto
    assert_parity(s.get_state().cpu().numpy(), Ut, what=p.name + " tiles")
    s.close()


def draw_amr(i):
    p, g = draw(200 + i, even=True, ngmin=2)
    p = p.with_(riemann=min(p.riemann, 1) if p.recon == 0 else p.riemann)
    rlo, rhi = [0, 0, 0], [1, 1, 1]
    for d in range(p.ndim):
        a = int(g.integers(0, p.nblk[d]))
        b = int(g.integers(a, p.nblk[d] + 1))
        rlo[d], rhi[d] = a, b
    return p, tuple(rlo), tuple(rhi), int(g.integers(1, 4))


def draw_amr16(i):
    """16^3 leaves (the fused leaf kernel's shape) with random boxes, boundaries,
    face-centric scheme and rank count."""
    g = np.random.Generator(np.random.PCG64(7000 + i))
    nblk = tuple(int(g.integers(2, 4)) for _ in range(3))
    bc = tuple((0, 0) if g.random() < 0.35 else (int(g.integers(1, 3)), int(g.integers(1, 3))) for _ in range(3))
    recon = int(g.choice([0, 1, 3]))
    riemann = int(g.integers(0, 3 if recon else 2))
    p = si.Problem(f"a16_{i}", 3, (16, 16, 16), nblk, 2, recon, riemann, int(g.integers(2, 4)), 0.3, bc=bc,
                   shock_thresh=float(g.uniform(0.2, 1.0)) if riemann == 2 else 0.0)
    rlo, rhi = [0, 0, 0], [1, 1, 1]
    for d in range(3):  # a non-empty box: the coarse-fine faces are the point
        a = int(g.integers(0, nblk[d]))
        rlo[d], rhi[d] = a, int(g.integers(a + 1, nblk[d] + 1))
    return p, tuple(rlo), tuple(rhi), int(g.integers(1, 4))


AMR = [draw_amr(i) for i in range(40)] + [draw_amr16(i) for i in range(8)]


@pytest.mark.parametrize("case", AMR, ids=ids)
def test_fuzz_amr(sp, case):
    p, rlo, rhi, nranks = case

    def ref(U):
        Uo, do = oracle.amr_step(p.config(), rlo, rhi, U)
        return Uo, do
    nl = sum(oracle.amr_leaves(p.config(), rlo, rhi))
    W = si.amr_primitive(p, rlo, rhi, "random", seed=73)
    U0 = oracle.prim_to_cons(p.ndim, p.gamma, W.reshape(p.nvar, nl, -1)).reshape(W.shape)
    try:
        Uo, do = ref(U0)
    except oracle.OracleError:
        pytest.skip("the oracle itself cannot step this random state")
    a = sp.Amr(p.config(), rlo, rhi)
    a.set_state(U0)
    dg = a.step(sync=True)
    assert abs(dg - do) <= 1e-13 * do
    assert_parity(a.get_state(), Uo, what=p.name + " amr")
    if nranks > 1 and nl >= nranks:
        grp = sp.AmrGroup(p.config(), rlo, rhi, nranks)
        for (first, count), m in zip(grp.leaves, grp.ranks):
            m.set_state(np.ascontiguousarray(U0[:, first:first + count]))
        assert grp.step(sync=True) == dg
        ref1 = a.get_state()
        for (first, count), m in zip(grp.leaves, grp.ranks):
            assert np.array_equal(m.get_state(), ref1[:, first:first + count])
        grp.close()
    a.close()
