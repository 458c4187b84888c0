"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Tolerance (reading R15, BASELINE.json north_star "max relative error
1e-12"): per conserved variable v, |gpu - oracle| <= 1e-12 |oracle| +
1e-15 max|oracle_v| for single stages / steps, absolute floor 1e-14 max|oracle_v|
for runs of hundreds of steps (a pure relative metric is undefined where a
momentum is ~0).  Block/guard-cell indexing is bit-exact.
"""
import numpy as np
import pytest

import oracle
import spark_inputs as si

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def sp():
    from paper_2401_03378_b200 import spark

    spark.lib()
    return spark


def cons(p, W):
    return oracle.prim_to_cons(p.ndim, p.gamma, W)


def assert_parity(g, o, rel=1e-12, absf=1e-15, what=""):
    g = np.asarray(g)
    o = np.asarray(o)
    assert g.shape == o.shape, (g.shape, o.shape)
    for v in range(o.shape[0]):
        scale = np.max(np.abs(o[v]))
        err = np.abs(g[v] - o[v])
        lim = rel * np.abs(o[v]) + absf * scale
        bad = err > lim
        assert not bad.any(), (f"{what} var {v}: {bad.sum()} cells over tolerance, max err {err.max():.3e}, "
                               f"max rel {np.max(err / (np.abs(o[v]) + 1e-300)):.3e}")


def make(sp, p, U=None, W=None):
    s = sp.Spark(p.config())
    if U is not None:
        s.set_state(np.ascontiguousarray(U))
    elif W is not None:
        s.set_primitive(np.ascontiguousarray(W))
    return s


def state(s):
    return s.get_state().cpu().numpy()


# ------------------------------------------------------------------ cases
STAGE_CASES = [
    si.Problem("1d_plm_hllc", 1, (8, 1, 1), (5, 1, 1), 2, 1, 1, 2, 0.8, bc=((1, 1),) * 3),
    si.Problem("1d_weno_hll_refl", 1, (7, 1, 1), (3, 1, 1), 3, 2, 0, 3, 0.8, bc=((2, 1), (1, 1), (1, 1))),
    si.Problem("1d_first_hllc_per", 1, (4, 1, 1), (3, 1, 1), 1, 0, 1, 2, 0.8, bc=((0, 0),) * 3),
    si.Problem("2d_plm_hllc", 2, (16, 16, 1), (3, 2, 1), 2, 1, 1, 2, 0.4, bc=((1, 2), (0, 0), (1, 1))),
    si.Problem("2d_weno_hllc_odd", 2, (12, 10, 1), (3, 3, 1), 3, 2, 1, 3, 0.4, bc=((2, 2), (0, 0), (1, 1))),
    si.Problem("2d_plm_hll_ng3", 2, (8, 6, 1), (2, 5, 1), 3, 1, 0, 2, 0.4, bc=((0, 0), (2, 1), (1, 1))),
    si.Problem("3d_plm_hllc", 3, (16, 16, 16), (2, 2, 2), 2, 1, 1, 2, 0.3, bc=((1, 1), (0, 0), (2, 1))),
    si.Problem("3d_weno_hllc", 3, (16, 16, 16), (2, 1, 2), 3, 2, 1, 3, 0.3, bc=((0, 0), (1, 2), (1, 1))),
    si.Problem("3d_weno_hll_odd", 3, (6, 5, 7), (3, 2, 2), 3, 2, 0, 3, 0.3, bc=((2, 1), (0, 0), (0, 0))),
    si.Problem("3d_first_hllc", 3, (4, 4, 4), (2, 3, 2), 1, 0, 1, 2, 0.3, bc=((1, 1),) * 3),
    # production 16^3 kernels: face-centric first order (halo on warps 6-7) with
    # reflecting y faces, PLM with reflecting x/y faces and RK3 (halo sign flips
    # in the in-S2 halo conversion), and 16x16x8 blocks (runtime-extent kernel)
    si.Problem("3d_first16_hll_refl", 3, (16, 16, 16), (2, 1, 2), 1, 0, 0, 2, 0.3, bc=((1, 1), (2, 2), (0, 0))),
    si.Problem("3d_plm16_hll_reflxy", 3, (16, 16, 16), (1, 2, 2), 2, 1, 0, 3, 0.3, bc=((2, 2), (2, 1), (1, 1))),
    si.Problem("3d_plm_16x16x8", 3, (16, 16, 8), (2, 2, 2), 2, 1, 1, 2, 0.3, bc=((0, 0), (1, 1), (2, 1))),
    # face-centric PLM-MC (one-barrier plane loop in 3-D): HLL with reflecting
    # faces, HLLC RK3, and the 2-D plane kernel
    si.Problem("3d_mc16_hll_refl", 3, (16, 16, 16), (2, 2, 1), 2, 3, 0, 2, 0.3, bc=((2, 2), (1, 2), (2, 2))),
    si.Problem("3d_mc16_hllc_rk3", 3, (16, 16, 16), (1, 2, 2), 2, 3, 1, 3, 0.3, bc=((0, 0), (2, 1), (1, 1))),
    si.Problem("2d_mc16_hllc_refl", 2, (16, 16, 1), (3, 2, 1), 2, 3, 1, 2, 0.4, bc=((2, 1), (2, 2), (1, 1))),
]


@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("ndim", [1, 2, 3])
def test_device_riemann(sp, kind, ndim):
    """The device Riemann solver (calcFlux of KB1) vs the oracle, face by face,
    sub- and supersonic states, every normal direction (regression for an nvcc
    miscompile of the HLLC K-side selects)."""
    g = np.random.Generator(np.random.PCG64(40 + ndim + 10 * kind))
    nv, n = ndim + 2, 4000
    W = np.empty((2, n, nv))
    W[:, :, 0] = g.uniform(0.05, 5.0, (2, n))
    W[:, :, 1:nv - 1] = g.uniform(-1, 1, (2, n, nv - 2)) * np.where(np.arange(n) % 4 == 0, 4.0, 1.0)[None, :, None]
    W[:, :, nv - 1] = g.uniform(0.01, 5.0, (2, n))
    for d in range(ndim):
        f = sp.selftest_riemann(kind, ndim, d, 1.4, W[0], W[1])
        order = [0, 1 + d] + [1 + e for e in range(ndim) if e != d] + [nv - 1]
        for q in range(0, n, 7):
            fo = np.empty(nv)
            fo[order] = oracle.riemann(kind, 1.4, W[0, q, order], W[1, q, order])
            assert np.allclose(f[q], fo, rtol=1e-12, atol=1e-13 * (np.abs(fo).max() + 1)), (q, d, f[q], fo)


@pytest.mark.parametrize("p", STAGE_CASES, ids=lambda p: p.name)
def test_prim_to_cons(sp, p):
    W = si.random_state(p, 3)
    s = make(sp, p, W=W)
    assert_parity(state(s), cons(p, W), rel=1e-15, absf=1e-16, what="prim->cons")


@pytest.mark.parametrize("p", STAGE_CASES, ids=lambda p: p.name)
def test_guard_fill_bitexact(sp, p):
    """KB2 materialised padded blocks == oracle fill_guardcells, bit for bit
    (index-encoded state: every block / cell / variable mix-up is visible)."""
    U = si.index_encoded(p)
    s = make(sp, p, U=U)
    P = s.fill_guardcells(padded=True).cpu().numpy()
    assert np.array_equal(P, oracle.fill_guardcells(p.config(), U))


@pytest.mark.parametrize("blocky", [False, True])
@pytest.mark.parametrize("p", STAGE_CASES, ids=lambda p: p.name)
def test_single_stage(sp, p, blocky):
    """One fused stage U_out = a U_n + b (U_prev + dt L(U_prev)) vs oracle_stage."""
    Up = cons(p, si.random_state(p, 10, blocky=blocky))
    Un = cons(p, si.random_state(p, 11, blocky=blocky))
    dt = 0.2 * p.cfl * oracle.dt_raw(p.config(), Up)
    s = make(sp, p, U=Up)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    for a, b in [(0.0, 1.0), (0.75, 0.25), (1.0 / 3.0, 2.0 / 3.0)]:
        g = s.stage_apply(dev(Up), dev(Un), a, b, dt).cpu().numpy()
        o = oracle.stage(p.config(), Up, Un, a, b, dt)
        assert_parity(g, o, what=f"stage a={a}")


@pytest.mark.parametrize("p", STAGE_CASES, ids=lambda p: p.name)
def test_step_cfl_dt(sp, p):
    """Two full SSP-RK steps with the CFL dt (computed and min-reduced on GPU)."""
    U0 = cons(p, si.random_state(p, 12, blocky=True))
    s = make(sp, p, U=U0)
    Uo = U0
    for _ in range(2):
        dtg = s.step(sync=True)
        Uo, dto = oracle.step(p.config(), Uo)
        assert abs(dtg - dto) <= 1e-13 * dto
    assert_parity(state(s), Uo, what="2 steps")


def test_cfl_min_exact(sp):
    p = STAGE_CASES[7]
    U = cons(p, si.random_state(p, 5))
    s = make(sp, p, U=U)
    o = oracle.dt_raw(p.config(), U)
    assert abs(s.cfl_min() - o) <= 4e-16 * o


# ------------------------------------------------------------ full configs
@pytest.mark.parametrize("name", ["c1_sod1d", "c2a_sod2d", "c2b_sod2d"])
def test_full_run(sp, name):
    """configs[0], configs[1]: run to t_end on GPU and in the oracle."""
    p = si.PRESETS[name]
    U0 = cons(p, si.initial_primitive(p))
    Uo, to, no = oracle.run(p.config(), U0, t_end=p.t_end)
    s = make(sp, p, U=U0)
    n = s.advance(10_000, t_end=p.t_end, check_every=32)
    t, steps, _ = s.time()
    assert steps == no and abs(t - to) <= 1e-14
    assert n == no
    # hundreds of steps: zero-valued momenta carry ulp noise of the O(1) flux
    # terms (reading R15: absolute floor 1e-14 max|o_v| for multi-step runs)
    assert_parity(state(s), Uo, absf=1e-14, what=name)


def test_c3_sedov2d_three_steps(sp):
    """configs[2] at full size (1024^2, WENO5 + HLLC, SSP-RK3): 3 steps."""
    p = si.PRESETS["c3_sedov2d"]
    U0 = cons(p, si.initial_primitive(p))
    Uo, _, _ = oracle.run(p.config(), U0, max_steps=3)
    s = make(sp, p, U=U0)
    for _ in range(3):
        s.step()
    assert_parity(state(s), Uo, what="c3")


def _oracle_subbox_step(p, G, lo, hi, margin, dt):
    """Oracle step on a sub-box [lo, hi) of the global conserved state G
    ([v][Z][Y][X]) extended by `margin` cells (exact there: the result of a
    step depends only on cells within S*NG); returns the [lo, hi) region."""
    N = [p.nblk[d] * p.nb[d] for d in range(3)]
    dxs = [(p.hi[d] - p.lo[d]) / N[d] for d in range(3)]
    elo, ehi, bc, sub_lo, sub_hi = [], [], [], [], []
    for d in range(3):
        if d >= p.ndim:
            elo.append(0), ehi.append(1), bc.append((1, 1)), sub_lo.append(0.0), sub_hi.append(1.0)
            continue
        a, b = max(0, lo[d] - margin), min(N[d], hi[d] + margin)
        elo.append(a)
        ehi.append(b)
        bc.append((p.bc[d][0] if a == 0 else si.BC_OUTFLOW, p.bc[d][1] if b == N[d] else si.BC_OUTFLOW))
        sub_lo.append(p.lo[d] + a * dxs[d])
        sub_hi.append(p.lo[d] + b * dxs[d])
    sub = G[:, elo[2]:ehi[2], elo[1]:ehi[1], elo[0]:ehi[0]]
    n = [ehi[d] - elo[d] for d in range(3)]
    q = p.with_(nb=tuple(n), nblk=(1, 1, 1), bc=tuple(bc), lo=tuple(sub_lo), hi=tuple(sub_hi))
    U, _ = oracle.step(q.config(), si.from_global(q, np.ascontiguousarray(sub)), dt_fixed=dt)
    R = si.to_global(q, U)
    return R[:, lo[2] - elo[2]:hi[2] - elo[2], lo[1] - elo[1]:hi[1] - elo[1], lo[0] - elo[0]:hi[0] - elo[0]]


C4_VARIANTS = {  # the bench's --recon / --riemann lines: same grid, other kernel instantiations
    "c4_sedov3d_plm": {}, "c4_sedov3d_weno": {},
    "c4_sedov3d_plm+mc": {"recon": 3}, "c4_sedov3d_plm+first": {"recon": 0},
    "c4_sedov3d_plm+hybrid": {"riemann": si.RIEMANN_HYBRID, "shock_thresh": 0.5},
}


@pytest.mark.parametrize("name", sorted(C4_VARIANTS))
def test_c4_sedov3d_sampled(sp, name):
    """configs[3] at full size (256^3 in 16^3 blocks) in the launch configuration
    bench.py times: one GPU step with the CFL dt; sampled sub-boxes (the blast
    centre, a domain corner, a block-boundary slab) recomputed by the oracle."""
    p = si.PRESETS[name.split("+")[0]].with_(**C4_VARIANTS[name])
    U0 = cons(p, si.initial_primitive(p))
    dt_o = oracle.dt(p.config(), U0)
    s = make(sp, p, U=U0)
    dt_g = s.step(sync=True)
    assert abs(dt_g - dt_o) <= 1e-13 * dt_o
    G = si.to_global(p, state(s))
    G0 = si.to_global(p, U0)
    margin = p.rk_stages * (3 if p.recon == 2 else 2)
    for lo, hi in [((120, 120, 120), (136, 136, 136)), ((0, 0, 0), (12, 12, 12)),
                   ((240, 8, 100), (256, 40, 116))]:
        o = _oracle_subbox_step(p, G0, lo, hi, margin, dt_g)
        g = G[:, lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]]
        assert_parity(g, o, what=f"{name} {lo}")


# ------------------------------------------------------------- invariants
@pytest.mark.parametrize("p", [STAGE_CASES[4].with_(bc=((0, 0),) * 3), STAGE_CASES[7].with_(bc=((0, 0),) * 3)],
                         ids=["2d", "3d"])
def test_uniform_state_bitwise(sp, p):
    """Every face flux is computed at one code site, so F+ - F- == 0 exactly."""
    U0 = cons(p, si.uniform_state(p, 4))
    s = make(sp, p, U=U0)
    for _ in range(3):
        s.step()
    U = state(s)
    for v in range(p.nvar):
        assert np.all(U[v] == U[v].flat[0])


def test_conservation_gpu(sp):
    p = si.PRESETS["c2b_sod2d"]
    U0 = cons(p, si.initial_primitive(p))
    s = make(sp, p, U=U0)
    for _ in range(40):
        s.step()
    U = state(s)
    for v in range(p.nvar):
        scale = np.abs(U0[v]).sum() + np.abs(U[v]).sum()
        assert abs(U[v].sum() - U0[v].sum()) <= 1e-13 * scale


def test_transposition_symmetry_gpu(sp):
    p = si.PRESETS["c3_sedov2d"].with_(nblk=(4, 4, 1))
    s = make(sp, p, U=cons(p, si.initial_primitive(p)))
    for _ in range(4):
        s.step()
    G = si.to_global(p, state(s))
    T = np.swapaxes(G, -1, -2).copy()
    T[[1, 2]] = T[[2, 1]]
    assert_parity(T, G, what="transpose")


# ------------------------------------------------------- virtual ranks
@pytest.mark.parametrize("nranks", [2, 4, 8])
@pytest.mark.parametrize("p", [
    si.Problem("v3", 3, (8, 8, 8), (2, 2, 2), 3, 2, 1, 3, 0.3, bc=((0, 0), (1, 2), (1, 1))),
    si.Problem("v3p", 3, (8, 8, 8), (4, 2, 2), 2, 1, 1, 2, 0.3, bc=((0, 0),) * 3),
    si.Problem("v2", 2, (16, 16, 1), (4, 4, 1), 2, 1, 1, 2, 0.4, bc=((0, 0), (1, 1), (1, 1))),
], ids=lambda p: p.name)
def test_virtual_ranks_bitwise(sp, p, nranks):
    """The N-rank result (halo exchange between sub-boxes) equals the 1-rank
    result bit for bit, and the global dt minimum is identical."""
    cfg = p.config()
    if not sp.check_config(cfg, nranks):
        pytest.skip("not divisible")
    U0 = cons(p, si.random_state(p, 8, blocky=True))
    one = make(sp, p, U=U0)
    grp = sp.LocalGroup(cfg, nranks)
    G0 = si.to_global(p, U0)
    for r, s in enumerate(grp.ranks):
        lo, n = sp.rank_box(cfg, r, nranks)
        sub = G0[:, lo[2] * p.nb[2]:(lo[2] + n[2]) * p.nb[2], lo[1] * p.nb[1]:(lo[1] + n[1]) * p.nb[1],
                 lo[0] * p.nb[0]:(lo[0] + n[0]) * p.nb[0]]
        q = p.with_(nblk=tuple(n))
        s.set_state(si.from_global(q, np.ascontiguousarray(sub)))
    for _ in range(3):
        d1 = one.step(sync=True)
        dn = grp.step(sync=True)
        assert d1 == dn
    G1 = si.to_global(p, state(one))
    for r, s in enumerate(grp.ranks):
        lo, n = sp.rank_box(cfg, r, nranks)
        q = p.with_(nblk=tuple(n))
        Gr = si.to_global(q, state(s))
        ref = G1[:, lo[2] * p.nb[2]:(lo[2] + n[2]) * p.nb[2], lo[1] * p.nb[1]:(lo[1] + n[1]) * p.nb[1],
                 lo[0] * p.nb[0]:(lo[0] + n[0]) * p.nb[0]]
        assert np.array_equal(Gr, ref)
    # face guards of the materialised padded blocks also agree with the 1-rank fill
    grp.close()


# ------------------------------------------------------ control / errors
def test_nonphysical_rollback(sp):
    p = STAGE_CASES[3]
    U = cons(p, si.random_state(p, 1))
    s = make(sp, p, U=U)
    U2 = U.copy()
    U2[3, 2, 0, 5, 5] = -50.0  # negative total energy -> p < 0
    s.set_state(U2)
    # the LOADED state is non-physical (flagged as step 0 by set_state's CFL
    # pass): steps are frozen and reported, nothing can be rolled back
    with pytest.raises(sp.NonPhysicalError, match="step 0.*not rolled back"):
        s.step(dt=1e-4, sync=True)
    t, n, _ = s.time()
    assert t == 0.0 and n == 0
    with pytest.raises(sp.NonPhysicalError):
        state(s)
    # (a step that itself fails is rolled back: tests/test_gpu_errors.py)
    # a physical state steps normally afterwards
    s.set_state(U)
    s.step(dt=1e-4, sync=True)
    # without a sync point the error surfaces at the next synchronising call
    s.set_state(U2)
    s.step(dt=1e-4)
    with pytest.raises(sp.NonPhysicalError):
        state(s)


def test_t_end_stop_and_copy_through(sp):
    p = si.PRESETS["c1_sod1d"]
    U0 = cons(p, si.initial_primitive(p))
    s = make(sp, p, U=U0)
    s.advance(10_000, t_end=0.05, check_every=4)
    t, n, _ = s.time()
    assert abs(t - 0.05) < 1e-15
    U1 = state(s)
    s.step(t_end=0.05)
    s.step(t_end=0.05)
    t2, n2, dt2 = s.time()
    assert t2 == t and n2 == n and dt2 == 0.0
    assert np.array_equal(state(s), U1)


def test_profile_counts(sp):
    p = STAGE_CASES[6]
    s = make(sp, p, U=cons(p, si.random_state(p, 2)))
    s.profile(True)
    for _ in range(3):
        s.step()
    ms, n, tot = s.profile_read()
    assert n == 3 * p.rk_stages and ms > 0.0 and tot == 3 * (p.rk_stages + 1)


def test_errors(sp):
    p = STAGE_CASES[0]
    s = sp.Spark(p.config())
    with pytest.raises(sp.SparkError):
        s.step()
    with pytest.raises(sp.SparkError):
        sp.Spark(p.with_(ng=1).config())


@pytest.mark.parametrize("p", [
    si.Problem("s3", 3, (16, 16, 16), (2, 2, 2), 3, 2, 1, 3, 0.3, bc=((0, 0), (0, 0), (0, 0))),
    si.Problem("s3m", 3, (8, 8, 8), (2, 3, 2), 2, 1, 1, 2, 0.3, bc=((0, 0), (1, 2), (0, 0))),
    si.Problem("s2", 2, (16, 16, 1), (3, 2, 1), 2, 1, 1, 2, 0.4, bc=((0, 0), (0, 0), (1, 1))),
], ids=lambda p: p.name)
def test_nccl_self_exchange_bitwise(sp, p):
    """One rank with an NCCL communicator: periodic faces go through pack ->
    ncclSend/ncclRecv (to self, the message order of exchange_nccl) -> KB1 slab
    reads, plus the dt all-reduce.  Must equal the local-wrap path bit for bit."""
    U0 = cons(p, si.random_state(p, 17, blocky=True))
    plain = make(sp, p, U=U0)
    viaccl = sp.Spark(p.config(), nccl_id=sp.nccl_unique_id())
    viaccl.set_state(U0)
    for _ in range(3):
        assert plain.step(sync=True) == viaccl.step(sync=True)
    assert np.array_equal(state(plain), state(viaccl))
    # padded blocks: interior and face guards identical; edges/corners that lie
    # across two exchanged faces are not exchanged (star stencil) and read NaN
    Pp = plain.fill_guardcells().cpu().numpy()
    Pn = viaccl.fill_guardcells().cpu().numpy()
    g = [p.ng if d < p.ndim else 0 for d in range(3)]
    k, j, i = np.meshgrid(*[np.arange(p.nb[d] + 2 * g[d]) for d in (2, 1, 0)], indexing="ij")
    outside = sum(((c < g[d]) | (c >= g[d] + p.nb[d])).astype(int) for c, d in ((i, 0), (j, 1), (k, 2)))
    face = outside <= 1
    assert np.array_equal(Pp[:, :, face], Pn[:, :, face])
    assert not np.isnan(Pn[:, :, face]).any()
    viaccl.close()


@pytest.mark.parametrize("variant", [0, 1, 2, 3])
@pytest.mark.parametrize("n", [1, 1000, 1_000_003])
def test_axpy_variants(sp, variant, n):
    """NEXT N4: the paper's AXPY thread mappings (alg:axpy-*) give exactly
    a*x + y (separate multiply and add, as numpy computes it)."""
    g = np.random.Generator(np.random.PCG64(n + variant))
    x, y = g.normal(size=n), g.normal(size=n)
    a = 0.7310585786300049
    yd = torch.from_numpy(y.copy()).cuda()
    sp.axpy(variant, a, torch.from_numpy(x).cuda(), yd)
    assert np.array_equal(yd.cpu().numpy(), a * x + y)
