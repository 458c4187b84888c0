"""CPU checks of the C-ABI library: it builds, loads, exports every symbol that
include/spark.h declares, and its host-only logic (config validation, process
grid, sub-boxes, halo plans) is consistent.  No compute calls (no GPU here)."""
import os
import re

import pytest

import spark_inputs as si
from paper_2401_03378_b200 import build as spark_build
from paper_2401_03378_b200 import spark

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    spark_build.build()


def header_functions():
    src = open(os.path.join(ROOT, "include", "spark.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(spark_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_exports():
    assert header_functions() == sorted(spark.EXPORTS)


def test_library_exports_every_symbol():
    L = spark.lib()
    for name in header_functions():
        assert hasattr(L, name), name
    assert L.spark_abi_version() == 3


def test_sm100a_code_in_library():
    """The .so carries sm_100a SASS (cross-compiled here)."""
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", spark.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("name", sorted(si.PRESETS))
def test_presets_valid(name):
    assert spark.check_config(si.PRESETS[name].config(), 1)


def test_config_rejections():
    base = si.PRESETS["c4_sedov3d_plm"]
    assert not spark.check_config(base.with_(ng=1).config())
    assert not spark.check_config(base.with_(recon=2, ng=2).config())
    assert not spark.check_config(base.with_(rk_stages=1).config())
    assert not spark.check_config(base.with_(nb=(32, 16, 16)).config())          # 512 threads
    assert not spark.check_config(base.with_(gamma=1.0).config())
    assert not spark.check_config(base.with_(bc=((0, 1), (1, 1), (1, 1))).config())  # half periodic
    assert not spark.check_config(base.config(), 3)                               # 16 % 3 != 0
    assert spark.check_config(base.config(), 8)
    # NEXT N2: MC (ng 2), WENO-Z (ng 3), gravity finite and zero along unused dims
    assert spark.check_config(base.with_(recon=3).config())
    assert not spark.check_config(base.with_(recon=4).config())
    assert spark.check_config(base.with_(recon=4, ng=3).config())
    assert not spark.check_config(base.with_(recon=5, ng=3).config())
    assert spark.check_config(base.with_(grav=(0.1, -2.0, 3.0)).config())
    assert not spark.check_config(base.with_(grav=(float("nan"), 0.0, 0.0)).config())
    c2 = si.PRESETS["c2b_sod2d"]
    assert spark.check_config(c2.with_(grav=(0.0, -1.0, 0.0)).config())
    assert not spark.check_config(c2.with_(grav=(0.0, 0.0, -1.0)).config())


@pytest.mark.parametrize("nranks", [1, 2, 4, 8])
@pytest.mark.parametrize("name", ["c4_sedov3d_plm", "c3_sedov2d", "c2b_sod2d", "c1_sod1d"])
def test_rank_boxes_partition_blocks(name, nranks):
    cfg = si.PRESETS[name].config()
    if not spark.check_config(cfg, nranks):
        pytest.skip("not divisible")
    seen = {}
    for r in range(nranks):
        lo, n = spark.rank_box(cfg, r, nranks)
        for bz in range(lo[2], lo[2] + n[2]):
            for by in range(lo[1], lo[1] + n[1]):
                for bx in range(lo[0], lo[0] + n[0]):
                    assert (bx, by, bz) not in seen
                    seen[(bx, by, bz)] = r
    nb = cfg["nblk"]
    assert len(seen) == nb[0] * nb[1] * nb[2]


@pytest.mark.parametrize("nranks", [2, 4, 8])
@pytest.mark.parametrize("bc", [si.BC_OUTFLOW, si.BC_PERIODIC])
def test_halo_plans_are_symmetric(nranks, bc):
    """Face (d, s) of rank r names peer q  <=>  face (d, 1-s) of q names r, and
    the slab sizes agree; peers are exactly the face-adjacent sub-boxes."""
    cfg = si.PRESETS["c4_sedov3d_weno"].with_(bc=((bc, bc),) * 3).config()
    pg = spark.rank_grid(cfg, nranks)
    assert pg[0] * pg[1] * pg[2] == nranks
    plans = [spark.halo_plan(cfg, r, nranks) for r in range(nranks)]
    for r in range(nranks):
        lo, n = spark.rank_box(cfg, r, nranks)
        for f in plans[r]:
            d, s, q = f["dim"], f["side"], f["peer"]
            edge = (lo[d] == 0) if s == 0 else (lo[d] + n[d] == cfg["nblk"][d])
            if q < 0:
                assert edge and (bc != si.BC_PERIODIC or pg[d] == 1)
                continue
            other = [g for g in plans[q] if g["dim"] == d and g["side"] == 1 - s][0]
            assert other["peer"] == r and other["cells"] == f["cells"]
            qlo, qn = spark.rank_box(cfg, q, nranks)
            want = (lo[d] + n[d]) % cfg["nblk"][d] if s else (lo[d] - qn[d]) % cfg["nblk"][d]
            assert qlo[d] == want
            cells = cfg["ng"]
            for e in range(3):
                if e != d:
                    cells *= n[e] * cfg["nb"][e]
            assert f["cells"] == cells


def test_required_bytes_scale():
    cfg = si.PRESETS["c4_sedov3d_plm"].config()
    b1 = spark.required_bytes(cfg, 0, 1)
    state = 5 * 256 ** 3 * 8
    assert 3 * state <= b1 < 3 * state + 4096
    b8 = spark.required_bytes(cfg, 0, 8)
    assert b8 < b1 / 7


def test_sub_box_cell_limit():
    """configs[4] (1024^3) fits one rank; 2048^3 needs >= 4 ranks (2^31 cells per sub-box)."""
    c5 = si.PRESETS["c5_sedov3d_plm"]
    assert spark.required_bytes(c5.config(), 0, 1) >= 3 * 5 * 1024 ** 3 * 8
    big = c5.with_(nblk=(128, 128, 128)).config()
    with pytest.raises(spark.SparkError):
        spark.required_bytes(big, 0, 1)
    with pytest.raises(spark.SparkError):
        spark.required_bytes(big, 0, 2)
    spark.required_bytes(big, 0, 8)


def test_product_path_does_not_touch_oracle():
    """The binding and the CUDA sources never import, link or name the oracle."""
    pkg = os.path.join(ROOT, "paper_2401_03378_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "spark_oracle" not in txt and "libspark_oracle" not in txt, f


def test_amr_host_plan_matches_oracle_leaf_count():
    """NEXT N3 host logic (no GPU): the leaf enumeration of spark_amr_leaves
    agrees with the oracle's and with spark_inputs' layout helper; invalid
    refinements are refused; the arena size grows with the fine leaves."""
    from paper_2401_03378_b200 import spark

    import oracle
    import spark_inputs as si

    p = si.Problem("a", 3, (8, 8, 8), (4, 3, 2), 2, 1, 1, 2, 0.3, bc=((0, 0), (1, 1), (2, 2)))
    for rlo, rhi in [((1, 1, 0), (3, 2, 2)), ((0, 0, 0), (0, 0, 0)), ((0, 0, 0), (4, 3, 2))]:
        assert spark.amr_leaves(p.config(), rlo, rhi) == oracle.amr_leaves(p.config(), rlo, rhi)
        assert sum(spark.amr_leaves(p.config(), rlo, rhi)) == len(si.amr_leaf_blocks(p, rlo, rhi))
    with pytest.raises(spark.SparkError):
        spark.amr_leaves(p.with_(nb=(7, 8, 8)).config(), (1, 1, 0), (3, 2, 2))
    with pytest.raises(spark.SparkError):
        spark.amr_leaves(p.config(), (1, 1, 0), (5, 2, 2))
    import ctypes

    def nbytes(rlo, rhi):
        n = ctypes.c_size_t()
        c, r = spark.to_cconfig(p.config()), spark._refine(rlo, rhi)
        assert spark.lib().spark_amr_required_bytes(ctypes.byref(c), ctypes.byref(r), ctypes.byref(n)) == 0
        return n.value

    assert nbytes((1, 1, 0), (3, 2, 2)) > nbytes((0, 0, 0), (0, 0, 0))


def test_amr_rank_partition_covers_the_leaves():
    """spark_amr_rank_leaves: contiguous, disjoint ranges covering every leaf."""
    from paper_2401_03378_b200 import spark

    import spark_inputs as si

    p = si.Problem("a", 2, (8, 8, 1), (4, 4, 1), 2, 1, 1, 2, 0.4)
    rlo, rhi = (1, 1, 0), (3, 3, 1)
    n = sum(spark.amr_leaves(p.config(), rlo, rhi))
    for nranks in (1, 2, 3, 7):
        ranges = [spark.amr_rank_leaves(p.config(), rlo, rhi, r, nranks) for r in range(nranks)]
        assert ranges[0][0] == 0 and sum(c for _, c in ranges) == n
        assert all(ranges[r][0] + ranges[r][1] == ranges[r + 1][0] for r in range(nranks - 1))
