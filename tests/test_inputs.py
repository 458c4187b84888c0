"""The seeded input generators (spark_inputs): layout round trips and the
device-side Sedov builder being bit-identical to the host one (run here with
torch on the CPU device)."""
import numpy as np
import pytest

import spark_inputs as si

torch = pytest.importorskip("torch")


@pytest.mark.parametrize("name", ["c3_sedov2d", "c4_sedov3d_plm"])
def test_sedov_device_equals_host(name):
    p = si.PRESETS[name].with_(nblk=(4, 4, 4) if si.PRESETS[name].ndim == 3 else (8, 8, 1))
    ref = si.sedov(p)
    got = si.sedov_device(p, device="cpu").numpy()
    assert np.array_equal(got, ref)
    cells, p_dep, _ = si.sedov_deposit(p)
    assert len(cells) == si._sedov_ndep(p, 3.5 * (p.hi[0] - p.lo[0]) / (p.nblk[0] * p.nb[0]))
    assert (ref[p.ndim + 1] == p_dep).sum() == len(cells)


def test_sedov_device_sub_boxes():
    p = si.PRESETS["c4_sedov3d_plm"].with_(nblk=(4, 4, 2))
    n = [p.nblk[d] * p.nb[d] for d in range(3)]
    # the four 32x32x32 boxes around the centre hold the whole deposit
    for lo in [(0, 0, 0), (32, 0, 0), (0, 32, 0), (32, 32, 0)]:
        box = (lo, (32, 32, n[2]))
        assert np.array_equal(si.sedov_device(p, box=box, device="cpu").numpy(), si.sedov(p, box=box))


def test_layout_round_trip():
    p = si.Problem("r", 3, (4, 3, 2), (2, 3, 2), 1, 1, 1, 2, 0.3)
    G = np.random.default_rng(1).random((5, 4, 9, 8))
    assert np.array_equal(si.to_global(p, si.from_global(p, G)), G)
