"""spark_step_host (end-to-end use with host buffers, copies pipelined in
chunks) gives bit for bit what set_state + step + get_state give, for any
chunk count, with aliased in/out buffers and back-to-back asynchronous calls
(each call's upload of chunk j waits for the previous call's download of j)."""
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


@pytest.mark.parametrize("p", [
    si.PRESETS["c4_sedov3d_plm"].with_(nblk=(4, 3, 2)),
    si.Problem("h2", 2, (16, 16, 1), (5, 3, 1), 3, 2, 1, 3, 0.4, bc=((0, 0), (1, 2), (1, 1))),
], ids=lambda p: p.name)
@pytest.mark.parametrize("nchunks", [1, 3, 16])
def test_step_host_equals_set_step_get(sp, p, nchunks):
    U0 = oracle.prim_to_cons(p.ndim, p.gamma, si.random_state(p, 7))
    ref = sp.Spark(p.config())
    ref.set_state(U0)
    want = []
    U = U0.copy()
    for _ in range(3):
        ref.set_state(U)
        ref.step()
        U = ref.get_state().cpu().numpy()
        want.append(U.copy())
    s = sp.Spark(p.config(), stream=torch.cuda.Stream())
    s.set_state(U0)
    host = torch.from_numpy(U0.copy()).pin_memory().numpy()
    for k in range(3):  # back to back, synchronised only at the end
        s.step_host(host, host, nchunks=nchunks)
    s.sync()
    assert np.array_equal(host, want[-1])
    t, n, _ = s.time()
    assert n == 3
    s.close()
    ref.close()
