"""spark_run: CUDA-graph replay of 3-step groups gives exactly the same results
as individual spark_step calls (same kernels, same arguments)."""
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


@pytest.mark.parametrize("name", ["c1_sod1d", "c2b_sod2d"])
def test_graph_run_bitwise(sp, name):
    p = si.PRESETS[name]
    U0 = oracle.prim_to_cons(p.ndim, p.gamma, si.initial_primitive(p))
    st = torch.cuda.Stream()
    a = sp.Spark(p.config(), stream=st)
    b = sp.Spark(p.config(), stream=st)
    a.set_state(U0)
    b.set_state(U0)
    for _ in range(10):
        a.step()
    b.run(10)  # 3 graph replays of 3 steps + 1 plain step
    st.synchronize()
    assert np.array_equal(a.get_state().cpu().numpy(), b.get_state().cpu().numpy())
    assert a.time() == b.time()
    # the cached graphs are reused, and re-captured when dt changes
    for _ in range(6):
        a.step(dt=1e-4)
    b.run(6, dt=1e-4)
    assert np.array_equal(a.get_state().cpu().numpy(), b.get_state().cpu().numpy())


def test_graph_run_to_t_end(sp):
    p = si.PRESETS["c1_sod1d"]
    U0 = oracle.prim_to_cons(1, 1.4, si.initial_primitive(p))
    st = torch.cuda.Stream()
    s = sp.Spark(p.config(), stream=st)
    s.set_state(U0)
    s.run(600, t_end=0.2)  # more steps than needed: the tail copies U through
    t, n, _ = s.time()
    Uo, to, no = oracle.run(p.config(), U0, t_end=0.2)
    assert abs(t - 0.2) < 1e-15 and n == no
    g = s.get_state().cpu().numpy()
    scale = np.abs(Uo).max(axis=tuple(range(1, Uo.ndim)), keepdims=True)
    assert np.all(np.abs(g - Uo) <= 1e-12 * np.abs(Uo) + 1e-14 * scale)
