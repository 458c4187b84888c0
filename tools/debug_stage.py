"""Debug helper: one stage on GPU vs oracle for a named test case; prints per-cell errors."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle, spark_inputs as si
from paper_2401_03378_b200 import spark
from tests.test_gpu_parity import STAGE_CASES
name = sys.argv[1]
p = [c for c in STAGE_CASES if c.name == name][0]
for rs in (0, 1):
    q = p.with_(riemann=rs)
    Up = oracle.prim_to_cons(q.ndim, q.gamma, si.random_state(q, 10))
    dt = 0.2 * q.cfl * oracle.dt_raw(q.config(), Up)
    s = spark.Spark(q.config()); s.set_state(Up)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    g = s.stage_apply(d(Up), d(Up), 0.0, 1.0, dt).cpu().numpy()
    o = oracle.stage(q.config(), Up, Up, 0.0, 1.0, dt)
    G = si.to_global(q, g); O = si.to_global(q, o)
    err = np.abs(G - O)
    print("riemann", rs, "max err per var", err.reshape(q.nvar, -1).max(axis=1))
    bad = np.argwhere(err[0] > 1e-10)
    print("bad cells (z,y,x):", bad[:20].tolist())
