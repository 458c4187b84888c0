import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle, spark_inputs as si
from paper_2401_03378_b200 import spark
from tests.test_gpu_parity import STAGE_CASES
p = STAGE_CASES[3]
U = oracle.prim_to_cons(p.ndim, p.gamma, si.random_state(p, 1))
s = spark.Spark(p.config())
U2 = U.copy(); U2[3, 2, 0, 5, 5] = -50.0
s.set_state(U2)
torch.cuda.synchronize()
sc = s.arena[:64].cpu().numpy()
print("status word", sc[40:44].view(np.int32), "acc", sc[24:32].view(np.float64))
try:
    print("dt", s.step(dt=1e-4, sync=True))
except Exception as e:
    print("raised", type(e).__name__, e)
sc = s.arena[:64].cpu().numpy()
print("status word", sc[40:44].view(np.int32))
