"""Small end-to-end run of every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck; one tool per process)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import spark_inputs as si  # noqa: E402
from paper_2401_03378_b200 import spark  # noqa: E402

cases = [
    si.Problem("s3p", 3, (16, 16, 16), (2, 1, 2), 2, 1, 1, 2, 0.3, bc=((1, 1), (0, 0), (2, 1))),
    si.Problem("s3w", 3, (16, 16, 16), (1, 2, 2), 3, 2, 1, 3, 0.3, bc=((0, 0), (1, 2), (1, 1))),
    si.Problem("s3o", 3, (6, 5, 7), (2, 2, 2), 3, 2, 0, 3, 0.3, bc=((2, 1), (0, 0), (0, 0))),
    si.Problem("s2w", 2, (16, 16, 1), (2, 3, 1), 3, 2, 1, 3, 0.4, bc=((0, 0), (1, 2), (1, 1))),
    si.Problem("s1", 1, (8, 1, 1), (4, 1, 1), 2, 1, 1, 2, 0.8, bc=((1, 1),) * 3),
]
for p in cases:
    W = si.random_state(p, 3, blocky=True)
    s = spark.Spark(p.config())
    s.set_primitive(W)
    for _ in range(2):
        s.step()
    s.fill_guardcells()
    U = s.get_state()
    s.stage_apply(U, U, 0.5, 0.5, 1e-4)
    torch.cuda.synchronize()
    s.close()
# multi-rank code paths on one GPU: virtual ranks and NCCL self-exchange
p = si.Problem("g", 3, (8, 8, 8), (2, 2, 2), 2, 1, 1, 2, 0.3, bc=((0, 0),) * 3)
grp = spark.LocalGroup(p.config(), 2)
for r, s in enumerate(grp.ranks):
    q = p.with_(nblk=spark.rank_box(p.config(), r, 2)[1])
    s.set_primitive(si.random_state(q, r))
grp.step()
grp.step()
torch.cuda.synchronize()
grp.close()
s = spark.Spark(p.config(), nccl_id=spark.nccl_unique_id())
s.set_primitive(si.random_state(p, 5))
s.step()
s.step()
torch.cuda.synchronize()
s.close()
x = torch.ones(1001, dtype=torch.float64, device="cuda")
y = torch.zeros(1001, dtype=torch.float64, device="cuda")
for v in range(4):
    spark.axpy(v, 0.5, x, y)
torch.cuda.synchronize()
print("sanitize case ok")
