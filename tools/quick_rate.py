"""Quick zone-update rate of a problem (for design experiments): python tools/quick_rate.py NAME [k=v ...]"""
import sys

import torch

sys.path.insert(0, ".")
import spark_inputs as si  # noqa: E402
from paper_2401_03378_b200 import spark  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1].endswith(".so"):  # a variant library (tools/ablate.sh)
    spark.LIB_PATH = sys.argv.pop(1)

p = si.PRESETS[sys.argv[1]]
kw = {}
for a in sys.argv[2:]:
    k, v = a.split("=")
    kw[k] = eval(v)
p = p.with_(**kw)
st = torch.cuda.Stream()
s = spark.Spark(p.config(), stream=st)
s.set_primitive(si.initial_primitive(p))
for _ in range(3):
    s.step()
st.synchronize()
s.profile(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
n = 10
for _ in range(n):
    s.step()
e1.record(st)
st.synchronize()
ms, launches, _ = s.profile_read()
print(f"{p.name} {kw}: {p.ncells * p.rk_stages * n / (e0.elapsed_time(e1) * 1e-3) / 1e9:.2f} Gzu/s, "
      f"stage kernel {ms / launches:.3f} ms/launch, {p.ncells / (ms / launches * 1e-3) / 1e9:.2f} Gcell-stages/s")
