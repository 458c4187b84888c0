#!/bin/bash
# Error histograms of the full C1/C2a/C2b runs for the production and the
# parity (--fmad=false, IEEE div/sqrt) builds (run under gpurun; one GPU).
mkdir -p gpurun_out
python tests/parity_runs.py > gpurun_out/parity_default.json 2> gpurun_out/parity_default.err
python tests/parity_runs.py --lib paper_2401_03378_b200/lib/libspark_strict.so > gpurun_out/parity_strict.json 2> gpurun_out/parity_strict.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/parity_default.json"))
s = json.load(open("gpurun_out/parity_strict.json"))
json.dump({"production": d, "strict": s}, open("gpurun_out/r02_parity_histogram.json", "w"), indent=1)
for tag, r in (("production", d), ("strict", s)):
    for c in r["cases"]:
        print(tag, c["case"], [f"{v['max_err_over_maxabs']:.2e}" for v in c["vars"]],
              "floor1e-15:", all(v["ok_floor_1e-15"] for v in c["vars"]))
PY
