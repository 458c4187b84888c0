"""Full runs of configs[0]/[1] with the parity build: is the 1e-14 floor of
reading R15 an FMA artefact?

``libspark_strict.so`` is the same CUDA source compiled with ``--fmad=false``
and ``-DSPARK_STRICT_MATH`` (no fused multiply-add anywhere, IEEE division and
square root, R15/R16).  Measured on B200
(profiles/r02_parity_histogram.json): over the 68-139 steps of C1/C2a/C2b
both builds leave the same error distribution — largest |g - o| / max|o_v|
2.4-3.9e-15 (production) and 2.5-2.7e-15 (strict), in 1-10 % of the cells
above 1e-15 — so the excess over the single-step floor 1e-15 comes from the
regrouped-but-equally-rounded formulas of the device code (multiplied-out
HLLC, reciprocal forms), accumulated over the run, not from contraction.
This test pins that finding: both builds meet 1e-14 and their largest errors
agree within a factor 3.
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def runs(lib: str) -> dict:
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "parity_runs.py"), "--lib", lib],
                       capture_output=True, text=True, timeout=1200, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_strict_build_same_error_floor_as_production():
    from paper_2401_03378_b200 import build

    build.build_strict()  # no-op when fresh (__graft_entry__.build() builds it); never silently skipped
    strict, prod = runs(build.STRICT_LIB), runs(build.LIB)
    assert strict["lib"] == "libspark_strict.so" and prod["lib"] == "libspark.so"
    for cs, cp in zip(strict["cases"], prod["cases"]):
        for c in (cs, cp):
            assert c["steps"] == c["oracle_steps"] and abs(c["t"] - c["oracle_t"]) <= 1e-14, c
            for v, s in enumerate(c["vars"]):
                assert s["ok_floor_1e-14"], (c["case"], v, s)
        es = max(s["max_err_over_maxabs"] for s in cs["vars"])
        ep = max(s["max_err_over_maxabs"] for s in cp["vars"])
        assert es < 3 * ep and ep < 3 * es, (cs["case"], es, ep)
