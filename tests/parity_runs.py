"""Full-run parity statistics, GPU (through the C ABI) vs the oracle (test helper).

    python tests/parity_runs.py [--lib PATH] [CASE ...]   -> one JSON object on stdout

For configs[0]/[1] (C1, C2a, C2b: hundreds of steps to t_end) it reports per
conserved variable the largest error relative to max|o_v| (the absolute floor
of reading R15), the largest error relative to |o| where |o| > 1e-12 max|o_v|,
whether the R15 tolerance holds at floor 1e-15 and at 1e-14, and a histogram
of err / max|o_v| over decades (cells with err == 0 counted apart).  Used by
tests/test_gpu_strict.py (the --fmad=false / IEEE-division build at the
original 1e-15 floor) and by tools/parity_histogram.sh (profiles/).
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

CASES = ["c1_sod1d", "c2a_sod2d", "c2b_sod2d"]
DECADES = list(range(-18, -9))


def stats(g: np.ndarray, o: np.ndarray) -> list[dict]:
    out = []
    for v in range(o.shape[0]):
        scale = float(np.max(np.abs(o[v])))
        err = np.abs(g[v] - o[v])
        rel_floor = err / scale
        big = np.abs(o[v]) > 1e-12 * scale
        hist = {"zero": int(np.sum(err == 0))}
        nz = rel_floor[err > 0]
        for d in DECADES:
            hist[f"1e{d}"] = int(np.sum((nz >= 10.0 ** d) & (nz < 10.0 ** (d + 1))))
        hist["above"] = int(np.sum(nz >= 10.0 ** (DECADES[-1] + 1)))
        out.append({
            "max_err_over_maxabs": float(rel_floor.max()),
            "max_rel_err": float(np.max(err[big] / np.abs(o[v][big]))) if big.any() else 0.0,
            "ok_floor_1e-15": bool(np.all(err <= 1e-12 * np.abs(o[v]) + 1e-15 * scale)),
            "ok_floor_1e-14": bool(np.all(err <= 1e-12 * np.abs(o[v]) + 1e-14 * scale)),
            "hist_err_over_maxabs": hist,
        })
    return out


def run_case(name: str) -> dict:
    import oracle
    import spark_inputs as si
    from paper_2401_03378_b200 import spark

    p = si.PRESETS[name]
    U0 = oracle.prim_to_cons(p.ndim, p.gamma, si.initial_primitive(p))
    Uo, to, no = oracle.run(p.config(), U0, t_end=p.t_end)
    s = spark.Spark(p.config())
    s.set_state(np.ascontiguousarray(U0))
    s.advance(10_000, t_end=p.t_end, check_every=32)
    t, steps, _ = s.time()
    g = s.get_state().cpu().numpy()
    s.close()
    return {"case": name, "steps": int(steps), "oracle_steps": int(no), "t": t, "oracle_t": to,
            "vars": stats(g, Uo)}


def main():
    args = sys.argv[1:]
    if "--lib" in args:
        i = args.index("--lib")
        os.environ["SPARK_LIB"] = args[i + 1]
        del args[i:i + 2]
    from paper_2401_03378_b200 import spark

    lib = spark.LIB_PATH
    spark.lib()
    res = {"lib": os.path.basename(lib), "cases": [run_case(c) for c in (args or CASES)]}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
