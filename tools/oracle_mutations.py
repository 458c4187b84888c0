"""Mutation check of the oracle's pins (test infrastructure; CPU only).

    python tools/oracle_mutations.py [--list] [NAME ...]

Each mutation is a plausible misreading of the method (a dropped term, a wrong
constant, sign or index) applied to a copy of ``oracle/spark_oracle.c``.  The
copy is compiled with the oracle's own flags into /tmp and the oracle pin tests
run against it (``SPARK_ORACLE_LIB``); a mutation is "caught" when at least one
pin fails.  The table it prints is recorded in DESIGN.md §3.
"""
from __future__ import annotations

import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

SRC = os.path.join(ROOT, "oracle", "spark_oracle.c")
PINS = ["tests/test_oracle_pins.py", "tests/test_oracle_n2.py", "tests/test_oracle_telescoping.py",
        "tests/test_oracle_weno_weights.py", "tests/test_oracle_hllc_star.py", "tests/test_oracle_shockdet.py", "tests/test_oracle_amr.py"]

# (name, exact text in spark_oracle.c, replacement, occurrence index or None for all)
MUTATIONS = [
    ("WENO-JS beta0 13/12 -> 1/12",
     "double b0 = 13.0 / 12.0 * (a - 2.0 * b + c)", "double b0 = 1.0 / 12.0 * (a - 2.0 * b + c)", 0),
    ("WENO-JS beta1 1/4 -> 3/4", "+ 0.25 * (b - d) * (b - d);", "+ 0.75 * (b - d) * (b - d);", 0),
    ("WENO-JS beta2 1/4 -> 1/2", "+ 0.25 * (3.0 * c - 4.0 * d + e)", "+ 0.5 * (3.0 * c - 4.0 * d + e)", 0),
    ("WENO-JS exponent 2 -> 1", "double a0 = 0.1 / ((eps + b0) * (eps + b0));", "double a0 = 0.1 / (eps + b0);", 0),
    ("WENO-JS eps 1e-6 -> 1e-40", "const double eps = 1e-6;", "const double eps = 1e-40;", 0),
    ("WENO-JS linear weight 0.6 -> 0.5", "double a1 = 0.6 / ((eps + b1)", "double a1 = 0.5 / ((eps + b1)", 0),
    ("WENO candidate q1 5c -> 4c", "double q1 = (-b + 5.0 * c + 2.0 * d) / 6.0;",
     "double q1 = (-b + 4.0 * c + 3.0 * d) / 6.0;", 0),
    ("PLM right state sign", "*wr = w1 - 0.5 * d1;", "*wr = w1 + 0.5 * d1;", 0),
    ("minmod keeps opposite signs", None, None, None),
    ("MC centred slope 1/2 -> 0.6", "0.5 * (dl + dr)", "0.6 * (dl + dr)", 0),
    ("HLLC S* sign of p_L", "double sstar = (pr - pl +", "double sstar = (pr + pl +", 0),
    ("HLLC star energy drops p/(rho(S-u))", "(sstar + p / (rho * (sk - un)))", "(sstar)", 0),
    ("HLL drops the dissipation term", "+ sl * sr * (ur[v] - ul[v])", "", 0),
    ("Davis speed S_R uses u_L only", "double sr = fmax(uL + cl, uR + cr);", "double sr = uL + cl;", 0),
    ("momentum flux drops p", "f[1] = rho * un * un + p;", "f[1] = rho * un * un;", 0),
    ("EOS kinetic energy 1/2 -> 1", "(u[ndim + 1] - 0.5 * ke / rho)", "(u[ndim + 1] - ke / rho)", 0),
    ("z divergence sign", "else L = -(div[0] + div[1]) - div[2];", "else L = -(div[0] + div[1]) + div[2];", 0),
    ("RK3 stage 2 weights 3/4,1/4 -> 2/3,1/3", "*a = 0.75; *b = 0.25;", "*a = 2.0 / 3.0; *b = 1.0 / 3.0;", 0),
    ("outflow map off by one", "if (bc == OBC_OUTFLOW) return g < 0 ? 0 : N - 1;",
     "if (bc == OBC_OUTFLOW) return g < 0 ? 1 : N - 1;", 0),
    ("reflect keeps the normal momentum", "if (v >= 1 && v <= c->ndim && flip[v - 1]) val = -val;", "", 0),
    ("positivity fallback removed",
     "if (!(wl[0] > 0.0) || !(wl[nv - 1] > 0.0) || !(wr[0] > 0.0) || !(wr[nv - 1] > 0.0)) {", "if (0) {", 0),
    ("positivity fallback tests rho only",
     "if (!(wl[0] > 0.0) || !(wl[nv - 1] > 0.0) || !(wr[0] > 0.0) || !(wr[nv - 1] > 0.0)) {",
     "if (!(wl[0] > 0.0) || !(wr[0] > 0.0)) {", 0),
    ("shockDet compression test reversed", "if (!(d < 0.0)) return 0;", "if (!(d > 0.0)) return 0;", 0),
    ("shockDet without the sound-speed dead band",
     "if (!(d * d * (rm * rp) > 1e-12 * gamma * (a > b ? a : b))) return 0;", "", 0),
    ("shockDet jump relative to max p", "double pmin = pm < pp ? pm : pp;", "double pmin = pm > pp ? pm : pp;", 0),
    ("shockDet face uses cell i only", "||\n           shock_cell(un[1], un[3], p[1], p[3], rho[1], rho[3], thresh, gamma);",
     ";", 0),
    ("hybrid picks HLLC at shocks", "? ORS_HLL : ORS_HLLC;", "? ORS_HLLC : ORS_HLL;", 0),
    ("AMR correction sign flipped", "*uq = side ? *uq + corr : *uq - corr;", "*uq = side ? *uq - corr : *uq + corr;", 0),
    ("AMR fluxBuff without the stage weight", "*bq = sb * (*bq + Fl[q]);", "*bq = *bq + Fl[q];", 0),
    ("AMR restriction takes one child", "if (n == 4) return ((s[0] + s[3]) + (s[1] + s[2])) * 0.25;",
     "if (n == 4) return s[0];", 0),
    ("AMR prolongation from the neighbour coarse cell", "cg[d] = d < c->ndim ? g[d] / 2 : g[d];",
     "cg[d] = d < c->ndim ? (g[d] + 1) / 2 : g[d];", 0),
    ("AMR face mean uses one fine face", "else if (nf == 2) fsum[v] = (s4[0] + s4[1]) * 0.5;",
     "else if (nf == 2) fsum[v] = s4[0];", 0),
    ("AMR fine dt spacing not halved", "const double f = leaf < ncl ? 1.0 : 0.5;", "const double f = 1.0;", 0),
    ("CFL uses sqrt(p/rho)", "double cs = sqrt(c->gamma * w[nv - 1] / w[0]);", "double cs = sqrt(w[nv - 1] / w[0]);", 0),
]


def apply(src: str, find: str, repl: str, occ):
    if occ is None:
        if find not in src:
            raise KeyError(find)
        return src.replace(find, repl)
    idx = -1
    for _ in range(occ + 1):
        idx = src.index(find, idx + 1)
    return src[:idx] + repl + src[idx + len(find):]


def extra_mutations(src: str):
    """Mutations that need context (found by pattern, listed in MUTATIONS with None)."""
    out = {}
    s = src
    i = s.find("static double minmod(")
    if i >= 0:
        j = s.index("}", i)
        body = s[i:j]
        out["minmod keeps opposite signs"] = s[:i] + body.replace("return 0.0;", "return a;", 1) + s[j:]
    return out


def run(name: str, text: str, tmp: str) -> tuple[bool, str]:
    c = os.path.join(tmp, "mut.c")
    so = os.path.join(tmp, "libmut.so")
    with open(c, "w") as f:
        f.write(text)
    subprocess.check_call(["gcc", *oracle.CFLAGS, "-o", so, c, "-lm"])
    pins = [p for p in PINS if os.path.exists(os.path.join(ROOT, p))]
    env = dict(os.environ, SPARK_ORACLE_LIB=so)
    # a mutation that makes a pin run away (e.g. a wrong CFL dt) fails by timeout
    r = subprocess.run([sys.executable, "-m", "pytest", *pins, "-q", "-rf", "-p", "no:cacheprovider", "-n", "4",
                        "--timeout", "120"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1800)
    failed = sorted({ln.split()[1].split("::")[-1].split("[")[0] for ln in r.stdout.splitlines()
                     if ln.startswith("FAILED")})
    return r.returncode != 0, (f"{len(failed)} pins fail: " + ", ".join(failed)) if failed else \
        r.stdout.strip().splitlines()[-1]


def main():
    src = open(SRC).read()
    extra = extra_mutations(src)
    want = [a for a in sys.argv[1:] if not a.startswith("--")]
    rows = []
    with tempfile.TemporaryDirectory() as tmp:
        for name, find, repl, occ in MUTATIONS:
            if want and not any(w in name for w in want):
                continue
            if "--list" in sys.argv:
                print(name)
                continue
            text = extra[name] if find is None else apply(src, find, repl, occ)
            if text == src:
                raise SystemExit(f"mutation {name!r} changed nothing")
            caught, why = run(name, text, tmp)
            rows.append((name, caught, why))
            print(f"{'caught' if caught else 'MISSED':7s} {name:42s} {why}", flush=True)
    if any(not c for _, c, _ in rows):
        sys.exit(1)


if __name__ == "__main__":
    main()
