"""The checked build really carries its bounds checks (CPU: SASS inspection):
KB1's production instantiation traps on a violation in libspark_checked.so
and carries no trap in libspark.so (the checks compile away)."""
import shutil
import subprocess

import pytest

from paper_2401_03378_b200 import build

CUOBJDUMP = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
KB1 = "stage_kernelILi3ELi1ELi1ELi16ELi16ELi16"  # 3-D PLM HLLC 16^3: the bench kernel


def traps(lib: str) -> int:
    """BPT.TRAP instructions in the SASS of the KB1 function of lib."""
    r = subprocess.run([CUOBJDUMP, "-sass", lib], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    n, inside, seen = 0, False, False
    for ln in r.stdout.splitlines():
        if "Function :" in ln:
            inside = KB1 in ln
            seen |= inside
        elif inside and "BPT.TRAP" in ln:
            n += 1
    assert seen, f"{KB1} not in {lib}"
    return n


def test_checked_build_traps_and_production_does_not():
    if not shutil.which(CUOBJDUMP) and not __import__("os").path.exists(CUOBJDUMP):
        pytest.skip("no cuobjdump")
    assert traps(build.build_checked()) > 0
    assert traps(build.build()) == 0
