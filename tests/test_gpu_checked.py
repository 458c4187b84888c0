"""The bounds-checked build (libspark_checked.so, -DSPARK_CHECKED) through the
KB1-heavy GPU tests: every shared-memory address KB1 forms must lie in the
launch's dynamic shared memory, every global address in one of the launch's
buffers, and every halo source the boundary map resolves inside the sub-box
or the received slab; a violation traps and fails the run.  This stands in
for compute-sanitizer memcheck, which the GPU pool refuses."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KB1_TESTS = ["tests/test_gpu_parity.py", "tests/test_gpu_shockdet.py", "tests/test_gpu_n2.py",
             "tests/test_gpu_fuzz_r02.py::test_fuzz_hybrid_steps", "tests/test_gpu_errors.py",
             "tests/test_gpu_host_step.py", "tests/test_gpu_telescoping.py", "tests/test_gpu_telescoping3d.py"]


def test_kb1_tests_pass_with_bounds_checks():
    from paper_2401_03378_b200 import build

    lib = build.build_checked()  # no-op when fresh (__graft_entry__.build() builds it)
    env = dict(os.environ, SPARK_LIB=lib)
    probe = subprocess.run([sys.executable, "-c", "from paper_2401_03378_b200 import spark; spark.lib(); "
                            "print(spark.LIB_PATH)"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert probe.returncode == 0 and probe.stdout.strip().endswith("libspark_checked.so"), probe.stderr[-2000:]
    r = subprocess.run([sys.executable, "-m", "pytest", *KB1_TESTS, "-m", "gpu", "-q", "-x", "-p", "no:cacheprovider"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1800)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
