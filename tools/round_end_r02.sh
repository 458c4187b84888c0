#!/bin/bash
# Round-2 end check (run under gpurun; one GPU): the whole GPU suite, smoke,
# the default bench line, the reference arm, a compute-sanitizer memcheck of a
# small 3-D step, and the stall-line attribution of KB1.
mkdir -p gpurun_out/end
O=gpurun_out/end
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gpu_all.log 2>&1; echo "tests rc=$?" >> $O/gpu_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
cat > /tmp/sanit.py <<'PY'
import sys; sys.path.insert(0, ".")
import numpy as np, oracle, spark_inputs as si
from paper_2401_03378_b200 import spark
for name, kw in [("c4_sedov3d_plm", {}), ("c4_sedov3d_weno", {}), ("c4_sedov3d_plm", {"riemann": 2, "shock_thresh": 0.5})]:
    p = si.PRESETS[name].with_(nblk=(2, 2, 2), **kw)
    s = spark.Spark(p.config()); s.set_primitive(si.initial_primitive(p))
    for _ in range(2): s.step()
    s.step_telescoping(); s.sync(); s.close()
p = si.Problem("a", 3, (8, 8, 8), (3, 3, 3), 2, 1, 1, 2, 0.3)
a = spark.Amr(p.config(), (1, 1, 1), (2, 2, 2))
W = si.amr_primitive(p, (1, 1, 1), (2, 2, 2), "pulse")
U = oracle.prim_to_cons(3, 1.4, W.reshape(5, W.shape[1], -1)).reshape(W.shape)
a.set_state(U); a.step(sync=True); a.close()
print("sanitizer workload ok")
PY
timeout 900 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python /tmp/sanit.py > $O/memcheck.log 2>&1; echo "memcheck rc=$?" >> $O/memcheck.log
R=/tmp/end; mkdir -p $R
Q="--no-cpu-baseline --no-calibration --no-secondary --e2e-steps 1"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:stage_kernel" -s 4 -c 2 -o $R/prof python bench.py --steps 3 --warmup 3 $Q > $O/ncu.log 2>&1
mkdir -p /tmp/cub && (cd /tmp/cub && cuobjdump -xelf all $GRAFT_REPO_ROOT/paper_2401_03378_b200/lib/libspark.so > /dev/null 2>&1)
CUB=$(grep -l "stage_kernelILi3ELi1ELi1ELi16ELi16ELi16" /tmp/cub/*.cubin 2>/dev/null | head -1)
python tools/ncu_lines.py $R/prof.ncu-rep "$CUB" "stage_kernel<(int)3, (int)1, (int)1" 40 > $O/ncu_lines_c4_plm.txt 2>&1
echo done
