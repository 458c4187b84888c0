#!/bin/bash
# Round-2 end check (run under gpurun; one GPU): the whole GPU suite, smoke,
# the default bench line, the reference arm and the stall-line attribution of KB1.
mkdir -p gpurun_out/end
O=gpurun_out/end
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gpu_all.log 2>&1; echo "tests rc=$?" >> $O/gpu_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
# (compute-sanitizer is closed on this pool: DESIGN.md §10)
R=/tmp/end; mkdir -p $R
Q="--no-cpu-baseline --no-calibration --no-secondary --e2e-steps 1"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:stage_kernel" -s 4 -c 2 -o $R/prof python bench.py --steps 3 --warmup 3 $Q > $O/ncu.log 2>&1
mkdir -p /tmp/cub && (cd /tmp/cub && cuobjdump -xelf all $GRAFT_REPO_ROOT/paper_2401_03378_b200/lib/libspark.so > /dev/null 2>&1)
CUB=$(grep -l "stage_kernelILi3ELi1ELi1ELi16ELi16ELi16" /tmp/cub/*.cubin 2>/dev/null | head -1)
python tools/ncu_lines.py $R/prof.ncu-rep "$CUB" "stage_kernel<(int)3, (int)1, (int)1" 40 > $O/ncu_lines_c4_plm.txt 2>&1
echo done
