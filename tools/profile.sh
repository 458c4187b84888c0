#!/bin/bash
# ncu evidence for the stage kernel (run under gpurun; one GPU).
# usage: tools/profile.sh TAG [CONFIG]
TAG=${1:-r1}; CFG=${2:-c4_sedov3d_plm}
CMD="python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline --no-calibration --e2e-steps 1"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 4 -c 2 -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_${TAG}.log 2>&1
echo "profile exit $?"
