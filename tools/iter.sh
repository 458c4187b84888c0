#!/bin/bash
# one design-iteration GPU call: parity subset + quick rates (run under gpurun)
T=${1:-it}
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_invariants.py -q -x -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1
echo tests_exit=$? >> gpurun_out/${T}_tests.log
tail -3 gpurun_out/${T}_tests.log
for c in c4_sedov3d_plm c4_sedov3d_weno c3_sedov2d; do timeout 120 python tools/quick_rate.py $c; done > gpurun_out/${T}_rates.log 2>&1
cat gpurun_out/${T}_rates.log
