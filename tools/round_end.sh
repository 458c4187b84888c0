#!/bin/bash
# full GPU check + refreshed bench lines + launch list (run under gpurun; one GPU)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_all.log 2>&1
echo tests_exit=$? >> gpurun_out/gpu_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
echo smoke_exit=$? >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_plm_full.log 2>&1
timeout 600 python bench.py --config c4_sedov3d_weno --no-calibration > gpurun_out/bench_weno_full.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
timeout 900 bash tools/profile.sh r01end c4_sedov3d_plm > gpurun_out/profile.log 2>&1
