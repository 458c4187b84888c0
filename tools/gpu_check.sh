#!/bin/bash
# correctness + both benches (run under gpurun)
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
echo tests_exit=$? >> gpurun_out/gpu_tests.log
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_plm.log 2>&1
python bench.py --config c4_sedov3d_weno --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_weno.log 2>&1
python bench.py --config c3_sedov2d --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c3.log 2>&1
