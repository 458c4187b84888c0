#!/bin/bash
# re-measure the secondary bench lines of profiles/ at the current commit (run under gpurun; one GPU)
mkdir -p gpurun_out
B="python bench.py --no-cpu-baseline --no-calibration --e2e-steps 1"
timeout 300 $B --config c3_sedov2d --steps 400 --warmup 5 > gpurun_out/rf_c3.log 2>&1
timeout 300 $B --recon first --steps 100 --warmup 5 > gpurun_out/rf_first.log 2>&1
timeout 300 $B --recon mc --steps 100 --warmup 5 > gpurun_out/rf_mc.log 2>&1
timeout 300 $B --recon wenoz --config c4_sedov3d_weno --steps 100 --warmup 5 > gpurun_out/rf_wenoz.log 2>&1
timeout 600 $B --config c5_sedov3d_plm --steps 10 --warmup 3 > gpurun_out/rf_c5plm.log 2>&1
timeout 900 $B --config c5_sedov3d_weno --steps 5 --warmup 3 > gpurun_out/rf_c5weno.log 2>&1
