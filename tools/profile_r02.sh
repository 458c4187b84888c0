#!/bin/bash
# Round-2 evidence (run under gpurun; one GPU): bench lines of every path, the
# ncu launch list of the default bench, and `ncu --set full` captures of the
# top kernel of each path (KB1 PLM and WENO5, the hybrid KB1, the N3 face
# kernel, the N1 tile face kernel).  Each ncu command runs only after its plain
# command has exited 0.
mkdir -p gpurun_out/r02 /tmp/r02
O=gpurun_out/r02
R=/tmp/r02   # ncu reports stay on the box (gpurun_out is capped at 64 MiB); summaries come back
Q="--no-cpu-baseline --no-calibration --no-secondary --e2e-steps 1"
run() { tag=$1; shift; timeout 600 python bench.py "$@" > $O/bench_$tag.json 2> $O/bench_$tag.err; echo "$tag rc=$?"; }
run c4_plm
run c4_weno --config c4_sedov3d_weno --no-calibration --no-secondary
run c4_hybrid --riemann hybrid $Q --steps 50
run c4_first --recon first $Q --steps 50
run c4_mc --recon mc $Q --steps 50
run c4_wenoz --recon wenoz --config c4_sedov3d_weno $Q --steps 20
run c3_weno2d --config c3_sedov2d $Q --steps 200
run c4_amr_plm --amr --steps 10 --warmup 3
run c4_tel_plm --telescoping $Q --steps 10
run reference --impl reference --steps 3 --warmup 3
CMD="python bench.py --steps 3 --warmup 3 $Q"
$CMD > $O/plain_plm.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4_plm.csv $CMD > /dev/null 2>&1
echo "launch list rc=$?"
cap() { tag=$1; kern=$2; skip=$3; cnt=$4; shift 4
  timeout 600 python bench.py "$@" > $O/plain_$tag.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$kern" -s $skip -c $cnt \
      -o $R/prof_$tag python bench.py "$@" > $O/ncu_$tag.log 2>&1
  echo "capture $tag rc=$?"
  python tools/ncu_summary.py $R/prof_$tag.ncu-rep > $O/ncu_full_$tag.txt 2>&1; }
cap c4_plm stage_kernel 4 2 --steps 3 --warmup 3 $Q
cap c4_weno stage_kernel 5 3 --config c4_sedov3d_weno --steps 3 --warmup 3 $Q
cap c4_hybrid stage_kernel 4 2 --riemann hybrid --steps 3 --warmup 3 $Q
cap c4_amr amr_leaf_kernel 6 1 --amr --steps 2 --warmup 3
cap c4_tel tt_face_kernel 6 1 --telescoping --steps 2 --warmup 3 $Q
python tools/fp64_count.py $R/prof_c4_plm.ncu-rep stage_kernel 16777216 > $O/instmix_c4_plm.txt 2>&1
python tools/fp64_count.py $R/prof_c4_weno.ncu-rep stage_kernel 16777216 > $O/instmix_c4_weno.txt 2>&1
python tools/fp64_count.py $R/prof_c4_hybrid.ncu-rep stage_kernel 16777216 > $O/instmix_c4_hybrid.txt 2>&1
python tools/make_ncu_summary.py $R/prof_c4_plm.ncu-rep $R/prof_c4_weno.ncu-rep "round-2 capture (tools/profile_r02.sh)" > $O/ncu_summary.log 2>&1
cp profiles/ncu_summary.json $O/ncu_summary.json
mkdir -p /tmp/cub && (cd /tmp/cub && cuobjdump -xelf all $GRAFT_REPO_ROOT/paper_2401_03378_b200/lib/libspark.so > /dev/null 2>&1)
CUB=$(grep -l "stage_kernelILi3ELi1ELi1ELi16ELi16ELi16" /tmp/cub/*.cubin 2>/dev/null | head -1)
python tools/ncu_lines.py $R/prof_c4_plm.ncu-rep "$CUB" "stage_kernel<(int)3, (int)1, (int)1" 40 > $O/ncu_lines_c4_plm.txt 2>&1
ls -la $R > $O/reports.txt
echo done
