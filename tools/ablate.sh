#!/bin/bash
# Design experiments: build variant libraries with -D flags (here, on CPU) and
# time them on the GPU box with tools/quick_rate.py.
#   here:     bash tools/ablate.sh build NAME "-DFLAG1 -DFLAG2" ...
#   gpurun:   bash tools/ablate.sh run CONFIG
set -e
D=paper_2401_03378_b200/lib/abl
if [ "$1" = build ]; then
    shift
    mkdir -p $D
    while [ $# -gt 0 ]; do
        python -m paper_2401_03378_b200.build --force --out=$D/$1.so $2 > /dev/null
        shift 2
    done
    ls $D
else
    cfg=${2:-c4_sedov3d_plm}
    for f in paper_2401_03378_b200/lib/libspark.so $(ls $D/*.so 2>/dev/null); do
        echo "== $f"; python tools/quick_rate.py $f $cfg; python tools/quick_rate.py $f $cfg
    done
fi
