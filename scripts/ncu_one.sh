#!/bin/bash
# One `ncu --set full` capture of kernel regex $2 under run_fwd.py args $3.. → gpurun_out/$1_{raw,src}.csv(.gz)
set -u
TAG=$1; K=$2; shift 2
O=gpurun_out; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -f -o $O/$TAG \
    python scripts/run_fwd.py "$@" > $O/$TAG.log 2>&1
ncu -i $O/$TAG.ncu-rep --page raw --csv > $O/${TAG}_raw.csv 2>/dev/null
ncu -i $O/$TAG.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip -9 > $O/${TAG}_src.csv.gz
xz -9 -T0 $O/$TAG.ncu-rep
