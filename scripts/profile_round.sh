#!/bin/bash
# Round profile capture (run under gpurun, 1 GPU): launch list of the bench command + one
# `ncu --set full` capture per hot kernel (config 2, Gaussian) + the τ kernel on a sparse input.
# Usage: bash scripts/profile_round.sh <tag>     → gpurun_out/<tag>_*.{csv,ncu-rep}
set -u
TAG=${1:-r01}
O=gpurun_out
mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > $O/${TAG}_launches_bench.log 2>&1
for K in tau_kernel out_kernel dkdv_kernel dq_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -f \
      -o $O/${TAG}_full_$K python scripts/run_fwd.py gaussian 1.0 bwd > $O/${TAG}_full_$K.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tau_kernel -s 1 -c 1 -f \
    -o $O/${TAG}_full_tau_planted05 python scripts/run_fwd.py planted 0.05 > $O/${TAG}_full_tau_planted05.log 2>&1

# keep the merge under gpurun's 64 MiB: CSV pages here, compressed reports
for R in $O/${TAG}_full_*.ncu-rep; do
  ncu -i $R --page raw --csv > ${R%.ncu-rep}_raw.csv 2>/dev/null
  ncu -i $R --page source --csv --print-source sass > ${R%.ncu-rep}_src.csv 2>/dev/null
  gzip -9 -c ${R%.ncu-rep}_src.csv > ${R%.ncu-rep}_src.csv.gz && rm ${R%.ncu-rep}_src.csv
  xz -9 -T0 $R 2>/dev/null || gzip -9 $R
done
du -sh $O
# drop compressed reports (largest first) until the directory is under 56 MiB
while [ $(du -sm $O | cut -f1) -gt 56 ]; do
  F=$(ls -S $O/*.ncu-rep.* 2>/dev/null | head -1); [ -z "$F" ] && break; rm -f "$F"
done
du -sh $O
