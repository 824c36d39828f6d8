#!/bin/bash
# ncu --set full of the first launch of each in-tree setup kernel of one configuration (GPU box):
#   tools/prof_setup_ncu.sh <cfg> <tag> <kernel-regex> [...]
# Reports stay in /tmp (large: source import); the raw-page CSV of each goes to gpurun_out/ for
# tools/ncu_summary.py-style reading here.
set -u
C=$1; T=$2; shift 2
O=gpurun_out
mkdir -p $O
for K in "$@"; do
  timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:$K -c 1 -f \
    -o /tmp/setup_${K}_cfg${C}_${T} python tools/prof_setup_kernels.py $C > /dev/null 2> $O/setup_${K}_cfg${C}_${T}.err
  ncu -i /tmp/setup_${K}_cfg${C}_${T}.ncu-rep --page raw --csv > $O/setup_${K}_cfg${C}_${T}.csv 2>/dev/null
done
ls -la $O | tail -12
