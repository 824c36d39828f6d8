#!/bin/bash
# Bench + ncu evidence for one configuration (run on the GPU box):
#   tools/profile_cfg.sh <cfg> <tag>
# 1. bench line (no profiler)                  -> gpurun_out/bench_cfg<cfg>_<tag>.json
# 2. launch list of ONE timed solve (ncu --metrics gpu__time_duration.sum, profiler range =
#    the bench's timed region via TLS_PROFILE_RANGE=1)  -> gpurun_out/launches_cfg<cfg>_<tag>.csv
# 3. ncu --set full of the first band-solve launch of that solve -> gpurun_out/ncu_band_cfg<cfg>_<tag>.ncu-rep
set -u
C=$1; T=$2; O=gpurun_out
mkdir -p $O
python bench.py --config $C --steps ${STEPS:-3} --warmup 3 > $O/bench_cfg${C}_${T}.json 2> $O/bench_cfg${C}_${T}.err || exit 1
TLS_PROFILE_RANGE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_cfg${C}_${T}.csv python bench.py --config $C --steps 1 --warmup 1 --no-cpu-baseline \
  > /dev/null 2> $O/launches_cfg${C}_${T}.err
TLS_PROFILE_RANGE=1 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:${KERNEL:-k_band_solve} -c 1 -f -o $O/ncu_band_cfg${C}_${T} python bench.py --config $C --steps 1 --warmup 1 \
  --no-cpu-baseline > /dev/null 2> $O/ncu_band_cfg${C}_${T}.err
ls -la $O
