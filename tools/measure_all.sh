#!/bin/bash
# Round-end measurement suite (GPU box): bench lines for all five configurations (with the CPU
# baseline), the reference arm, ncu launch lists of the timed solves, ncu --set full of the band
# kernel.  Outputs under gpurun_out/m/ (ncu reports stay in /tmp: only their raw-page CSV travels).
mkdir -p gpurun_out/m
R=${ROUND:-r02}
for c in ${CONFIGS:-5 2 1 3 4}; do
  timeout 1500 python bench.py --config $c > gpurun_out/m/bench_cfg${c}_$R.json 2> gpurun_out/m/bench_cfg${c}_$R.err
done
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/m/bench_reference_cfg5_$R.json 2>/dev/null
for c in ${NCU_CONFIGS:-2 3 5}; do
  TLS_PROFILE_RANGE=1 timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
    -c 40000 --csv --log-file gpurun_out/m/launches_cfg${c}_$R.csv \
    python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2> gpurun_out/m/ncu_launch_cfg${c}.err
done
for c in ${FULL_CONFIGS:-3}; do
  TLS_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off -k regex:k_band_solve -c 1 --set full --import-source on \
    --clock-control none -f -o /tmp/band_cfg${c}_$R python bench.py --config $c --steps 1 --warmup 3 \
    --no-cpu-baseline > /dev/null 2> gpurun_out/m/ncu_full_cfg${c}.err
  ncu -i /tmp/band_cfg${c}_$R.ncu-rep --page raw --csv > gpurun_out/m/ncu_band_cfg${c}_$R.csv 2>/dev/null
done
du -sh gpurun_out
echo done
