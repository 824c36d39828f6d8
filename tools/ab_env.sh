#!/bin/bash
# A/B of a tuning env var on one config, alternating runs (GPU box): VAR, VALUES, CONFIG, REPS
mkdir -p gpurun_out/ab
for rep in $(seq 1 ${REPS:-2}); do
  for v in $VALUES; do
    env $VAR=$v timeout 600 python bench.py --config ${CONFIG:-3} --steps 5 --warmup 3 --no-cpu-baseline \
      > gpurun_out/ab/${VAR}_${v}_$rep.json 2> /dev/null
    python -c "
import json; d=json.loads([l for l in open('gpurun_out/ab/${VAR}_${v}_$rep.json') if l.startswith('{')][-1])
print('$VAR=$v rep $rep', round(d['value'],1), round(d['loop_roofline']['frac'],3), d['clocks']['sm_mhz'])"
  done
done
