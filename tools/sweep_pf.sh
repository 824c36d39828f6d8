#!/bin/bash
# Band-solve prefetch-distance sweep (run on the GPU box): one bench line per (config, pf).
mkdir -p gpurun_out/pf
for c in ${CONFIGS:-3 2}; do
  for pf in ${PFS:-2 3 4 6}; do
    TLS_BAND_PF=$pf timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline \
      > gpurun_out/pf/c${c}_pf${pf}.json 2> gpurun_out/pf/c${c}_pf${pf}.err
  done
done
python - <<'PY'
import glob, json
for f in sorted(glob.glob("gpurun_out/pf/*.json")):
    try:
        d = json.loads([l for l in open(f) if l.startswith("{")][-1])
        print(f, round(d["value"], 1), round(d["roofline"]["frac"], 3), round(d["loop_roofline"]["frac"], 3),
              d["clocks"]["sm_mhz"])
    except Exception as e:
        print(f, "failed", e)
PY
