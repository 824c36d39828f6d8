#!/bin/bash
# Block-tridiagonal coarse solve (tls_coarse_chain): A/B on configuration 2 (forced on vs the
# default dense inverse), the ncu launch list of one configuration-5 solve and ncu --set full of
# the first launches of the chain kernels.  Outputs under gpurun_out/chain/.
O=gpurun_out/chain
mkdir -p $O
python bench.py --config 2 --no-cpu-baseline > $O/bench_cfg2_dense.json 2> $O/bench_cfg2_dense.err
TLS_A0_CHAIN_MIN=4096 python bench.py --config 2 --no-cpu-baseline > $O/bench_cfg2_chain.json 2> $O/bench_cfg2_chain.err
TLS_PROFILE_RANGE=1 timeout 2400 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
  -c 90000 --csv --log-file $O/launches_cfg5_chain.csv \
  python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2> $O/ncu_launch_cfg5.err
TLS_PROFILE_RANGE=1 timeout 1200 ncu --profile-from-start off -k regex:"k_chain_spmv|k_symv_tiles|k_reduce_tiles" -c 6 --set full \
  --import-source on --clock-control none -f -o /tmp/chain_cfg5 python bench.py --config 5 --steps 1 --warmup 3 \
  --no-cpu-baseline > /dev/null 2> $O/ncu_full_chain.err
ncu -i /tmp/chain_cfg5.ncu-rep --page raw --csv > $O/ncu_chain_cfg5.csv 2>/dev/null
ls -la $O
