#!/bin/bash
# same-box A/B of the reduced-pencil routes on one configuration's setup (GPU box):
#   old     H = F^T A_II F by sparse-row gathers + two triangular solves, no ring-column skipping
#   direct  M = C^T A_GG C - I by two full GEMMs
#   ctac    the same with the zero blocks of C skipped
#   p32     ctac with 32-column subspace-iteration blocks
export CID=${CID:-5} REPS=1
for rep in $(seq 1 ${ROUNDS:-2}); do
  VAR=TLS_PENCIL_DIRECT VALUES="0" bash tools/setup_env_ab.sh 2>&1 | grep setup | sed 's/^/old    /'
  TLS_PENCIL_CTAC=0 VAR=TLS_PENCIL_DIRECT VALUES="1" bash tools/setup_env_ab.sh 2>&1 | grep setup | sed 's/^/direct /'
  VAR=TLS_PENCIL_DIRECT VALUES="1" bash tools/setup_env_ab.sh 2>&1 | grep setup | sed 's/^/ctac   /'
  VAR=TLS_CHEB_P VALUES="32" bash tools/setup_env_ab.sh 2>&1 | grep setup | sed 's/^/p32    /'
done
