#!/bin/bash
# A/B of the decoder sweep variants on the bench workload (4096 mu, c0_nm)
for v in 0 1 2; do   # 0: per-output sweep (default), 1: chained tensor-core sweep
  echo "DDNM_SWEEP=$v"
  DDNM_SWEEP=$v python tools/prof_solve.py c0_nm 4096
  DDNM_SWEEP=$v DDNM_PROF=1 python tools/prof_solve.py c0_nm 4096 | sed -n 2p
done
