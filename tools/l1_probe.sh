#!/bin/bash
# does the sweep speed up when W1 fits in L1?  G=2 with the Jacobian rows in L2
# (93 KB smem, ~160 KB L1) vs G=4 (187 KB smem, ~60 KB L1); phase profile
for cfg in "4 2" "2 2" "2 0"; do
  set -- $cfg
  echo "slots=$1 jlevel=$2"
  DDNM_JLEVEL=$2 python tools/prof_solve.py c0_nm 4096 $1 | grep "solve"
  DDNM_JLEVEL=$2 DDNM_PROF=1 python tools/prof_solve.py c0_nm 4096 $1 | sed -n 2p
done
