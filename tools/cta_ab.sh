#!/bin/bash
# CTAs per SM x slots: 1 x 512 threads x 4 slots (default) vs 2 x 256 x 2, 4 x 128 x 1
echo "default"; python tools/prof_solve.py c0_nm 4096 | grep "solve \|CTAs"
echo "2x256 G2 L2"; DDNM_THREADS=256 DDNM_JLEVEL=2 python tools/prof_solve.py c0_nm 4096 2 | grep "solve \|CTAs"
echo "2x256 G2 L1"; DDNM_THREADS=256 DDNM_JLEVEL=1 python tools/prof_solve.py c0_nm 4096 2 | grep "solve \|CTAs"
echo "4x128 G1 L2"; DDNM_THREADS=128 DDNM_JLEVEL=2 python tools/prof_solve.py c0_nm 4096 1 | grep "solve \|CTAs"
echo "4x128 G1 L0"; DDNM_THREADS=128 DDNM_JLEVEL=0 python tools/prof_solve.py c0_nm 4096 1 | grep "solve \|CTAs"
echo "2x256 G2 L2 ls"; DDNM_THREADS=256 DDNM_JLEVEL=2 python tools/prof_solve.py c0_ls 4096 2 | grep "solve \|CTAs"
echo "default ls"; python tools/prof_solve.py c0_ls 4096 | grep "solve \|CTAs"
