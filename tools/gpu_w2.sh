set -x
python tools/prof_wide.py c0_nm 4096 2 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/w2_launches.csv python tools/prof_wide.py c0_nm 4096 1 > gpurun_out/w2_ncu.log 2>&1
tail -2 gpurun_out/w2_ncu.log
