timeout 300 python tools/wide_check.py c0_nm 4096 2>&1 | tail -2
timeout 300 python tools/wide_spec_check.py c0_nm 700 2>&1 | tail -3
timeout 300 python tools/wide_check.py tiny_nm 64 2>&1 | tail -2
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/w8_launches.csv python tools/prof_wide.py c0_nm 4096 1 > gpurun_out/w8_ncu.log 2>&1
tail -1 gpurun_out/w8_ncu.log
