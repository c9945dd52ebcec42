timeout 300 python tools/wide_check.py c0_nm 4096 2>&1 | tail -1
DDNM_STEP2=0 timeout 300 python tools/wide_check.py c0_nm 4096 2>&1 | tail -1
DDNM_STEP_FULL=1 timeout 300 python tools/wide_check.py c0_nm 4096 2>&1 | tail -1
timeout 300 python tools/wide_spec_check.py c0_nm 700 2>&1 | tail -3
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/w9_launches.csv python tools/prof_wide.py c0_nm 4096 1 > gpurun_out/w9_ncu.log 2>&1
tail -1 gpurun_out/w9_ncu.log
