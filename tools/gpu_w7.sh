timeout 300 python tools/wide_check.py c0_nm 4096 2>&1 | tail -2
timeout 300 python tools/wide_spec_check.py c0_nm 700 2>&1 | tail -8
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/w7_launches.csv python tools/prof_wide.py c0_nm 4096 1 > gpurun_out/w7_ncu.log 2>&1
tail -1 gpurun_out/w7_ncu.log
ncu --set full --clock-control none --import-source on -k regex:k_wide_dec -s 3 -c 1 -o gpurun_out/w7_dec -f python tools/prof_wide.py c0_nm 4096 1 > gpurun_out/w7_ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_wide_rows -s 3 -c 1 -o gpurun_out/w7_rows -f python tools/prof_wide.py c0_nm 4096 1 > gpurun_out/w7_ncu3.log 2>&1
ls -la gpurun_out/*.ncu-rep
