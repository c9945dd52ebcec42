ncu --set full --clock-control none --import-source on -k regex:k_wide_dec -s 3 -c 1 -o gpurun_out/w10_dec -f python tools/prof_wide.py c0_nm 4096 1 > gpurun_out/w10_ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_dd_step2 -s 3 -c 1 -o gpurun_out/w10_step -f python tools/prof_wide.py c0_nm 4096 1 > gpurun_out/w10_ncu3.log 2>&1
ls gpurun_out/*.ncu-rep
