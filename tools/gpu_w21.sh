ncu --set full --clock-control none --import-source on -k regex:k_wide_rows -s 3 -c 1 -o gpurun_out/w21_rows_c3 -f python tools/prof_wide.py c3_nm 1024 1 > gpurun_out/w21.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_wide_dec -s 3 -c 1 -o gpurun_out/w21_dec_c3 -f python tools/prof_wide.py c3_nm 1024 1 > gpurun_out/w21b.log 2>&1
ls -la gpurun_out/w21*
