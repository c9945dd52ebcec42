timeout 600 python tools/wide_check.py c3_nm 1024 2>&1 | tail -2
timeout 600 python tools/wide_check.py c4_nm 256 2>&1 | tail -1
timeout 300 python tools/wide_check.py c0_nm 4096 2>&1 | tail -2
timeout 300 python tools/wide_spec_check.py c0_nm 700 2>&1 | tail -3
timeout 300 python tools/wide_check.py tiny_nm 37 2>&1 | tail -2
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/w22_c3.csv python tools/prof_wide.py c3_nm 1024 1 > /dev/null 2>&1
python tools/ncu_agg.py gpurun_out/w22_c3.csv 2>/dev/null | head -3
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/w22_c0.csv python tools/prof_wide.py c0_nm 4096 1 > /dev/null 2>&1
python tools/ncu_agg.py gpurun_out/w22_c0.csv 2>/dev/null | head -4
