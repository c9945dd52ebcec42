python tools/prof_wide.py c0_nm 4096 4 | tail -1
python tools/prof_wide.py c3_nm 1024 3 | tail -1
python tools/prof_wide.py c4_nm 256 3 | tail -1
