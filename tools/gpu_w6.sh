timeout 120 python tools/wide_dbg.py 341 2000 500 37 1 2>&1 | grep -v "^  File\|^    " | tail -6
timeout 300 python tools/wide_spec_check.py c0_nm 1024 2>&1 | tail -8
timeout 300 python tools/wide_spec_check.py tiny_nm 200 2>&1 | tail -8
