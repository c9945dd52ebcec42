export DDNM_WIDE_SYNC=1
timeout 120 python tools/wide_dbg.py 341 2>&1 | grep -v "^  File\|^    " | tail -5
