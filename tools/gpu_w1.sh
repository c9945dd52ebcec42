set -x
timeout 300 python tools/wide_check.py c0_nm 64 2>&1 | tail -5
timeout 300 python tools/wide_check.py c0_nm 4096 2>&1 | tail -3
timeout 300 python tools/wide_check.py tiny_nm 64 2>&1 | tail -3
