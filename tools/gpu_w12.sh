touch paper_2305_15163_b200/csrc/ddnm_wide.cu
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -E "error" | head -3
for B in 1 16 64 256 1024; do timeout 300 python tools/wide_check.py c0_nm $B 2>&1 | tail -1; done
timeout 600 python tools/wide_check.py c3_nm 1024 2>&1 | tail -2
timeout 600 python tools/wide_check.py c4_nm 256 2>&1 | tail -2
timeout 600 python tools/wide_check.py c3s_nm 1024 2>&1 | tail -2
timeout 600 python tools/wide_check.py dd16_nm 256 2>&1 | tail -2
timeout 600 python tools/wide_check.py tiny42_nm 64 2>&1 | tail -2
