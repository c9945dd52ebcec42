python -m pytest tests -m gpu -q --maxfail=60 -p no:cacheprovider 2>&1 | tail -6
sed -i 's/__global__ void __launch_bounds__(WROW_THREADS, NH == 2 ? 3 : 2) k_wide_rows/__global__ void __launch_bounds__(WROW_THREADS, 2) k_wide_rows/' paper_2305_15163_b200/csrc/ddnm_wide.cu
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -E "error" | head -3
echo "== rows (8,5) with 255 regs, still 3 CTAs requested"
python tools/prof_wide.py c3_nm 1024 3 | tail -1
python tools/prof_wide.py c4_nm 256 3 | tail -1
