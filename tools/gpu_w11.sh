for v in "2 2" "4 2" "4 4" "8 2" "4 3"; do
  set -- $v
  touch paper_2305_15163_b200/csrc/ddnm_wide.cu
  DDNM_NVCC_EXTRA="-DDDNM_WIDE_HU=$1 -DDDNM_WIDE_SU=$2" python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -E "error" | head -3
  echo "== HU=$1 SU=$2"
  ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/w11.csv python tools/prof_wide.py c0_nm 4096 1 > /dev/null 2>&1
  python tools/ncu_agg.py gpurun_out/w11.csv | grep "k_wide_dec"
  python tools/prof_wide.py c0_nm 4096 3 | tail -1
done
