python tools/prof_wide.py c0_nm 4096 3 | tail -1
for c in "c3_nm 1024" "c4_nm 256"; do
  set -- $c
  python tools/prof_wide.py $1 $2 2 | tail -1
  ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/w15_$1.csv python tools/prof_wide.py $1 $2 1 > /dev/null 2>&1
  python tools/ncu_agg.py gpurun_out/w15_$1.csv | head -7
done
