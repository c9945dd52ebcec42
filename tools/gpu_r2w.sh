# Round-2 (wide engine) measurements: bench lines, ncu launch list, full captures
set -x
python bench.py --steps 10 --warmup 3 > gpurun_out/r2w_bench.json 2> gpurun_out/r2w_bench.err; echo "bench exit $?"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2w_bench_reference.json 2>&1; echo "ref exit $?"
B="python bench.py --steps 1 --warmup 3 --no-cpu --no-subdomain --no-weak"
$B > gpurun_out/r2w_b1.json 2> gpurun_out/r2w_b1.err; echo "exit $?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r2w_launches.csv $B > gpurun_out/r2w_ncu1.log 2>&1
for k in k_wide_dec k_wide_rows k_dd_step2; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 125 -c 1 -o gpurun_out/r2w_$k -f $B > gpurun_out/r2w_ncu_$k.log 2>&1
done
python tools/ncu_summary_wide.py gpurun_out/r2w_launches.csv gpurun_out/r2w_k_wide_dec.ncu-rep gpurun_out/r2w_k_wide_rows.ncu-rep gpurun_out/r2w_k_dd_step2.ncu-rep gpurun_out/r2w_ncu_summary.json > /dev/null
DDNM_PROF=1 python tools/prof_solve.py c0_nm 4096 2>&1 | tail -3
