set -x
python bench.py --steps 10 --warmup 3 > gpurun_out/r2k_bench.json 2> gpurun_out/r2k_bench.err
echo "bench exit $?"
tail -3 gpurun_out/r2k_bench.err
python bench.py --steps 1 --warmup 3 --no-cpu --no-subdomain --no-weak > gpurun_out/r2k_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2k_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu --no-subdomain --no-weak > gpurun_out/r2k_ncu_launch.log 2>&1
echo "ncu launches exit $?"
python tools/prof_solve.py c0_nm 4096 > gpurun_out/r2k_prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_solve -s 2 -c 1 \
    -o gpurun_out/r2k_ksolve python tools/prof_solve.py c0_nm 4096 > gpurun_out/r2k_ncu.log 2>&1
echo "ncu full exit $?"
