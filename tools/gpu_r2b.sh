# round 2, call b: GPU tests, then one ncu --set full capture of k_solve at config 2
set -x
python -m pytest tests -m gpu -q --maxfail=30 -p no:cacheprovider > gpurun_out/r2b_pytest.log 2>&1
echo "pytest exit $?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r2b_pytest.log | tail -30
python tools/prof_solve.py c0_nm 4096 > gpurun_out/r2b_prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_solve -s 1 -c 1 \
    -o gpurun_out/r2b_ksolve python tools/prof_solve.py c0_nm 4096 > gpurun_out/r2b_ncu.log 2>&1
echo "ncu exit $?"
tail -5 gpurun_out/r2b_ncu.log
