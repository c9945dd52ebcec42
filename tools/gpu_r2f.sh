set -x
python -m pytest tests -m gpu -q --maxfail=40 -p no:cacheprovider -rA 2>&1 | grep -E "passed|failed|FAILED|Error|n_iter equal|undetermined|assert" > gpurun_out/r2f_pytest.log
tail -60 gpurun_out/r2f_pytest.log
python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err
echo "bench exit $?"
tail -3 gpurun_out/r2f_bench.err
