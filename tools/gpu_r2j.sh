set -x
python -m pytest tests -m gpu -q --maxfail=40 -p no:cacheprovider -rA 2>&1 | grep -E "passed|failed|FAILED|Error|n_iter equal|undetermined|assert" > gpurun_out/r2j_pytest.log
tail -40 gpurun_out/r2j_pytest.log
python bench.py --steps 10 --warmup 3 > gpurun_out/r2j_bench.json 2> gpurun_out/r2j_bench.err
echo "bench exit $?"
tail -3 gpurun_out/r2j_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2j_bench_ref.json 2>&1
tail -c 600 gpurun_out/r2j_bench_ref.json
