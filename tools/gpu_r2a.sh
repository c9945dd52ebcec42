set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -q --maxfail=30 -p no:cacheprovider > gpurun_out/r2a_pytest.log 2>&1
echo "pytest exit $?"
tail -30 gpurun_out/r2a_pytest.log
python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
echo "bench exit $?"
tail -c 3000 gpurun_out/r2a_bench.json
tail -5 gpurun_out/r2a_bench.err
