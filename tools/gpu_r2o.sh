set -x
python -m pytest tests -m gpu -q --maxfail=40 -p no:cacheprovider 2>&1 | tail -5
python bench.py --steps 10 --warmup 3 > gpurun_out/r2o_bench.json 2> gpurun_out/r2o_bench.err
echo "bench exit $?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2o_smoke.log 2>&1; echo "smoke exit $?"; tail -2 gpurun_out/r2o_smoke.log
