set -x
python -m pytest tests -m gpu -q --maxfail=40 -p no:cacheprovider 2>&1 | tail -3
python bench.py --steps 10 --warmup 3 > gpurun_out/r2n_bench.json 2> gpurun_out/r2n_bench.err
echo "bench exit $?"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2n_bench_ref.json 2>&1
echo "ref exit $?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2n_smoke.log 2>&1; echo "smoke exit $?"; tail -2 gpurun_out/r2n_smoke.log
