python -m pytest tests -m gpu -q --maxfail=60 -p no:cacheprovider 2>&1 | tail -12
python bench.py --steps 10 --warmup 3 > gpurun_out/w17_bench.json 2> gpurun_out/w17_bench.err; echo "bench exit $?"; tail -3 gpurun_out/w17_bench.err
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
