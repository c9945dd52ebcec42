python -m pytest tests -m gpu -q --maxfail=60 -p no:cacheprovider 2>&1 | tail -30
python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/w14_bench.json 2> gpurun_out/w14_bench.err; echo "bench exit $?"; tail -3 gpurun_out/w14_bench.err
