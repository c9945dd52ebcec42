set -x
python -m pytest tests -m gpu -q --maxfail=60 -p no:cacheprovider 2>&1 | tail -5
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash tools/gpu_r2w.sh
