# DMMA hidden layer (hidden_range) vs per-unit DFMA, configs 2 and 3
for i in 1 2; do
echo "== c0 DMMA"; python tools/prof_solve.py c0_nm 4096 | grep solve
echo "== c0 DFMA"; DDNM_HIDDEN_SCALAR=1 python tools/prof_solve.py c0_nm 4096 | grep solve
done
echo "== c3 DMMA"; python tools/prof_solve.py c3_nm 1024 | grep solve
echo "== c3 DFMA"; DDNM_HIDDEN_SCALAR=1 python tools/prof_solve.py c3_nm 1024 | grep solve
python -m pytest tests/test_gpu_parity.py tests/test_units.py -m gpu -q -x 2>&1 | tail -2
