# configs 3/4 with more slots (eval buffers in L2 for config 4), config 2 level-1 Jacobian rows
echo "== c3"; python tools/prof_solve.py c3_nm 1024 | grep -E "slots|solve"
echo "== c4"; python tools/prof_solve.py c4_nm 256 | grep -E "slots|solve"
echo "== c4 2 slots"; python tools/prof_solve.py c4_nm 256 2 | grep -E "slots|solve"
echo "== c4 no eb in L2"; DDNM_NO_EB_GLOBAL=1 python tools/prof_solve.py c4_nm 256 | grep -E "slots|solve"
echo "== c0"; python tools/prof_solve.py c0_nm 4096 | grep -E "slots|solve"
echo "== c0 level 1 (interface rows in smem, 217 KB)"; DDNM_JLEVEL=1 DDNM_SMEM_SOFT_CAP=232448 python tools/prof_solve.py c0_nm 4096 4 | grep -E "slots|solve"
python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "c3_nm or c4_nm or subdomain or units or dd16" 2>&1 | tail -2
