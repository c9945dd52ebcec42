# device phase profile (DDNM_PROF=1) of configs 2/3/4, config 4 slot counts
echo "== c0 prof"; DDNM_PROF=1 python tools/prof_solve.py c0_nm 4096
echo "== c3 prof"; DDNM_PROF=1 python tools/prof_solve.py c3_nm 1024
echo "== c4 (default planner)"; python tools/prof_solve.py c4_nm 256 | grep -E "slots|solve"
echo "== c4 1 slot"; python tools/prof_solve.py c4_nm 256 1 | grep -E "slots|solve"
echo "== c4 prof"; DDNM_PROF=1 python tools/prof_solve.py c4_nm 256
python -m pytest tests/test_subdomain.py tests/test_units.py -m gpu -q 2>&1 | tail -2
