# config 2 (c0_nm, 4096 mu): hidden layer DMMA vs DFMA, and slot count / Jacobian-row level
run() { echo "== $1"; shift; env "$@" python tools/prof_solve.py c0_nm 4096 $SLOTS | grep -E "slots|solve"; }
SLOTS=0 run "default (DMMA hidden)" X=1
SLOTS=0 run "DFMA hidden" DDNM_HIDDEN_SCALAR=1
SLOTS=2 run "G=2 level 2" DDNM_JLEVEL=2
SLOTS=2 run "G=2 level 1" DDNM_JLEVEL=1
SLOTS=3 run "G=3 level 2" DDNM_JLEVEL=2
SLOTS=4 run "G=4 level 2" DDNM_JLEVEL=2
echo "== c3"; python tools/prof_solve.py c3_nm 1024 | grep -E "slots|solve"
echo "== c3 DFMA hidden"; DDNM_HIDDEN_SCALAR=1 python tools/prof_solve.py c3_nm 1024 | grep -E "slots|solve"
