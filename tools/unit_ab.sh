# A/B of evaluation-unit splits on config 2 (c0_nm, 4096 mu) and config 3 (c3_nm, 1024 mu)
for cfg in "none" "90 0" "90 1" "60 0" "45 0" "45 1" "30 0"; do
  set -- $cfg
  if [ "$1" = "none" ]; then
    echo "== whole blocks"; python tools/prof_solve.py c0_nm 4096 | tail -2
  else
    echo "== UNIT_ROWS=$1 JLEVEL=$2"
    DDNM_UNIT_ROWS=$1 DDNM_JLEVEL=$2 python tools/prof_solve.py c0_nm 4096 | grep -E "slots|solve"
  fi
done
for r in 256 128 64; do
  echo "== c3 UNIT_ROWS=$r"; DDNM_UNIT_ROWS=$r python tools/prof_solve.py c3_nm 1024 | grep -E "slots|solve"
done
