for cfg in "4 2" "3 1" "3 2" "2 0" "2 1"; do
  set -- $cfg
  echo "slots=$1 jlevel=$2"
  DDNM_JLEVEL=$2 python tools/prof_solve.py c0_nm 4096 $1 | grep solve
done
