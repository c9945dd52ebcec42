# constraint-unit chunk size (interface outputs per unit) at configs 3 and 4
for gc in 256 512 1024 3000; do
  echo "== c3 gchunk $gc"; DDNM_UNIT_GAM=$gc python tools/prof_solve.py c3_nm 1024 | grep -E "slots|solve"
  echo "== c4 gchunk $gc"; DDNM_UNIT_GAM=$gc python tools/prof_solve.py c4_nm 256 | grep -E "slots|solve"
done
