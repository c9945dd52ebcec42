# planner ranking (soft cap first) and config-3 unit sizes vs slots per CTA
echo "== c4"; python tools/prof_solve.py c4_nm 256 | grep -E "slots|solve"
echo "== dd16"; python tools/prof_solve.py dd16_nm 1024 | grep -E "slots|solve"
echo "== c0"; python tools/prof_solve.py c0_nm 4096 | grep -E "slots|solve"
for h in 1536 1024 768; do for r in 256 128; do
  echo "== c3 hidden $h rows $r"; DDNM_UNIT_HIDDEN=$h DDNM_UNIT_ROWS=$r python tools/prof_solve.py c3_nm 1024 | grep -E "slots|solve"
  echo "== c3 hidden $h rows $r 4 slots"; DDNM_UNIT_HIDDEN=$h DDNM_UNIT_ROWS=$r python tools/prof_solve.py c3_nm 1024 4 2>&1 | grep -E "slots|solve|Error"
done; done
