python -m pytest tests -m gpu -q --maxfail=40 -p no:cacheprovider -rA 2>&1 | grep -E "passed|failed|FAILED|Error|assert" | tail -30
echo "== dd16"; python tools/prof_solve.py dd16_nm 256 | grep -E "slots|solve"
