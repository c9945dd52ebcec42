set -x
python -m pytest tests -m gpu -q --maxfail=30 -p no:cacheprovider -rA 2>&1 | grep -E "passed|failed|FAILED|Error|n_iter equal|undetermined" > gpurun_out/r2d_pytest.log
tail -40 gpurun_out/r2d_pytest.log
bash tools/slot_ab2.sh > gpurun_out/r2d_slot_ab.log 2>&1
cat gpurun_out/r2d_slot_ab.log
