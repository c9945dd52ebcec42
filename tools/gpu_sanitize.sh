# compute-sanitizer (one tool per call) over every kernel family on small cases
TOOL=${1:-memcheck}
python tools/sanitize_case.py > gpurun_out/sanitize_plain.log 2>&1 && \
compute-sanitizer --tool $TOOL --print-limit 50 python tools/sanitize_case.py > gpurun_out/sanitize_$TOOL.log 2>&1
echo "rc $?"
tail -25 gpurun_out/sanitize_$TOOL.log
