# one compute-sanitizer tool per call: bash tools/r2_san.sh memcheck|racecheck|synccheck
TOOL=$1
python tools/sanitize_case.py > gpurun_out/san_plain_$TOOL.log 2>&1 && \
timeout 1500 compute-sanitizer --tool $TOOL --print-limit 50 --error-exitcode 9 python tools/sanitize_case.py > gpurun_out/san_$TOOL.log 2>&1
echo "rc $?" >> gpurun_out/san_$TOOL.log
